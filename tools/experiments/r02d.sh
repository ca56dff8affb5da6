export VPIPE_LOOPBACK_TIMEOUT=120
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29517"
timeout 600 $TR --nproc-per-node 2 bench.py --gpus 2 --dry-run --steps 3 --warmup 3 > gpurun_out/r02d_dry2.json 2> gpurun_out/r02d_dry2.err; echo dry2_rc=$?
tail -c 1500 gpurun_out/r02d_dry2.json; tail -5 gpurun_out/r02d_dry2.err
timeout 600 $TR --nproc-per-node 8 bench.py --gpus 8 --dry-run --steps 3 --warmup 3 > gpurun_out/r02d_dry8.json 2> gpurun_out/r02d_dry8.err; echo dry8_rc=$?
tail -c 1500 gpurun_out/r02d_dry8.json; tail -5 gpurun_out/r02d_dry8.err
timeout 600 $TR --nproc-per-node 4 bench.py --gpus 4 --dry-run --workload input --steps 3 --warmup 3 > gpurun_out/r02d_dry4_input.json 2> gpurun_out/r02d_dry4_input.err; echo dry4in_rc=$?
tail -c 800 gpurun_out/r02d_dry4_input.json; tail -5 gpurun_out/r02d_dry4_input.err
timeout 600 $TR --nproc-per-node 2 bench.py --gpus 2 --dry-run --impl reference --steps 2 --warmup 1 > gpurun_out/r02d_ref2.json 2> gpurun_out/r02d_ref2.err; echo ref2_rc=$?
tail -c 600 gpurun_out/r02d_ref2.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02d_ref.json 2> gpurun_out/r02d_ref.err; echo ref_rc=$?
tail -c 900 gpurun_out/r02d_ref.json
timeout 300 python bench.py --workload input > gpurun_out/r02d_input.json 2> gpurun_out/r02d_input.err; echo in_rc=$?
tail -c 1800 gpurun_out/r02d_input.json
timeout 300 python bench.py --workload input --ids zipf --no-cpu-baseline > gpurun_out/r02d_input_zipf.json 2> gpurun_out/r02d_input_zipf.err; echo inz_rc=$?
tail -c 1500 gpurun_out/r02d_input_zipf.json
timeout 300 python bench.py > gpurun_out/r02d_bench.json 2> gpurun_out/r02d_bench.err; echo bench_rc=$?
tail -c 2500 gpurun_out/r02d_bench.json
