# early-release K1 + parallel split-K: GPU tests of the output layer, headline bench A/B, small-shape probes
export VP_NH=2 VP_LOCKSTEP=8
timeout 1500 python -m pytest tests/test_gpu_output_layer.py -x -q --durations=8 > gpurun_out/r02k_pytest.log 2>&1; echo pytest_rc=$?
tail -14 gpurun_out/r02k_pytest.log
for rep in 1 2; do
  timeout 300 python bench.py --no-cpu-baseline --no-graph > gpurun_out/r02k_bench_$rep.json 2>/dev/null; echo bench_rc=$?
  python -c "import json;d=json.loads(open('gpurun_out/r02k_bench_$rep.json').read().splitlines()[-1]);print('default', d['value'], d['clocks']['sm_mhz'], {k:round(v['avg_ms'],3) for k,v in d['roofline']['gemms'].items()})"
  timeout 300 python bench.py --no-cpu-baseline --no-graph --no-e2e --opt policyb_logits=1 > gpurun_out/r02k_bench_pb_$rep.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r02k_bench_pb_$rep.json').read().splitlines()[-1]);print('policyb_logits=1', d['value'], d['clocks']['sm_mhz'], {k:round(v['avg_ms'],3) for k,v in d['roofline']['gemms'].items()})"
done
echo "== config0-shaped dX / dW (T=1024 h=512 V=32000)"
for ws in 0 1; do for k in "dx 16" "dw -4"; do set -- $k; VP_T=1024 VP_H=512 VP_WS=$ws VP_SPLIT=-1 timeout 60 ./tools/gemm_probe $1 $2 2 2 50 32000 | tail -1 | sed "s/^/ws=$ws /"; done; done
echo "== llama 8-way shard dX (T=8192 h=4096 V=16032)"
for mk in 128 64; do VP_MINKB=$mk VP_SPLIT=-1 timeout 60 ./tools/gemm_probe dx 16 2 2 30 16032 | tail -1 | sed "s/^/minkb=$mk /"; done
for s in 1 2 3; do VP_SPLIT=$s VP_WS=0 timeout 60 ./tools/gemm_probe dx 16 2 2 30 16032 | tail -1 | sed "s/^/split=$s /"; done
echo "== config sweeps through bench"
timeout 300 python bench.py --tokens 1024 --hidden 512 --vocab 32000 --no-cpu-baseline --no-e2e > gpurun_out/r02k_c0.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/r02k_c0.json').read().splitlines()[-1]);print('c0', d['value'], d['graph'], {k:round(v['tflops'],1) for k,v in d['roofline']['gemms'].items()})"
timeout 300 python bench.py --tokens 1024 --hidden 512 --vocab 32000 --no-cpu-baseline --no-e2e --opt split_workspace=0 > gpurun_out/r02k_c0_nows.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/r02k_c0_nows.json').read().splitlines()[-1]);print('c0 nows', d['value'], {k:round(v['tflops'],1) for k,v in d['roofline']['gemms'].items()})"
