#!/bin/bash
# round record: headline bench line (with clock samples), BASELINE configs as bench lines, vocab sweep (configs[4])
timeout 300 python bench.py > gpurun_out/r01h_bench.json 2>/dev/null; echo headline rc=$?
timeout 300 python bench.py --tokens 8192 --hidden 4096 --vocab 128256 --no-cpu-baseline > gpurun_out/r01h_llama.json 2>/dev/null; echo llama rc=$?
timeout 300 python bench.py --tokens 4096 --hidden 3584 --vocab 32000 --no-cpu-baseline > gpurun_out/r01h_gemma_shard8.json 2>/dev/null; echo gemma rc=$?
timeout 300 python bench.py --tokens 1024 --hidden 512 --vocab 32000 --no-cpu-baseline > gpurun_out/r01h_c1.json 2>/dev/null; echo c1 rc=$?
timeout 600 python tools/vocab_sweep.py > gpurun_out/r01h_vocab_sweep.log 2>&1; echo sweep rc=$?
