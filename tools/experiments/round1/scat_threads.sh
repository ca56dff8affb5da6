#!/bin/bash
for rep in 1 2; do for t in 256 128 64; do timeout 120 python bench.py --workload input --no-e2e --opt scatter_threads=$t 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$t', d['value'], d['ms_per_step'], d['roofline']['phase_ms'])"; done; done
timeout 600 python -m pytest tests/test_gpu_input_layer.py -m gpu -q 2>&1 | tail -1
