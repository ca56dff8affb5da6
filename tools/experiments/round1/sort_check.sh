#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_input_layer.py tests/test_gpu_output_layer.py -m gpu -q -x 2>&1 | tail -2
for i in 1 2; do timeout 120 python bench.py --workload input 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['value'], d['ms_per_step'], d['roofline']['phase_ms'], d['roofline']['frac'])"; done
timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_sort|k_segment|k_input" -c 6 python bench.py --workload input --steps 1 --warmup 1 --no-e2e 2>&1 | grep -E "k_sort|k_segment|k_input|duration" | head -12
