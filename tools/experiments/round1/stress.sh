#!/bin/bash
for i in 1 2; do timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1; done
for i in 1 2 3; do timeout 300 ./tools/gemm_selftest 2>&1 | tail -1; done
for i in 1 2 3; do timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1; done
for i in $(seq 1 5); do timeout 200 python bench.py --no-cpu-baseline --no-e2e --no-graph --steps 30 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['value']), d['clocks']['sm_mhz'])"; done
