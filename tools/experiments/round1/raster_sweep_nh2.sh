#!/bin/bash
# in-step A/B of GEMM tile rasterisation with 256x512 pair tiles (nh=2), interleaved, plus ncu DRAM bytes per GEMM
B="python bench.py --no-cpu-baseline --no-e2e --steps 8 --warmup 3"
CFGS=("" "--opt raster_logits=16" "--opt raster_logits=8" "--opt raster_dx=8" "--opt raster_dx=32" "--opt raster_dx=-8" "--opt raster_dw=-8" "--opt raster_dw=0" "--opt raster_dw=16" "--opt raster_dw=-2")
for rep in 1 2; do
  for cfg in "${CFGS[@]}"; do
    out=$(timeout 200 $B $cfg 2>/dev/null)
    echo "$out" | python -c "import json,sys; d=json.loads(sys.stdin.read()); g=d['roofline']['gemms']; print('%-34s %8.0f tok/s %6.2f ms | logits %.2f dx %.2f dw %.2f | clk %s' % ('$cfg' or 'default', d['value'], d['ms_per_step'], g['logits']['avg_ms'], g['dx']['avg_ms'], g['dw']['avg_ms'], d['clocks']['sm_mhz']))"
  done
done
for cfg in "${CFGS[@]}"; do
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_sm100 -c 3 --csv \
    python bench.py --no-cpu-baseline --no-e2e --steps 1 --warmup 1 $cfg 2>/dev/null > /tmp/n.csv
  python - "$cfg" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open('/tmp/n.csv')) if len(r) > 10]
hdr = rows[0]; ki = hdr.index('Kernel Name'); mi = hdr.index('Metric Name'); vi = hdr.index('Metric Value'); ui = hdr.index('Metric Unit'); ii = hdr.index('ID')
d = {}
for r in rows[1:]:
    d.setdefault(r[ii], {})[r[mi]] = (r[vi], r[ui])
print('%-34s' % (sys.argv[1] or 'default'), ' | '.join('%s rd %s%s wr %s%s t %s%s' % (k, v['dram__bytes_read.sum'][0], v['dram__bytes_read.sum'][1][:1], v['dram__bytes_write.sum'][0], v['dram__bytes_write.sum'][1][:1], v['gpu__time_duration.sum'][0], v['gpu__time_duration.sum'][1]) for k, v in d.items()))
PY
done
