#!/bin/bash
sample() { nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader,nounits -lms 100 > /tmp/clk.csv & echo $!; }
summ() { python - "$1" <<'PY'
import sys, statistics
v=[l.split(',') for l in open('/tmp/clk.csv') if l.strip()]
v=v[len(v)//4:]
print("   %s: clk median %.0f MHz  power median %.0f W (%d samples)" % (sys.argv[1], statistics.median(float(a) for a,b in v), statistics.median(float(b) for a,b in v), len(v)))
PY
}
for shape in k1 dx dw; do
P=$(sample); python - $shape <<'PY'
import torch, time, sys
s=sys.argv[1]
g=torch.Generator(device='cuda').manual_seed(0)
x=torch.randn(8192,4096,device='cuda',generator=g).to(torch.bfloat16)
w=(torch.randn(256000,4096,device='cuda',generator=g)*0.02).to(torch.bfloat16)
p=(torch.randn(8192,256000,device='cuda',generator=g)*4e-6).to(torch.bfloat16)
f={'k1':lambda: x@w.T, 'dx':lambda: p@w, 'dw':lambda: p.T@x}[s]
for _ in range(2): f()
torch.cuda.synchronize(); t=time.time(); n=0
e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True); e0.record()
while time.time()-t<4: f(); n+=1
e1.record(); torch.cuda.synchronize(); ms=e0.elapsed_time(e1)/n
print("cublas %s: %.3f ms %.0f TFLOP/s" % (s, ms, 2*8192*4096*256000/ms/1e9))
PY
kill $P; summ cublas_$shape
done
for k in "k1 0 2" "dx 16 2" "dw -4 2"; do set -- $k; P=$(sample); VP_NH=$3 timeout 120 ./tools/gemm_probe $1 $2 0 0 250 | head -1; kill $P; summ ours_$1; done
