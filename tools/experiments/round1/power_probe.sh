#!/bin/bash
# clocks / power of cuBLAS vs our tcgen05 GEMM on the same shapes (sustained loops)
sample() { nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader,nounits -lms 100 > /tmp/clk.csv & echo $!; }
summ() { python - "$1" <<'PY'
import sys, statistics
v=[l.split(',') for l in open('/tmp/clk.csv') if l.strip()]
v=v[len(v)//4:]
print("   %s: clk median %.0f MHz  power median %.0f W (%d samples)" % (sys.argv[1], statistics.median(float(a) for a,b in v), statistics.median(float(b) for a,b in v), len(v)))
PY
}
P=$(sample); python - <<'PY'
import torch, time
a=torch.randn(8192,8192,device='cuda',dtype=torch.bfloat16); b=torch.randn(8192,8192,device='cuda',dtype=torch.bfloat16)
for _ in range(3): a@b
torch.cuda.synchronize(); t=time.time(); n=0
e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True); e0.record()
while time.time()-t<4: a@b; n+=1
e1.record(); torch.cuda.synchronize(); ms=e0.elapsed_time(e1)/n
print("cublas 8192^3: %.3f ms %.0f TFLOP/s" % (ms, 2*8192**3/ms/1e9))
PY
kill $P; summ cublas8192
P=$(sample); python - <<'PY'
import torch, time
x=torch.randn(8192,4096,device='cuda',dtype=torch.bfloat16); w=(torch.randn(256000,4096,device='cuda')*0.02).to(torch.bfloat16)
for _ in range(2): x@w.T
torch.cuda.synchronize(); t=time.time(); n=0
e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True); e0.record()
while time.time()-t<4: x@w.T; n+=1
e1.record(); torch.cuda.synchronize(); ms=e0.elapsed_time(e1)/n
print("cublas logits 8192x256000x4096 (bf16 out): %.3f ms %.0f TFLOP/s" % (ms, 2*8192*4096*256000/ms/1e9))
PY
kill $P; summ cublas_logits
for k in sq8192 k1 dx dw; do
  P=$(sample); timeout 120 ./tools/gemm_probe $k 0 0 0 250 | sed 's/^/ours /'; kill $P; summ ours_$k
done

