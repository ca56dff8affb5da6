# one-shard combine with batched loads: kernel time (ncu launch list, headline) and bitwise check vs the previous build
for v in base head; do
  if [ $v = head ]; then unset VPIPE_LIB; else export VPIPE_LIB=build_variants/pre_ap/libvpipe_b200.so; fi
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_alg2_combine --csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-graph 2>/dev/null | grep k_alg2_combine | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' '; echo " <- $v k_alg2_combine us"
  python - <<PY
import sys, torch
sys.path[:0] = ['.', 'oracle', 'tests']
import oracle
from gpu_helpers import device_case
from paper_2411_05288_b200 import vocab_math as vm
ctx = vm.Context(0)
res = {}
for p, (T, h, V) in ((1, (700, 256, 6000)), (3, (333, 136, 3000))):
    X, W, g = oracle.random_instance(T, h, V, 3)
    _, _, b, Wd = device_case(X, W, g)
    o = vm.run_alg2(ctx, b, vm.shard_weights(Wd, p)); ctx.sync()
    res[p] = {'loss': o.loss.cpu(), 'gx': o.grad_x.cpu()}
torch.save(res, 'gpurun_out/r02bd_$v.pt')
PY
done
python -c "
import torch
a=torch.load('gpurun_out/r02bd_base.pt'); b=torch.load('gpurun_out/r02bd_head.pt')
print('bitwise equal outputs:', all(torch.equal(a[p][k], b[p][k]) for p in a for k in a[p]))"
