# A/B (interleaved): alg2 local combine with the loss fused in (head) vs a separate k_loss (base);
# configs[0] eager / graph and the headline; plus a bitwise check of the two builds' outputs
for rep in 1 2 3; do
  for v in base head; do
    if [ $v = head ]; then unset VPIPE_LIB; else export VPIPE_LIB=build_variants/pre_ap/libvpipe_b200.so; fi
    timeout 300 python bench.py --tokens 1024 --hidden 512 --vocab 32000 --no-cpu-baseline --no-e2e --steps 50 > gpurun_out/r02ba_c0.json 2>/dev/null
    python -c "
import json
c=json.loads(open('gpurun_out/r02ba_c0.json').read().splitlines()[-1])
print('$v', 'c0', round(c['value']/1e6,3), 'graph', round(c['graph']['value']/1e6,3), 'launches/step', c['gpu_launches']/c['steps'])"
  done
done
for v in base head; do
  if [ $v = head ]; then unset VPIPE_LIB; else export VPIPE_LIB=build_variants/pre_ap/libvpipe_b200.so; fi
  python - <<PY
import sys, torch
sys.path[:0] = ['.', 'oracle', 'tests']
import oracle
from gpu_helpers import device_case
from paper_2411_05288_b200 import vocab_math as vm
X, W, g = oracle.random_instance(700, 256, 6000, 3)
_, _, b, Wd = device_case(X, W, g)
ctx = vm.Context(0)
o = vm.run_alg2(ctx, b, vm.shard_weights(Wd, 3)); ctx.sync()
torch.save({'loss': o.loss.cpu(), 'gx': o.grad_x.cpu(), 'gw': o.grad_w_full().cpu()}, 'gpurun_out/r02ba_$v.pt')
PY
done
python -c "
import torch
a=torch.load('gpurun_out/r02ba_base.pt'); b=torch.load('gpurun_out/r02ba_head.pt')
print('bitwise equal outputs:', all(torch.equal(a[k], b[k]) for k in a))"
