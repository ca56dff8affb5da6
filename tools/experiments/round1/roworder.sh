#!/bin/bash
for rep in 1 2; do for o in 0 1; do timeout 120 python bench.py --workload input --no-e2e --opt scatter_row_order=$o 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('row_order=$o', d['value'], d['ms_per_step'], d['roofline']['phase_ms'])"; done; done
timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_rows|k_scatter" -c 8 python bench.py --workload input --steps 1 --warmup 1 --no-e2e --opt scatter_row_order=1 2>&1 | grep -E "^  [a-z_<>v]|duration" | head -12
timeout 600 python -c "
import sys; sys.path[:0]=['.','tests','oracle']
import numpy as np, torch, oracle
from paper_2411_05288_b200 import vocab_math as vm
ctx=vm.Context(0); ctx.set_option('scatter_row_order',1)
for T,V in ((16384,256000),(5000,300),(777,50)):
    rng=np.random.default_rng(T)
    tok=rng.integers(0,V,T); h=64
    g=torch.randn(T,h).to(torch.bfloat16)
    W=torch.zeros(V,h,dtype=torch.bfloat16,device='cuda')
    for p in (1,3):
        for s in vm.shard_weights(W,p) if V%p==0 else vm.shard_weights(W,1):
            dE=vm.input_backward(ctx,g.cuda(),torch.from_numpy(tok).cuda(),s)
            ref=oracle.input_backward_f32(g.float().numpy(),tok,s.rows(),s.row_begin)
            ctx.sync(); assert np.array_equal(dE.cpu().numpy(),ref),(T,V,p)
print('row-order scatter bit-exact')
"
