# debug: fused exchange captured on a 1-rank NCCL group vs eager on the same context
import os, sys
sys.path[:0] = [os.getcwd(), os.path.join(os.getcwd(), "oracle"), os.path.join(os.getcwd(), "tests")]
import torch, numpy as np, oracle
from gpu_helpers import device_case
from paper_2411_05288_b200 import vocab_math as vm
stream = torch.cuda.Stream()
with torch.cuda.stream(stream):
    X, W, g = oracle.random_instance(256, 128, 1024, 8)
    _, _, batch, Wd = device_case(X, W, g)
    shards = vm.shard_weights(Wd, 1)
    nctx = vm.Context(0)
    nctx.comm_init(1, 0, vm.Context.unique_id())
    nctx.set_option("force_collectives", 1)
    for ov in (1, 0):
        nctx.set_option("overlap_c1", ov)
        states = [vm.ShardState(nctx, 256, 128, shards[0].rows())]
        outs = vm._alloc_outputs(nctx, batch, shards)
        vm.run_alg2(nctx, batch, shards, states=states, outputs=outs)
        nctx.sync()
        e_gx = outs[1].clone(); e_loss = outs[0].clone()
        outs[1].zero_(); outs[0].zero_()
        graph = vm.capture(nctx, lambda: vm.run_alg2(nctx, batch, shards, states=states, outputs=outs))
        graph.launch(); nctx.sync(); torch.cuda.synchronize()
        d = (outs[1] - e_gx).abs()
        print("overlap", ov, "loss eq", torch.equal(outs[0], e_loss), "gx eq", torch.equal(outs[1], e_gx),
              "max diff", d.max().item(), "rows differing", int((d.amax(1) > 0).sum()), "gx zero rows", int((outs[1].abs().amax(1) == 0).sum()))
        graph.close()
