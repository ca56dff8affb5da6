"""Worker of tests/test_gpu_loopback.py::test_fused_c1_across_processes
(launched by torchrun, one process per rank, all on cuda:0): the loopback
group spans processes, so the fused C1's peer buffers are CUDA IPC mappings.
Each rank runs two alg2 steps and checks them against the CPU oracle."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.join(os.path.dirname(HERE), "oracle"))
sys.path.insert(0, HERE)
from gpu_helpers import GRAD_REL_L2, LOSS_ABS, device_case, oracle, rel_l2  # noqa: E402
from paper_2411_05288_b200 import dist as vpd  # noqa: E402
from paper_2411_05288_b200 import vocab_math as vm  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    ctx = vm.Context(0)
    vpd.init_comm(ctx, loopback=True)
    T, h, V = 384, 128, 2048 * world
    report = {"rank": rank}
    for step in range(2):
        X, W, g = oracle.random_instance(T, h, V, 70 + step)
        Xb, Wb, batch, Wd = device_case(X, W, g)
        rb, re = vpd.shard_rows(V, world, rank)
        out = vm.run_alg2(ctx, batch, [vm.EmbeddingShard(Wd[rb:re], rank, rb, re)])
        ctx.sync()
        ref = oracle.oracle_output_layer(Xb, g, Wb, want_softmax=False)
        report[f"loss_err_{step}"] = float(np.abs(out.loss.double().cpu().numpy() - ref.loss).max())
        report[f"gx_rel_{step}"] = rel_l2(out.grad_x[:, :h].double().cpu().numpy(), ref.grad_x)
        report[f"gw_rel_{step}"] = rel_l2(out.grad_w[0][:, :h].double().cpu().numpy(), ref.grad_w[rb:re])
    # the input layer's peer pull reads the owners' rows through the IPC mappings
    tok = torch.from_numpy(np.random.default_rng(5).integers(0, V, 777).astype(np.int64)).cuda()
    Wfull = torch.from_numpy(np.random.default_rng(6).standard_normal((V, h)).astype(np.float32)).to(
        torch.bfloat16).cuda()
    rb, re = vpd.shard_rows(V, world, rank)
    emb = vm.input_forward_gathered(ctx, tok, vm.EmbeddingShard(Wfull[rb:re], rank, rb, re))
    ctx.sync()
    report["input_exact"] = bool(torch.equal(emb, Wfull[tok]))
    report["peer_input"] = ctx.peer_input_count
    report["fused"] = ctx.fused_c1_count
    report["ok"] = all(report[f"loss_err_{s}"] <= LOSS_ABS and report[f"gx_rel_{s}"] <= GRAD_REL_L2 and
                       report[f"gw_rel_{s}"] <= GRAD_REL_L2 for s in range(2)) and report["fused"] == 2 and \
        report["input_exact"] and report["peer_input"] == 1
    with open(os.path.join(sys.argv[1], f"rank{rank}.json"), "w") as f:
        json.dump(report, f)
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
