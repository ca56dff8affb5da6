"""Shared helpers for the GPU parity tests (host side only)."""
import numpy as np
import torch

import oracle
from paper_2411_05288_b200 import vocab_math as vm


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round to bf16 (RNE) and widen back to float64: the operands both sides see."""
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16).to(torch.float64).numpy()


def pad8(h: int) -> int:
    return (h + 7) // 8 * 8


def to_dev_bf16(a: np.ndarray, hp: int) -> torch.Tensor:
    t = torch.zeros(a.shape[0], hp, dtype=torch.bfloat16, device="cuda")
    t[:, :a.shape[1]] = torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16).cuda()
    return t


def rel_l2(a, b) -> float:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def device_case(X, W, labels):
    """bf16-rounded reference operands -> (host X, host W, batch, W_dev)."""
    Xb, Wb = bf16_round(X), bf16_round(W)
    hp = pad8(X.shape[1])
    batch = vm.TokenBatch(to_dev_bf16(Xb, hp), torch.from_numpy(np.asarray(labels, np.int64)).cuda())
    return Xb, Wb, batch, to_dev_bf16(Wb, hp)


def run_device(ctx, alg, batch, Wd, p, h, fault_scale=1.0, with_softmax=True):
    shards = vm.shard_weights(Wd, p)
    fn = {"naive": vm.run_naive, "alg1": vm.run_alg1, "alg2": vm.run_alg2}[alg]
    kw = {} if alg == "naive" else {"fault_scale": fault_scale}
    out = fn(ctx, batch, shards, with_softmax=with_softmax, **kw)
    ctx.sync()
    res = {
        "loss": out.loss.cpu().numpy().astype(np.float64),
        "grad_x": out.grad_x[:, :h].cpu().numpy().astype(np.float64),
        "grad_w": out.grad_w_full()[:, :h].cpu().numpy().astype(np.float64),
    }
    if with_softmax:
        res["softmax"] = out.softmax.cpu().numpy().astype(np.float64)
    return res, out


# north_star tolerances (BASELINE.json): loss 1e-3 absolute; gradients 1e-2 relative L2
LOSS_ABS = 1e-3
GRAD_REL_L2 = 1e-2
SOFTMAX_ABS = 4e-3  # bf16 storage of P: 2^-8 relative at values <= 1


def assert_parity(res, ref, what=""):
    dl = np.abs(res["loss"] - ref.loss).max()
    gx = rel_l2(res["grad_x"], ref.grad_x)
    gw = rel_l2(res["grad_w"], ref.grad_w)
    msg = f"{what}: loss {dl:.2e} gx {gx:.2e} gw {gw:.2e}"
    assert dl <= LOSS_ABS, msg
    assert gx <= GRAD_REL_L2, msg
    assert gw <= GRAD_REL_L2, msg
    if "softmax" in res and ref.softmax is not None:
        ds = np.abs(res["softmax"] - ref.softmax).max()
        assert ds <= SOFTMAX_ABS, f"{what}: softmax {ds:.2e}"
    return dl, gx, gw


__all__ = ["oracle", "bf16_round", "pad8", "to_dev_bf16", "rel_l2", "device_case", "run_device", "assert_parity",
           "LOSS_ABS", "GRAD_REL_L2", "SOFTMAX_ABS"]
