"""N > 1 host logic on CPU (world_size 2, gloo): the sharding of the
vocabulary over ranks, the NCCL-id bootstrap helper, the max-over-ranks
timing, and the C1/C2 exchange protocol that libvpipe_b200.so runs with NCCL
(all-gather of the packed [2 x T] stats, k-ordered merge, combine and sum
all-reduce) — each rank computing its shard with the CPU oracle — checked
against the monolithic oracle (<= 1e-10, the reference's grid tolerance); and the fused
exchange's ownership protocol (owner combine in rank order + gather of the owned
rows), bitwise against the one-process combine."""
import json
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _merge(parts_m, parts_s):
    # the order of k_merge_stats (vocab_kernels.cuh) == merge_max_sum (VM.cpp:91-99)
    m = parts_m[0].copy()
    for pm in parts_m[1:]:
        m = np.maximum(m, pm)
    s = np.zeros_like(m)
    for pm, ps in zip(parts_m, parts_s):
        s += ps * np.exp(pm - m)
    return m, s


def _worker(rank, world, port, out_path, case):
    sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
    import oracle
    from paper_2411_05288_b200 import dist as vpd
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, h, V, seed = case["n"], case["h"], case["V"], case["seed"]
    X, W, g = oracle.random_instance(n, h, V, seed)
    if case.get("labels_in_shard0"):
        g = g % (V // world)
    rb, re = vpd.shard_rows(V, world, rank)
    Wk = W[rb:re]
    # pass S of this rank (alg2_pass_S, VM.cpp:181-191) on its shard only
    Y = X @ Wk.T
    m_loc = Y.max(axis=1)
    e = np.exp(Y - m_loc[:, None])
    s_loc = e.sum(axis=1)
    sm = e / s_loc[:, None]
    A = sm @ Wk
    B = np.zeros_like(X)
    own = (g >= rb) & (g < re)
    B[own] = Wk[g[own] - rb]
    # C1: one all-gather of the packed [2 x T] stats, merge in rank order
    packed = torch.from_numpy(np.stack([m_loc, s_loc]))
    gathered = [torch.zeros_like(packed) for _ in range(world)]
    dist.all_gather(gathered, packed)
    gm, gs = _merge([t[0].numpy() for t in gathered], [t[1].numpy() for t in gathered])
    scale = s_loc * np.exp(m_loc - gm) / gs
    gx = torch.from_numpy(A * scale[:, None] - B)
    dist.all_reduce(gx)  # sum over ranks (C1's dX reduce)
    loss = np.zeros(n)
    loss[own] = gm[own] + np.log(gs[own]) - Y[own, g[own] - rb]
    lt = torch.from_numpy(loss)
    dist.all_reduce(lt)
    # pass T: this rank's dW rows
    gy = sm * scale[:, None]
    gy[np.nonzero(own)[0], g[own] - rb] -= 1.0
    gw = torch.from_numpy(gy.T @ X)
    gws = [torch.zeros_like(gw) for _ in range(world)]
    dist.all_gather(gws, gw)
    # helpers used by bench.py
    uid = vpd.broadcast_bytes(bytes(range(128)) if rank == 0 else None)
    mx = vpd.max_over_ranks(float(rank + 1))
    if rank == 0:
        ref = oracle.oracle_output_layer(X, g, W)
        rm, rs = oracle.merge_max_sum([oracle.local_stats(X, W, world, k)[0] for k in range(world)],
                                      [oracle.local_stats(X, W, world, k)[1] for k in range(world)])
        res = {
            "stats": max(float(np.abs(gm - rm).max()), float(np.abs(gs - rs).max())),
            "grad_x": float(np.abs(gx.numpy() - ref.grad_x).max()),
            "loss": float(np.abs(lt.numpy() - ref.loss).max()),
            "grad_w": float(np.abs(torch.cat(gws).numpy() - ref.grad_w).max()),
            "uid_ok": uid == bytes(range(128)),
            "max_over_ranks": mx,
            "ranges": [vpd.shard_rows(V, world, k) for k in range(world)],
        }
        json.dump(res, open(out_path, "w"))
    dist.destroy_process_group()


@pytest.mark.parametrize("case", [
    {"n": 16, "h": 16, "V": 64, "seed": 0},
    {"n": 8, "h": 4, "V": 16, "seed": 2},
    {"n": 12, "h": 8, "V": 32, "seed": 1, "labels_in_shard0": True},
])
def test_two_rank_exchange_protocol_matches_the_oracle(tmp_path, case):
    out = str(tmp_path / "res.json")
    mp.spawn(_worker, args=(2, _free_port(), out, case), nprocs=2, join=True)
    r = json.load(open(out))
    assert r["stats"] <= 1e-12
    assert r["grad_x"] <= 1e-10 and r["loss"] <= 1e-10 and r["grad_w"] <= 1e-10
    assert r["uid_ok"] and r["max_over_ranks"] == 2.0
    V = case["V"]
    assert r["ranges"] == [[0, V // 2], [V // 2, V]]


def test_shard_rows_errors():
    from paper_2411_05288_b200 import dist as vpd
    assert vpd.shard_rows(256000, 8, 7) == (224000, 256000)
    with pytest.raises(ValueError, match="V not divisible by p"):
        vpd.shard_rows(10, 3, 0)


def _fused_worker(rank, world, port, out_path, case):
    # The fused C1 of libvpipe_b200.so (fused_c1, vocab_capi.cu / k_alg2_combine_owned)
    # restated on CPU: token rows owned in blocks of R = ceil(T/N) rounded up to
    # 32; rank k's A_k rows reach their owners (the routed dX epilogue; here a
    # gather), the label rows B come from each label's owner, every owner sums
    # its rows over k in rank order, and the owned rows are gathered.  Checked
    # bitwise against the one-process combine in the same order, and against
    # the oracle.
    sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
    import oracle
    from paper_2411_05288_b200 import dist as vpd
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, h, V, seed = case["n"], case["h"], case["V"], case["seed"]
    X, W, g = oracle.random_instance(n, h, V, seed)
    rb, re = vpd.shard_rows(V, world, rank)
    Wk = W[rb:re]
    Y = X @ Wk.T
    m_loc = Y.max(axis=1)
    e = np.exp(Y - m_loc[:, None])
    s_loc = e.sum(axis=1)
    A = (e / s_loc[:, None]) @ Wk
    own_lab = (g >= rb) & (g < re)
    B = np.zeros_like(X)
    B[own_lab] = Wk[g[own_lab] - rb]
    packed = torch.from_numpy(np.stack([m_loc, s_loc]))
    gathered = [torch.zeros_like(packed) for _ in range(world)]
    dist.all_gather(gathered, packed)
    ms = [t[0].numpy() for t in gathered]
    ss = [t[1].numpy() for t in gathered]
    gm, gs = _merge(ms, ss)
    # routing: every rank's A_k and B_k (only the owners' rows are used)
    As = [torch.zeros(n, h, dtype=torch.float64) for _ in range(world)]
    Bs = [torch.zeros(n, h, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(As, torch.from_numpy(A))
    dist.all_gather(Bs, torch.from_numpy(B))
    bounds = [vpd.shard_rows(V, world, k) for k in range(world)]
    R = -(-n // world)
    R = -(-R // 32) * 32
    lo, hi = min(n, rank * R), min(n, (rank + 1) * R)
    G = np.zeros((R, h))
    for i in range(lo, hi):  # the owner's combine, k in rank order
        acc = np.zeros(h)
        for k in range(world):
            sc = ss[k][i] * np.exp(ms[k][i] - gm[i]) / gs[i]
            b = Bs[k][i].numpy() if bounds[k][0] <= g[i] < bounds[k][1] else 0.0
            acc = acc + (As[k][i].numpy() * sc - b)
        G[i - lo] = acc
    Gs = [torch.zeros(R, h, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(Gs, torch.from_numpy(G))
    gx = torch.cat(Gs)[:n].numpy()
    if rank == 0:
        # one process, every shard, the same order
        want = np.zeros((n, h))
        for i in range(n):
            acc = np.zeros(h)
            for k in range(world):
                sc = ss[k][i] * np.exp(ms[k][i] - gm[i]) / gs[i]
                b = Bs[k][i].numpy() if bounds[k][0] <= g[i] < bounds[k][1] else 0.0
                acc = acc + (As[k][i].numpy() * sc - b)
            want[i] = acc
        ref = oracle.oracle_output_layer(X, g, W)
        json.dump({"bitwise": bool(np.array_equal(gx, want)), "oracle": float(np.abs(gx - ref.grad_x).max()),
                   "R": R}, open(out_path, "w"))
    dist.destroy_process_group()


@pytest.mark.parametrize("case", [
    {"n": 64, "h": 8, "V": 32, "seed": 3},    # T = N * R exactly
    {"n": 45, "h": 8, "V": 32, "seed": 4},    # ragged: rank 1 owns 13 rows
    {"n": 7, "h": 4, "V": 16, "seed": 5},     # rank 1 owns nothing
])
def test_two_rank_fused_exchange_protocol(tmp_path, case):
    out = str(tmp_path / "res.json")
    mp.spawn(_fused_worker, args=(2, _free_port(), out, case), nprocs=2, join=True)
    r = json.load(open(out))
    assert r["bitwise"] and r["oracle"] <= 1e-10 and r["R"] % 32 == 0
