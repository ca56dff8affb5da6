"""Python mirror of the reference vocab-math API over device tensors.

Same names, argument order and error behaviour as the reference's
/root/reference/proj/include/vpipe/vocab_math.hpp (VM.hpp) so the parity
tests read like P/tests/test_vocab_math.cpp; the arithmetic is the sm_100a
path behind include/vpipe_b200.h (libvpipe_b200.so) — there is no other.

PyTorch only provides device memory and the stream (plumbing): every
tensor here is a CUDA tensor handed to the C ABI by pointer.

    ctx = Context(0)
    batch = TokenBatch(X_bf16, labels_i64)            # device tensors
    shards = shard_weights(W_bf16, p)                  # row views of W
    out = run_alg2(ctx, batch, shards)                 # loss, grad_x, grad_w, stats

std::invalid_argument in the reference maps to ValueError here.
"""
from __future__ import annotations

import ctypes
import weakref
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import torch

from . import _lib
from ._lib import check, vp_batch_t, vp_shard_t, vp_stats_t


def _p(t: Optional[torch.Tensor]) -> ctypes.c_void_p:
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def _need_cuda(t: torch.Tensor, dtype: torch.dtype, what: str) -> None:
    if not t.is_cuda:
        raise ValueError(f"{what}: expected a CUDA tensor")
    if t.dtype != dtype:
        raise ValueError(f"{what}: expected {dtype}, got {t.dtype}")


class Context:
    """One device (vp_ctx_t).  Runs on torch's current stream of that device
    so torch-allocated buffers and the library's kernels stay ordered."""

    def __init__(self, device: int = 0, cta_group: int = 2):
        self.lib = _lib.load()
        self.device = int(device)
        self._states = weakref.WeakSet()  # states must die before the context
        h = ctypes.c_void_p()
        check(self.lib.vp_ctx_create(self.device, ctypes.byref(h)))
        self.handle = h
        with torch.cuda.device(self.device):
            self.stream = torch.cuda.current_stream()
            self.use_stream(self.stream)
        if cta_group != 2:
            self.set_option("cta_group", cta_group)

    def use_stream(self, stream: torch.cuda.Stream) -> None:
        self.stream = stream
        check(self.lib.vp_ctx_set_stream(self.handle, ctypes.c_void_p(stream.cuda_stream)))

    def set_option(self, key: str, value: int) -> None:
        check(self.lib.vp_ctx_set_option(self.handle, key.encode(), int(value)))

    def reserve(self, n_tok: int, h: int, p: int = 1) -> None:
        check(self.lib.vp_ctx_reserve(self.handle, n_tok, h, p))

    def sync(self) -> None:
        """Waits for the stream and raises deferred device-side argument errors."""
        check(self.lib.vp_ctx_sync(self.handle))

    @property
    def launches(self) -> int:
        return int(self.lib.vp_ctx_launch_count(self.handle))

    @property
    def fused_c1_count(self) -> int:
        """Fused C1 exchanges run so far (dX GEMM -> owner over peer memory)."""
        return int(self.lib.vp_ctx_fused_c1_count(self.handle))

    @property
    def peer_input_count(self) -> int:
        """Input forwards that pulled their rows over peer memory."""
        return int(self.lib.vp_ctx_peer_input_count(self.handle))

    def gemm_timing(self, enable: bool):
        """Accumulated (ms, launches) per GEMM kind since the last call
        (logits, logits_f32, dx, dw), then switches event timing on/off."""
        ms = (ctypes.c_double * 4)()
        n = (ctypes.c_int64 * 4)()
        check(self.lib.vp_ctx_gemm_timing(self.handle, int(enable), ms, n))
        names = ("logits", "logits_f32", "dx", "dw")
        return {k: (ms[i], n[i]) for i, k in enumerate(names)}

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        check(_lib.load().vp_comm_unique_id(buf))
        return buf.raw

    @staticmethod
    def loopback_id() -> bytes:
        """Id of a loopback group (ranks may share one GPU; see vpipe_b200.h)."""
        buf = ctypes.create_string_buffer(128)
        check(_lib.load().vp_comm_loopback_id(buf))
        return buf.raw

    @property
    def comm_backend(self) -> str:
        return self.lib.vp_ctx_comm_backend(self.handle).decode()

    def comm_init(self, nranks: int, rank: int, uid: bytes) -> None:
        buf = ctypes.create_string_buffer(uid, 128)
        check(self.lib.vp_ctx_comm_init(self.handle, nranks, rank, buf))

    def comm_info(self):
        n, r = ctypes.c_int(), ctypes.c_int()
        check(self.lib.vp_ctx_comm_info(self.handle, ctypes.byref(n), ctypes.byref(r)))
        return n.value, r.value

    def close(self) -> None:
        if getattr(self, "handle", None):
            for st in list(self._states):
                st.close()
            check(self.lib.vp_ctx_destroy(self.handle))
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def init_group(ctxs: Sequence["Context"]) -> None:
    """vp_comm_init_all: ctxs[k] becomes rank k of one group — NCCL when the
    contexts sit on distinct GPUs, the loopback backend when some share one."""
    arr = (ctypes.c_void_p * len(ctxs))(*[c.handle.value for c in ctxs])
    check(_lib.load().vp_comm_init_all(arr, len(ctxs)))


@dataclass
class TokenBatch:
    """VM.hpp:15-18.  X bf16 [n_tok, h] (h % 8 == 0), labels int64 [n_tok]."""
    X: torch.Tensor
    labels: Optional[torch.Tensor]

    def c(self) -> vp_batch_t:
        _need_cuda(self.X, torch.bfloat16, "TokenBatch.X")
        if self.X.dim() != 2 or self.X.stride(1) != 1:
            raise ValueError("TokenBatch: X must be a row-major 2-D tensor")
        if self.labels is not None:
            _need_cuda(self.labels, torch.int64, "TokenBatch.labels")
            if self.labels.numel() != self.X.shape[0]:
                raise ValueError("TokenBatch: labels/X row mismatch")
        return vp_batch_t(self.X.data_ptr(), self.X.stride(0),
                          0 if self.labels is None else self.labels.data_ptr(), self.X.shape[0], self.X.shape[1])


@dataclass
class EmbeddingShard:
    """VM.hpp:21-31: rows [row_begin, row_end) of W (a device view)."""
    W: torch.Tensor
    index: int = 0
    row_begin: int = 0
    row_end: int = 0

    def rows(self) -> int:
        return self.row_end - self.row_begin

    def owns(self, vocab_row: int) -> bool:
        return self.row_begin <= vocab_row < self.row_end

    def c(self) -> vp_shard_t:
        _need_cuda(self.W, torch.bfloat16, "EmbeddingShard.W")
        if self.W.shape[0] != self.rows():
            raise ValueError("EmbeddingShard: W rows != row_end - row_begin")
        return vp_shard_t(self.W.data_ptr(), self.W.stride(0), self.row_begin, self.row_end, self.index)


@dataclass
class GlobalStats:
    """VM.hpp:45-48: fp32 [n_tok] device tensors."""
    m: torch.Tensor
    sum: torch.Tensor

    @staticmethod
    def empty(n: int, device) -> "GlobalStats":
        return GlobalStats(torch.empty(n, dtype=torch.float32, device=device),
                           torch.empty(n, dtype=torch.float32, device=device))

    def c(self) -> vp_stats_t:
        return vp_stats_t(self.m.data_ptr(), self.sum.data_ptr())


LocalStats = GlobalStats  # VM.hpp:58-61 has the same two fields


class ShardState:
    """VM.hpp:34-43.  Device buffers owned by the library (vp_state_t)."""

    def __init__(self, ctx: Context, n_tok: int, h: int, rows: int):
        self.ctx = ctx
        self.n_tok, self.h, self.rows = int(n_tok), int(h), int(rows)
        hdl = ctypes.c_void_p()
        check(ctx.lib.vp_state_create(ctx.handle, self.n_tok, self.h, self.rows, ctypes.byref(hdl)))
        self.handle = hdl
        self.has_grad_terms = False
        ctx._states.add(self)

    def local_stats(self) -> LocalStats:
        dev = torch.device("cuda", self.ctx.device)
        out = GlobalStats.empty(self.n_tok, dev)
        check(self.ctx.lib.vp_state_copy_local_stats(self.ctx.handle, self.handle, _p(out.m), _p(out.sum)))
        return out

    @property
    def m_local(self) -> torch.Tensor:
        return self.local_stats().m

    @property
    def sum_local(self) -> torch.Tensor:
        return self.local_stats().sum

    @property
    def A(self) -> torch.Tensor:
        out = torch.empty(self.n_tok, self.h, dtype=torch.float32, device=torch.device("cuda", self.ctx.device))
        check(self.ctx.lib.vp_state_copy_grad_terms(self.ctx.handle, self.handle, _p(out), self.h))
        return out

    def softmax(self, stats: GlobalStats) -> torch.Tensor:
        """This shard's columns of the global softmax (assemble_forward, VM.cpp:281-286)."""
        out = torch.empty(self.n_tok, self.rows, dtype=torch.float32, device=torch.device("cuda", self.ctx.device))
        check(self.ctx.lib.vp_shard_softmax(self.ctx.handle, self.handle, stats.c(), _p(out), self.rows))
        return out

    def softmax_local(self) -> torch.Tensor:
        """softmax' (VM.hpp:38): the state's own stats make the Eq. 5 factor 1."""
        return self.softmax(self.local_stats())

    def close(self) -> None:
        if getattr(self, "handle", None) and getattr(self.ctx, "handle", None):
            check(self.ctx.lib.vp_state_destroy(self.handle))
        self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class ShardGrads:  # VM.hpp:63-66
    grad_x_partial: torch.Tensor
    grad_w: torch.Tensor


@dataclass
class BarrierResult:  # VM.hpp:99-102
    stats: GlobalStats
    grad_x: torch.Tensor


@dataclass
class OutputResult:  # VM.hpp:51-56 (+ the stats; softmax assembled on request)
    loss: torch.Tensor
    grad_x: torch.Tensor
    grad_w: List[torch.Tensor]
    stats: GlobalStats
    states: List[ShardState] = field(default_factory=list)
    softmax: Optional[torch.Tensor] = None

    def grad_w_full(self) -> torch.Tensor:
        return torch.cat(self.grad_w, dim=0)


def _states_arr(states: Sequence[ShardState]):
    return (ctypes.c_void_p * len(states))(*[s.handle.value for s in states])


def _shards_arr(shards: Sequence[EmbeddingShard]):
    return (vp_shard_t * len(shards))(*[s.c() for s in shards])


def _dev(ctx: Context) -> torch.device:
    return torch.device("cuda", ctx.device)


# ---------------------------------------------------------------------------
# VM.hpp entry points
# ---------------------------------------------------------------------------
def shard_weights(W: torch.Tensor, p: int) -> List[EmbeddingShard]:
    """VM.cpp:65-80: p contiguous row views of W (no copy)."""
    if p < 1:
        raise ValueError("shard_weights: p must be >= 1")
    V = W.shape[0]
    if V % p != 0:
        raise ValueError("shard_weights: V not divisible by p")
    rows = V // p
    return [EmbeddingShard(W[k * rows:(k + 1) * rows], k, k * rows, (k + 1) * rows) for k in range(p)]


def alg1_pass_S(ctx: Context, batch: TokenBatch, shard: EmbeddingShard,
                state: Optional[ShardState] = None) -> ShardState:
    """VM.cpp:151-162."""
    st = state or ShardState(ctx, batch.X.shape[0], batch.X.shape[1], shard.rows())
    b, s = batch.c(), shard.c()
    check(ctx.lib.vp_alg1_pass_S(ctx.handle, ctypes.byref(b), ctypes.byref(s), st.handle))
    st.has_grad_terms = False
    return st


def alg2_pass_S(ctx: Context, batch: TokenBatch, shard: EmbeddingShard,
                state: Optional[ShardState] = None) -> ShardState:
    """VM.cpp:181-191."""
    st = state or ShardState(ctx, batch.X.shape[0], batch.X.shape[1], shard.rows())
    b, s = batch.c(), shard.c()
    check(ctx.lib.vp_alg2_pass_S(ctx.handle, ctypes.byref(b), ctypes.byref(s), st.handle))
    st.has_grad_terms = True
    return st


def merge_max_sum(ctx: Context, parts, fault_scale: float = 1.0,
                  out: Optional[GlobalStats] = None) -> GlobalStats:
    """VM.cpp:82-101.  `parts` is a list of ShardState (C1 of alg1: NCCL
    all-gather under a comm) or of LocalStats (device m/sum pairs)."""
    if len(parts) == 0:
        raise ValueError("merge_max_sum: empty input")
    if isinstance(parts[0], ShardState):
        n = parts[0].n_tok
        out = out or GlobalStats.empty(n, _dev(ctx))
        check(ctx.lib.vp_merge_max_sum(ctx.handle, _states_arr(parts), len(parts), float(fault_scale), out.c()))
        return out
    n = parts[0].m.numel()
    for prt in parts:
        if prt.m.numel() != n or prt.sum.numel() != n:
            raise ValueError("merge_max_sum: length mismatch")
    m = torch.stack([prt.m.float() for prt in parts]).contiguous()
    s = torch.stack([prt.sum.float() for prt in parts]).contiguous()
    out = out or GlobalStats.empty(n, _dev(ctx))
    check(ctx.lib.vp_merge_stats_raw(ctx.handle, _p(m), _p(s), len(parts), n, n, float(fault_scale), out.c()))
    return out


def alg1_pass_T(ctx: Context, state: ShardState, stats: GlobalStats, batch: TokenBatch, shard: EmbeddingShard,
                grad_x_partial: Optional[torch.Tensor] = None,
                grad_w: Optional[torch.Tensor] = None) -> ShardGrads:
    """VM.cpp:164-179."""
    n, h = batch.X.shape
    gx = grad_x_partial if grad_x_partial is not None else torch.empty(n, h, dtype=torch.float32, device=_dev(ctx))
    gw = grad_w if grad_w is not None else torch.empty(shard.rows(), h, dtype=torch.float32, device=_dev(ctx))
    b, s = batch.c(), shard.c()
    check(ctx.lib.vp_alg1_pass_T(ctx.handle, state.handle, stats.c(), ctypes.byref(b), ctypes.byref(s),
                                 _p(gx), gx.stride(0), _p(gw), gw.stride(0)))
    return ShardGrads(gx, gw)


def reduce_grad_x(ctx: Context, partials: Sequence[torch.Tensor], out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """C2 of alg1 (VM.cpp:322)."""
    n, h = partials[0].shape
    out = out if out is not None else torch.empty(n, h, dtype=torch.float32, device=_dev(ctx))
    arr = (ctypes.c_void_p * len(partials))(*[t.data_ptr() for t in partials])
    check(ctx.lib.vp_reduce_grad_x(ctx.handle, arr, len(partials), n, h, partials[0].stride(0), _p(out),
                                   out.stride(0)))
    return out


def alg2_barrier_C1(ctx: Context, states: Sequence[ShardState], shards: Sequence[EmbeddingShard],
                    batch: TokenBatch, fault_scale: float = 1.0, grad_x: Optional[torch.Tensor] = None,
                    stats: Optional[GlobalStats] = None) -> BarrierResult:
    """VM.cpp:193-211 (fault path :337-350)."""
    if len(states) == 0:
        raise ValueError("alg2_barrier_C1: no states")
    for st in states:
        if not st.has_grad_terms:
            raise ValueError("alg2_barrier_C1: A/B terms missing")
    n, h = batch.X.shape
    gx = grad_x if grad_x is not None else torch.empty(n, h, dtype=torch.float32, device=_dev(ctx))
    stats = stats or GlobalStats.empty(n, _dev(ctx))
    b = batch.c()
    check(ctx.lib.vp_alg2_barrier_C1(ctx.handle, _states_arr(states), _shards_arr(shards), len(states),
                                     ctypes.byref(b), float(fault_scale), stats.c(), _p(gx), gx.stride(0)))
    return BarrierResult(stats, gx)


def alg2_pass_T(ctx: Context, state: ShardState, stats: GlobalStats, batch: TokenBatch, shard: EmbeddingShard,
                grad_w: Optional[torch.Tensor] = None) -> torch.Tensor:
    """VM.cpp:213-225."""
    gw = grad_w if grad_w is not None else torch.empty(shard.rows(), batch.X.shape[1], dtype=torch.float32,
                                                       device=_dev(ctx))
    b, s = batch.c(), shard.c()
    check(ctx.lib.vp_alg2_pass_T(ctx.handle, state.handle, stats.c(), ctypes.byref(b), ctypes.byref(s), _p(gw),
                                 gw.stride(0)))
    return gw


def output_loss(ctx: Context, states: Sequence[ShardState], shards: Sequence[EmbeddingShard], stats: GlobalStats,
                batch: TokenBatch, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """loss_i = m_i + log(sum_i) - Y[i, g_i] at the owner (VM.cpp:287-292)."""
    loss = out if out is not None else torch.empty(batch.X.shape[0], dtype=torch.float32, device=_dev(ctx))
    b = batch.c()
    check(ctx.lib.vp_output_loss(ctx.handle, _states_arr(states), _shards_arr(shards), len(states), stats.c(),
                                 ctypes.byref(b), _p(loss)))
    return loss


def _alloc_outputs(ctx, batch, shards):
    n, h = batch.X.shape
    dev = _dev(ctx)
    return (torch.empty(n, dtype=torch.float32, device=dev), torch.empty(n, h, dtype=torch.float32, device=dev),
            [torch.empty(s.rows(), h, dtype=torch.float32, device=dev) for s in shards], GlobalStats.empty(n, dev))


def _run(fn_name, ctx, batch, shards, fault_scale, states, outputs, with_softmax, chunk_tokens=None):
    n, h = batch.X.shape
    rows_per_state = n if chunk_tokens is None else max(1, min(int(chunk_tokens), n))
    states = states or [ShardState(ctx, rows_per_state, h, s.rows()) for s in shards]
    loss, gx, gw, stats = outputs or _alloc_outputs(ctx, batch, shards)
    b = batch.c()
    gw_arr = (ctypes.c_void_p * len(gw))(*[t.data_ptr() for t in gw])
    args = [ctx.handle, ctypes.byref(b), _shards_arr(shards), _states_arr(states), len(shards)]
    if chunk_tokens is not None:
        args.append(int(chunk_tokens))
    if fn_name != "vp_naive_partitioned_output":
        args.append(float(fault_scale))
    args += [stats.c(), _p(loss), _p(gx), gx.stride(0), gw_arr, gw[0].stride(0)]
    check(getattr(ctx.lib, fn_name)(*args))
    for st in states:
        st.has_grad_terms = fn_name == "vp_run_alg2"
    if chunk_tokens is not None and with_softmax:
        raise ValueError("run_alg2_chunked: states hold only the last chunk (no softmax assembly)")
    out = OutputResult(loss, gx, gw, stats, states)
    if with_softmax:
        out.softmax = torch.cat([st.softmax(stats) for st in states], dim=1)
    return out


def naive_partitioned_output(ctx: Context, batch: TokenBatch, shards: Sequence[EmbeddingShard],
                             states=None, outputs=None, with_softmax: bool = False) -> OutputResult:
    """VM.cpp:103-149 (3 barriers; stores and re-reads fp32 logits)."""
    if len(shards) == 0:
        raise ValueError("naive: no shards")
    return _run("vp_naive_partitioned_output", ctx, batch, shards, 1.0, states, outputs, with_softmax)


def run_alg1(ctx: Context, batch: TokenBatch, shards: Sequence[EmbeddingShard], fault_scale: float = 1.0,
             states=None, outputs=None, with_softmax: bool = False) -> OutputResult:
    """VM.cpp:303-326."""
    return _run("vp_run_alg1", ctx, batch, shards, fault_scale, states, outputs, with_softmax)


def run_alg2(ctx: Context, batch: TokenBatch, shards: Sequence[EmbeddingShard], fault_scale: float = 1.0,
             states=None, outputs=None, with_softmax: bool = False) -> OutputResult:
    """VM.cpp:328-361."""
    return _run("vp_run_alg2", ctx, batch, shards, fault_scale, states, outputs, with_softmax)


def run_alg2_chunked(ctx: Context, batch: TokenBatch, shards: Sequence[EmbeddingShard], chunk_tokens: int,
                     fault_scale: float = 1.0, states=None, outputs=None) -> OutputResult:
    """Memory-bounded run_alg2 (SURVEY §8f-2, R/PAPER.md:498): token chunks of
    at most chunk_tokens rows through S -> C1 -> T with states (P) sized for
    one chunk; dW accumulates over the chunks (vp_run_alg2_chunked)."""
    return _run("vp_run_alg2_chunked", ctx, batch, shards, fault_scale, states, outputs, False, chunk_tokens)


def oracle_output_layer(ctx: Context, batch: TokenBatch, W: torch.Tensor, logit_shift: Optional[torch.Tensor] = None,
                        with_softmax: bool = False) -> OutputResult:
    """VM.cpp:31-63: the monolithic layer (p = 1, Algorithm 2).  logit_shift
    (fp32 [n_tok], VM.cpp:41-43) is added per row to the logits in the K1
    epilogue; the results are shift-invariant."""
    if logit_shift is not None:
        _need_cuda(logit_shift, torch.float32, "logit_shift")
        if logit_shift.numel() != batch.X.shape[0]:
            raise ValueError("oracle_output_layer: logit_shift size mismatch")
    check(ctx.lib.vp_ctx_set_logit_shift(ctx.handle, _p(logit_shift)))
    try:
        return run_alg2(ctx, batch, shard_weights(W, 1), with_softmax=with_softmax)
    finally:
        check(ctx.lib.vp_ctx_set_logit_shift(ctx.handle, _p(None)))


def shard_logits(ctx: Context, batch: TokenBatch, shard: EmbeddingShard) -> torch.Tensor:
    """ShardState::Y (VM.hpp:35) on demand: fp32 X W_k^T [n_tok, rows] (one GEMM)."""
    out = torch.empty(batch.X.shape[0], shard.rows(), dtype=torch.float32, device=_dev(ctx))
    b, s = batch.c(), shard.c()
    check(ctx.lib.vp_shard_logits(ctx.handle, ctypes.byref(b), ctypes.byref(s), _p(out), out.stride(0)))
    return out


def shard_label_rows(ctx: Context, batch: TokenBatch, shard: EmbeddingShard) -> torch.Tensor:
    """ShardState::B (VM.hpp:41) on demand: fp32 G_k W_k [n_tok, h]."""
    out = torch.empty(batch.X.shape[0], batch.X.shape[1], dtype=torch.float32, device=_dev(ctx))
    b, s = batch.c(), shard.c()
    check(ctx.lib.vp_shard_label_rows(ctx.handle, ctypes.byref(b), ctypes.byref(s), _p(out), out.stride(0)))
    return out


def run_naive(ctx: Context, batch: TokenBatch, shards: Sequence[EmbeddingShard], **kw) -> OutputResult:
    """VM.cpp:299-301."""
    return naive_partitioned_output(ctx, batch, shards, **kw)


def input_forward(ctx: Context, tokens: torch.Tensor, shard: EmbeddingShard, out: Optional[torch.Tensor] = None,
                  accumulate: bool = False) -> torch.Tensor:
    """VM.cpp:227-236: bf16 [n_tok, h]; negative tokens raise at ctx.sync()."""
    _need_cuda(tokens, torch.int64, "input_forward tokens")
    n, h = tokens.numel(), shard.W.shape[1]
    if out is None:
        out = torch.empty(n, h, dtype=torch.bfloat16, device=_dev(ctx))
    s = shard.c()
    check(ctx.lib.vp_input_forward(ctx.handle, _p(tokens), n, h, ctypes.byref(s), _p(out), out.stride(0),
                                   int(accumulate)))
    return out


def input_forward_gathered(ctx: Context, tokens: torch.Tensor, shard: EmbeddingShard,
                           out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """The whole input layer forward over the group (input_forward on every
    shard + the all-reduce, R/PAPER.md:582) as an owner gather: every rank gets
    W[tokens] (bf16 [n_tok, h]); bit-exact, about half the bytes."""
    _need_cuda(tokens, torch.int64, "input_forward tokens")
    n, h = tokens.numel(), shard.W.shape[1]
    if out is None:
        out = torch.empty(n, h, dtype=torch.bfloat16, device=_dev(ctx))
    s = shard.c()
    check(ctx.lib.vp_input_forward_gathered(ctx.handle, _p(tokens), n, h, ctypes.byref(s), _p(out), out.stride(0)))
    return out


def input_grad_broadcast(ctx: Context, grad_out: torch.Tensor, root: int) -> torch.Tensor:
    """The pre-backward broadcast of the embedding gradient (R/PAPER.md:582), in place."""
    if grad_out.dtype not in (torch.bfloat16, torch.float32):
        raise ValueError("input_grad_broadcast: grad_out must be bf16 or fp32")
    n, h = grad_out.shape
    check(ctx.lib.vp_input_grad_broadcast(ctx.handle, _p(grad_out), grad_out.stride(0),
                                          int(grad_out.dtype == torch.float32), n, h, int(root)))
    return grad_out


def input_backward(ctx: Context, grad_out: torch.Tensor, tokens: torch.Tensor, shard: EmbeddingShard,
                   out: Optional[torch.Tensor] = None, accumulate: bool = False) -> torch.Tensor:
    """VM.cpp:238-251: fp32 [rows, h], ascending-i deterministic scatter-add."""
    _need_cuda(tokens, torch.int64, "input_backward tokens")
    if grad_out.shape[0] != tokens.numel():
        raise ValueError("input_backward: grad/token length mismatch")
    if grad_out.dtype not in (torch.bfloat16, torch.float32):
        raise ValueError("input_backward: grad_out must be bf16 or fp32")
    n, h = grad_out.shape
    if out is None:
        out = torch.empty(shard.rows(), h, dtype=torch.float32, device=_dev(ctx))
    s = shard.c()
    check(ctx.lib.vp_input_backward(ctx.handle, _p(grad_out), grad_out.stride(0),
                                    int(grad_out.dtype == torch.float32), _p(tokens), n, h, ctypes.byref(s),
                                    _p(out), out.stride(0), int(accumulate)))
    return out


def input_backward_gathered(ctx: Context, grad_out: Optional[torch.Tensor], tokens: torch.Tensor,
                            shard: EmbeddingShard, root: int, h: Optional[int] = None,
                            grad_is_f32: bool = False, out: Optional[torch.Tensor] = None,
                            accumulate: bool = False) -> torch.Tensor:
    """input_grad_broadcast from `root` + input_backward of this rank's shard
    (vp_input_backward_gathered): grad_out [n_tok, h] is read on `root` only
    (None elsewhere); each rank reads just the rows its shard owns."""
    _need_cuda(tokens, torch.int64, "input_backward tokens")
    n = tokens.numel()
    if grad_out is not None:
        if grad_out.shape[0] != n:
            raise ValueError("input_backward: grad/token length mismatch")
        if grad_out.dtype not in (torch.bfloat16, torch.float32):
            raise ValueError("input_backward: grad_out must be bf16 or fp32")
        h = grad_out.shape[1]
        grad_is_f32 = grad_out.dtype == torch.float32
        ldg = grad_out.stride(0)
    else:
        h = h if h is not None else shard.W.shape[1]
        ldg = h
    if out is None:
        out = torch.empty(shard.rows(), h, dtype=torch.float32, device=_dev(ctx))
    s = shard.c()
    check(ctx.lib.vp_input_backward_gathered(ctx.handle, _p(grad_out), ldg, int(grad_is_f32), _p(tokens), n, h,
                                             ctypes.byref(s), _p(out), out.stride(0), int(accumulate), int(root)))
    return out


def workspace_query(n_tok: int, h: int, rows: int, nranks: int = 1) -> dict:
    """Device memory plan of one rank (vp_workspace_query; no GPU needed):
    bytes of one shard state, of the context workspace and of the peer
    buffers of the fused exchanges."""
    a, b, c = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    check(_lib.load().vp_workspace_query(n_tok, h, rows, nranks, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
    return {"state_bytes": a.value, "ctx_bytes": b.value, "peer_bytes": c.value}


def allreduce_sum(ctx: Context, t: torch.Tensor) -> torch.Tensor:
    """In-place sum over the context's NCCL group (no-op without one)."""
    if t.dtype not in (torch.float32, torch.bfloat16):
        raise ValueError("allreduce_sum: fp32 or bf16 only")
    check(ctx.lib.vp_allreduce_sum(ctx.handle, _p(t), t.numel(), 0 if t.dtype == torch.float32 else 1))
    return t


# ---------------------------------------------------------------------------
# Pipeline integration: executing a reference DeviceProgram's vocabulary passes
class Program:
    """A reference DeviceProgram (schedule.hpp:95-100) in serialize_program's text
    form (schedule.cpp:512-529), parsed by the library (vp_program_parse)."""

    def __init__(self, text: str):
        self.lib = _lib.load()
        h = ctypes.c_void_p()
        check(self.lib.vp_program_parse(text.encode(), ctypes.byref(h)))
        self.handle = h
        b, p, n = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        check(self.lib.vp_program_info(h, ctypes.byref(b), ctypes.byref(p), ctypes.byref(n)))
        self.barriers, self.p, self.n = b.value, p.value, n.value

    def validate(self) -> List[str]:
        """validate_dependencies (schedule.cpp:390-447) on the vocabulary passes."""
        buf = ctypes.create_string_buffer(1 << 16)
        cnt = ctypes.c_int()
        check(self.lib.vp_program_validate(self.handle, buf, len(buf), ctypes.byref(cnt)))
        return [ln for ln in buf.value.decode().split("\n") if ln]

    def close(self) -> None:
        if getattr(self, "handle", None):
            self.lib.vp_program_destroy(self.handle)
        self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class ProgramResult:
    loss: List[torch.Tensor]          # per microbatch
    grad_x: List[torch.Tensor]        # per microbatch
    stats: List[GlobalStats]          # per microbatch
    grad_w: List[torch.Tensor]        # per local shard, accumulated over the microbatches
    states: List[List[ShardState]]    # [shard][microbatch]


def run_program(ctx: Context, program: Program, batches: Sequence[TokenBatch], shards: Sequence[EmbeddingShard],
                states=None, outputs: Optional[ProgramResult] = None) -> ProgramResult:
    """Executes the program's vocabulary passes (vp_program_run): locally every
    device with one shard each, or this rank's device in an NCCL group."""
    n = program.n
    if len(batches) != n:
        raise ValueError("run_program: one TokenBatch per microbatch")
    dev = _dev(ctx)
    if outputs is None:
        T, h = batches[0].X.shape
        states = states or [[ShardState(ctx, b.X.shape[0], b.X.shape[1], s.rows()) for b in batches] for s in shards]
        outputs = ProgramResult(
            [torch.empty(b.X.shape[0], dtype=torch.float32, device=dev) for b in batches],
            [torch.empty(b.X.shape[0], b.X.shape[1], dtype=torch.float32, device=dev) for b in batches],
            [GlobalStats.empty(b.X.shape[0], dev) for b in batches],
            [torch.empty(s.rows(), h, dtype=torch.float32, device=dev) for s in shards], states)
    r = outputs
    bs = (vp_batch_t * n)(*[b.c() for b in batches])
    st = (ctypes.c_void_p * (len(shards) * n))(*[x.handle.value for row in r.states for x in row])
    stats = (vp_stats_t * n)(*[x.c() for x in r.stats])
    loss = (ctypes.c_void_p * n)(*[t.data_ptr() for t in r.loss])
    gx = (ctypes.c_void_p * n)(*[t.data_ptr() for t in r.grad_x])
    gw = (ctypes.c_void_p * len(shards))(*[t.data_ptr() for t in r.grad_w])
    check(ctx.lib.vp_program_run(ctx.handle, program.handle, bs, _shards_arr(shards), len(shards), st, stats, loss,
                                 gx, r.grad_x[0].stride(0), gw, r.grad_w[0].stride(0)))
    return r


class Graph:
    """CUDA graph of the context's work (vp_ctx_capture_begin/_end), replayed
    with one launch.  Run the captured calls once eagerly first (workspace)."""

    def __init__(self, ctx: Context, handle: ctypes.c_void_p):
        self.ctx, self.handle = ctx, handle

    def launch(self) -> None:
        check(self.ctx.lib.vp_graph_launch(self.handle, self.ctx.handle))

    def close(self) -> None:
        if getattr(self, "handle", None):
            self.ctx.lib.vp_graph_destroy(self.handle)
        self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def capture(ctx: Context, fn) -> Graph:
    """Captures everything fn() issues on ctx into a Graph."""
    check(ctx.lib.vp_ctx_capture_begin(ctx.handle))
    try:
        fn()
    finally:
        h = ctypes.c_void_p()
        rc = ctx.lib.vp_ctx_capture_end(ctx.handle, ctypes.byref(h))
    check(rc)
    return Graph(ctx, h)


def pad_vocab_size(V: int, p: int) -> int:
    """cost_model.cpp:49-55."""
    if V < 1 or p < 1:
        raise ValueError("pad_vocab_size: V and p must be >= 1")
    a = 2 * p
    return (V + a - 1) // a * a
