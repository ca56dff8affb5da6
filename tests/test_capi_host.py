"""CPU-side checks of the drop-in boundary: the C-ABI library loads, exports
every symbol include/vpipe_b200.h declares, and the host logic that needs
no GPU behaves like the reference (no compute calls here)."""
import ctypes
import os
import re
import subprocess

import pytest
import torch

from paper_2411_05288_b200 import _lib
from paper_2411_05288_b200 import vocab_math as vm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "vpipe_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|void\*|const char\*)\s+(vp_\w+)\s*\(", src, re.M)))


def test_header_declares_the_abi():
    syms = declared_symbols()
    assert len(syms) >= 30
    assert set(syms) == set(_lib.SIGNATURES), set(syms) ^ set(_lib.SIGNATURES)


def test_library_loads_and_exports_every_declared_symbol():
    lib = _lib.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (vp_\w+)$", out, re.M))
    assert set(declared_symbols()) <= exported
    assert lib.vp_abi_version() == 1


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "-lelf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass and "UTMALDG" in sass and "LDTM" in sass  # tcgen05.mma, TMA, tcgen05.ld
    assert "HMMA" not in sass.replace("UTCHMMA", "")  # no legacy mma.sync path


def test_context_creation_fails_loudly_without_a_gpu():
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    lib = _lib.load()
    h = ctypes.c_void_p()
    rc = lib.vp_ctx_create(0, ctypes.byref(h))
    assert rc != 0 and lib.vp_last_error()
    with pytest.raises(Exception):
        vm.Context(0)


def test_null_and_shape_errors_map_to_einval():
    lib = _lib.load()
    assert lib.vp_ctx_sync(None) == _lib.VP_EINVAL
    assert b"null context" in lib.vp_last_error()
    with pytest.raises(ValueError):
        _lib.check(lib.vp_ctx_set_option(None, b"cta_group", 2))


def test_peer_memory_entry_points_reject_a_null_context():
    # the exchange counters and the group backward (vp_input_backward_gathered)
    lib = _lib.load()
    assert lib.vp_ctx_fused_c1_count(None) == -1
    assert lib.vp_ctx_peer_input_count(None) == -1
    rc = lib.vp_input_backward_gathered(None, None, 8, 0, None, 4, 8, None, None, 8, 0, 0)
    assert rc == _lib.VP_EINVAL and b"null argument" in lib.vp_last_error()


def test_workspace_query_plans_the_headline_and_an_8_way_shard():
    # host-only memory plan (vp_workspace_query): P dominates a shard state
    T, h, V = 8192, 4096, 256000
    one = vm.workspace_query(T, h, V, 1)
    P = T * V * 2
    stats = 3 * (V // 128) * T * 4
    A = T * h * 4
    assert P + stats + A <= one["state_bytes"] <= P + stats + A + 8 * 2**20  # + per-row arrays, fix lists
    assert one["peer_bytes"] == 0 and one["ctx_bytes"] > T * h * 2
    eight = vm.workspace_query(T, h, V // 8, 8)
    assert eight["state_bytes"] < one["state_bytes"] // 6
    assert eight["peer_bytes"] >= 8 * (T // 8) * h * 4  # slots of the fused exchange
    total = eight["state_bytes"] + eight["ctx_bytes"] + eight["peer_bytes"]
    assert total < 4 * 2**30  # an 8-way shard of the headline fits in a few GB of the 180 GB
    lib = _lib.load()
    assert lib.vp_workspace_query(0, h, V, 1, None, None, None) == _lib.VP_EINVAL


def test_shard_weights_views_and_errors():
    W = torch.arange(12 * 8, dtype=torch.float32).reshape(12, 8).to(torch.bfloat16)
    shards = vm.shard_weights(W, 3)
    assert [(s.index, s.row_begin, s.row_end, s.rows()) for s in shards] == [(0, 0, 4, 4), (1, 4, 8, 4),
                                                                                 (2, 8, 12, 4)]
    assert torch.equal(torch.cat([s.W for s in shards]), W)
    assert shards[1].owns(4) and not shards[1].owns(8)
    with pytest.raises(ValueError, match="V not divisible by p"):
        vm.shard_weights(W, 5)
    with pytest.raises(ValueError, match="p must be >= 1"):
        vm.shard_weights(W, 0)


def test_pad_vocab_size():
    assert vm.pad_vocab_size(256008, 24) == 256032
    assert vm.pad_vocab_size(256000, 8) == 256000
    with pytest.raises(ValueError):
        vm.pad_vocab_size(0, 1)
