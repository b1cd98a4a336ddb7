"""The C-ABI library loads and exports every symbol its headers declare (CPU only)."""
import ctypes
import os
import re

import pytest

from paper_2511_20048_b200 import spa

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    for h in ("spa.h", "spa_debug.h"):
        text = open(os.path.join(ROOT, "include", h)).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        names |= set(re.findall(r"\b(spa_[a-z0-9_]+)\s*\(", text))
    return sorted(names)


def test_header_declares_the_north_star_calls():
    d = _declared()
    for name in ("spa_kv_alloc", "spa_kv_append", "spa_fork_request", "spa_decode_attention", "spa_merge_splits"):
        assert name in d


@pytest.mark.parametrize("name", _declared())
def test_symbol_exported(name):
    L = spa.lib()
    assert hasattr(L, name), name
    assert name in spa._SIGS, f"{name} has no ctypes signature"


def test_abi_version_and_errors():
    assert spa.spa_abi_version() == 1
    cfg = spa.spa_pool_config(1, 8, 3, 64, 16, 4)   # 8 % 3 != 0
    h = ctypes.c_void_p()
    st = spa.lib().spa_pool_create(ctypes.byref(cfg), None, None, ctypes.byref(h))
    assert st == spa.SPA_ERR_INVALID_ARG
    assert b"num_kv_heads" in spa.lib().spa_last_error()


def test_metadata_only_pool_refuses_device_work():
    pool = spa.Pool(1, 4, 2, 64, 8)
    r = pool.alloc()
    pool.append([r], [3])
    plan = spa.Plan(pool)
    plan.plan([r])
    st = spa.lib().spa_decode_attention(plan.h, 0, None, 0, 0, None, 0, 0, None, 0, 0, 1.0, None)
    assert st == spa.SPA_ERR_NO_DEVICE


def test_no_torch_types_in_header():
    text = open(os.path.join(ROOT, "include", "spa.h")).read()
    for bad in ("torch", "at::", "Tensor"):
        assert bad not in text


def test_peer_argument_errors_without_device():
    """F1 peer calls validate their arguments before touching a device."""
    L = spa.lib()
    h = ctypes.c_void_p()
    for rank, world, nb, nbufs in ((2, 2, 64, 1), (0, 9, 64, 1), (0, 2, 0, 1), (0, 2, 64, 0), (-1, 2, 64, 1)):
        assert L.spa_peer_create(rank, world, nb, nbufs, ctypes.byref(h)) == spa.SPA_ERR_INVALID_ARG
        assert h.value is None
    assert L.spa_decode_attention_fused_gather(None, None, 0, None, 0, 0, 0, 1, 1.0, None) == spa.SPA_ERR_INVALID_ARG
    assert L.spa_peer_connect_local(None, 2) == spa.SPA_ERR_INVALID_ARG
    assert L.spa_peer_destroy(None) == spa.SPA_OK
    assert spa.Peer.buffer_bytes(3, 10, 128) == 7680 + 120
    assert spa.Peer.buffer_bytes(3, 10, 128, with_lse=False) == 7680
