"""CPU-side checks of the C-ABI library: it loads, exports every symbol the
header declares, and validates arguments on the host (no GPU needed: every
rejected call returns before touching the device)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2602_06283_b200 import build
    build.build()
    from paper_2602_06283_b200 import _lib
    return _lib.lib()


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "socket_b200.h")).read()
    return sorted(set(re.findall(r"\b(socket_[a-z_]+)\s*\(", txt)))


def test_exports_match_header(L):
    from paper_2602_06283_b200 import _lib
    declared = header_symbols()
    assert sorted(_lib.EXPORTS) == declared
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r" T (socket_\w+)", out))
    missing = [s for s in declared if s not in exported]
    assert not missing, missing


def test_library_is_sm100a(L):
    from paper_2602_06283_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_slots(L):
    assert L.socket_version() == 4
    assert [L.socket_code_slots(x) for x in (0, 1, 8, 9, 16, 17, 32, 33, 60, 64, 65, 128)] == \
        [0, 8, 8, 16, 16, 32, 32, 64, 64, 64, 96, 128]


def _cfg(**kw):
    from paper_2602_06283_b200._lib import SocketCfg
    base = dict(B=1, H_q=4, H_kv=1, d=128, N_max=64, L=16, P=8, tau=0.5, sm_scale=0.088, group_mode=0)
    base.update(kw)
    return SocketCfg(**base)


@pytest.mark.parametrize("bad,status", [
    (dict(L=0), 1), (dict(P=0), 1), (dict(P=17), 1), (dict(tau=0.0), 1),
    (dict(tau=-1.0), 1), (dict(d=64), 2), (dict(d=0), 1), (dict(H_q=6, H_kv=4), 1),
    (dict(N_max=100), 1), (dict(group_mode=7), 1), (dict(L=200), 2), (dict(scoring=2), 1),
    (dict(flags=4), 1), (dict(index_base=-1), 1),
])
def test_invalid_config_rejected(L, bad, status):
    c = _cfg(**bad)
    dummy = ctypes.c_void_p(16)
    st = L.socket_hash_keys(ctypes.byref(c), dummy, None, 0, 1, dummy, dummy, None, None)
    assert st == status
    assert len(L.socket_last_error()) > 0


def test_invalid_arguments_rejected(L):
    c = _cfg()
    d = ctypes.c_void_p(16)
    # null required pointer
    assert L.socket_hash_keys(ctypes.byref(c), None, None, 0, 1, d, d, None, None) == 1
    # V without vnorm
    assert L.socket_hash_keys(ctypes.byref(c), d, d, 0, 1, d, d, None, None) == 1
    # range past N_max
    assert L.socket_hash_keys(ctypes.byref(c), d, None, 60, 5, d, d, None, None) == 1
    # k <= 0, sink + window > k
    assert L.socket_topk(ctypes.byref(c), d, d, 0, 0, 0, d, d, None, None, 0, None) == 1
    assert L.socket_topk(ctypes.byref(c), d, d, 4, 3, 2, d, d, None, None, 0, None) == 1
    assert L.socket_topk(ctypes.byref(c), d, d, 65, 0, 0, d, d, None, None, 0, None) == 1
    # sparse decode with too small a workspace (checked on the host, no launch)
    need = L.socket_workspace_bytes(ctypes.byref(c), 4, 16)
    assert need > 0
    assert L.socket_sparse_decode(ctypes.byref(c), d, d, d, d, d, 16, d, None, None, d, 16, None) == 4
    # shard protocol: rank / shard count / Q out of range
    assert L.socket_topk_resolve(ctypes.byref(c), d, 2, 2, d, None) == 1
    assert L.socket_topk_resolve(ctypes.byref(c), d, 65, 0, d, None) == 1
    assert L.socket_topk_digest(ctypes.byref(c), d, d, 4, 0, 0, 0, 64, d, None, 0, None) == 1
    assert L.socket_topk_digest(ctypes.byref(c), d, d, 4, 0, 0, 2, 2, d, None, 0, None) == 1
    assert L.socket_topk_bracket(ctypes.byref(c), d, 2, 64, 0, d, None) == 1
    assert L.socket_topk_emit(ctypes.byref(c), d, d, 4, 3, 2, d, d, d, None, None, 0, None) == 1
    # the decode step and sampling are single-buffer calls: index_base must be 0
    cs = _cfg(index_base=64)
    need = L.socket_workspace_bytes(ctypes.byref(cs), 7, 8)
    assert L.socket_decode_step(ctypes.byref(cs), d, d, d, d, d, d, d, None, 0, None, None, 8, 0, 0,
                                d, d, d, d, None, d, need, None) == 2
    # null cfg
    assert L.socket_query_tables(None, d, d, d, None) == 1


def test_workspace_sizes(L):
    c = _cfg(B=2, H_q=32, H_kv=8, N_max=32768, L=60)
    # score LUT: one 64-KB image per selection row (KV_SHARED: 2*8 rows)
    assert L.socket_workspace_bytes(ctypes.byref(c), 2, 0) == 2 * 8 * 65536
    c2 = _cfg(B=2, H_q=32, H_kv=8, N_max=32768, L=60, group_mode=1)
    assert L.socket_workspace_bytes(ctypes.byref(c2), 2, 0) == 2 * 32 * 65536
    # decode: split partials (m, l, o[128]) per (b, q head, split) + one ticket per unit
    w = L.socket_workspace_bytes(ctypes.byref(c), 4, 3277)
    assert w >= 2 * 32 * 130 * 4 + 2 * 8 * 4
    # top-k: rows that fit one cluster's shared memory need no workspace; 1M-key
    # rows keep their key slices in it (4 B per key)
    assert L.socket_workspace_bytes(ctypes.byref(c), 3, 3277) == 0
    c3 = _cfg(B=1, H_q=32, H_kv=8, N_max=1 << 20, L=60)
    assert L.socket_workspace_bytes(ctypes.byref(c3), 3, 104858) == 8 * (1 << 20) * 4
