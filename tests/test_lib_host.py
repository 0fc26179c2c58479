"""libcvr.so on a host without a GPU: it loads, exports every entry point include/cvr.h
declares, and its host-side validation / layout logic works (no compute calls)."""
import ctypes
import os
import re

import pytest

import cvr_synth as cs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2605_29232_b200 import build
    build.build()
    from paper_2605_29232_b200 import lib
    return lib()


def header_functions():
    src = open(os.path.join(ROOT, "include", "cvr.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cvr_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_header_symbol(L):
    fns = header_functions()
    assert len(fns) >= 15
    for f in fns:
        assert hasattr(L, f), f"libcvr.so does not export {f}"
    assert b"sm_100a" in L.cvr_version()


def test_binding_mirrors_header():
    from paper_2605_29232_b200 import _cvr
    assert sorted(n for n, _, _ in _cvr._SIGS) == header_functions()


def test_create_validates_on_host(L):
    from paper_2605_29232_b200 import CvrError, CvrModel
    m = CvrModel(cs.C2, max_batch=4096, max_nnz=1 << 20, allocate=False)
    assert m.x0_ld == 1728 and m.workspace_bytes > 4096 * 1728 * 2 * 2
    m.close()
    m1 = CvrModel(cs.C1, max_batch=256, allocate=False)
    assert m1.x0_ld == 144                                   # fp32 rows padded to 16 bytes
    m1.close()
    with pytest.raises(CvrError, match="act_dtype"):
        CvrModel(cs.C2.with_(act_dtype="f32"), max_batch=16, allocate=False)
    with pytest.raises(CvrError, match="cross_rank"):
        CvrModel(cs.C2.with_(cross_rank=100), max_batch=16, allocate=False)
    with pytest.raises(CvrError, match="world_size"):
        CvrModel(cs.C2, max_batch=16, world_size=2, rank=2, allocate=False)


def test_calls_before_workspace_are_state_errors(L):
    from paper_2605_29232_b200 import CvrModel
    m = CvrModel(cs.C1, max_batch=8, allocate=False)
    ids = (ctypes.c_int * 1)(0)
    ptrs = (ctypes.c_void_p * 1)(16)
    st = (ctypes.c_int64 * 1)(64)
    assert L.cvr_load_tables(m.h, 1, ids, ptrs, st) == 4      # CVR_E_STATE
    assert b"workspace" in L.cvr_last_error(m.h)
    assert L.cvr_dense(m.h, 16, 1, 16, None) == 4
    m.close()


def test_shard_layout_host(L):
    from paper_2605_29232_b200 import CvrModel
    cfg = cs.C3S
    m = CvrModel(cfg, max_batch=8192, max_nnz=1, world_size=8, rank=3, allocate=False)
    s, r = m.shard_buffer_bytes(65536)
    assert s == r == 65536 * 13 * 128 * 2                    # T_pad = ceil(100/8) = 13 slots
    m.close()


def test_nccl_boundary_host(L):
    """S4's boundary on a host without a GPU: the library resolves NCCL at run time (the process's libnccl.so.2)
    and hands out 128-byte unique ids; cvr_comm_init / cvr_exchange before a workspace are state errors."""
    import ctypes as C
    from paper_2605_29232_b200 import CvrModel
    from paper_2605_29232_b200._cvr import comm_unique_id, cvr_nccl_id
    a, b = comm_unique_id(), comm_unique_id()
    assert len(a) == 128 and a != b
    m = CvrModel(cs.C3S, max_batch=64, max_nnz=1, world_size=2, rank=1, allocate=False)
    uid = cvr_nccl_id()
    C.memmove(C.addressof(uid), a, 128)
    assert L.cvr_comm_init(m.h, C.byref(uid), 2, 1) == 4                      # CVR_E_STATE (no workspace)
    assert L.cvr_exchange(m.h, 16, 16, 128, 16, None) == 4
    m.close()


def test_executor_and_serving_args_host(L):
    """Host-side validation of the executor / serving entry points (no GPU needed to reject bad arguments)."""
    import ctypes as C
    import numpy as np
    from paper_2605_29232_b200 import CvrModel
    m = CvrModel(cs.C2, max_batch=64, max_nnz=1, allocate=False)
    assert L.cvr_warm_graphs(m.h, 64, 16, 16) == 4                           # CVR_E_STATE (no workspace)
    from paper_2605_29232_b200._cvr import cvr_call_record
    rec = cvr_call_record()
    assert L.cvr_call_info(m.h, 0, C.byref(rec)) == 4
    m.close()
    t = np.array([0.0, 0.1, 0.05])                                            # arrivals must not decrease
    n = np.ones(3, np.int32)
    lat, bof, disp = np.zeros(3), np.zeros(3, np.int32), np.zeros(3)
    nb = C.c_int()
    assert L.cvr_batcher_simulate(3, t.ctypes.data, n.ctypes.data, 0.001, 8, 0, 16, 0.0, 0.0, lat.ctypes.data,
                                  bof.ctypes.data, disp.ctypes.data, C.byref(nb)) == 1   # CVR_E_ARG


def test_executor_lanes_host(L):
    """Option "lanes" on the host: 1-4 only, unsharded only; the workspace covers every lane (each holds its own copy
    of the model's state); the sub-contexts follow later options."""
    from paper_2605_29232_b200 import CvrModel
    from paper_2605_29232_b200._cvr import CvrError
    one = CvrModel(cs.C2, max_batch=256, max_nnz=1 << 12, allocate=False)
    two = CvrModel(cs.C2, max_batch=256, max_nnz=1 << 12, allocate=False, lanes=2)
    four = CvrModel(cs.C2, max_batch=256, max_nnz=1 << 12, allocate=False, lanes=4)
    assert two.workspace_bytes == 2 * one.workspace_bytes and four.workspace_bytes == 4 * one.workspace_bytes
    assert two.executor_slot(0) == 0 and two.executor_slot(1) == 2 and two.executor_slot(2) == 1
    for bad in (0, 5):
        with pytest.raises(CvrError):
            CvrModel(cs.C2, max_batch=256, allocate=False, lanes=bad)
    with pytest.raises(CvrError):
        CvrModel(cs.C3S, max_batch=64, max_nnz=1, world_size=2, rank=1, allocate=False, lanes=2)
    two.set_option("u_bn", 64)        # forwarded to the sub-context
    with pytest.raises(CvrError):
        two.set_option("u_bn", 65)
    for m in (one, two, four):
        m.close()
