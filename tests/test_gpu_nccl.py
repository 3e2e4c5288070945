"""NCCL plumbing of DSINF_TP_NCCL on one GPU: a 1-rank communicator through the C ABI, and the
symmetric-memory all-reduce buffers (ncclMemAlloc + ncclCommWindowRegister(NCCL_WIN_COLL_SYMMETRIC))
the model uses for its per-layer all-reduces."""
import ctypes as C

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2207_00032_b200 import _capi as capi  # noqa: E402


def test_one_rank_comm_symmetric_window_allreduce():
    torch.cuda.set_device(0)
    uid = (C.c_uint8 * 128)()
    capi.check(capi.lib.dsinf_nccl_get_unique_id(uid))
    comm = C.c_void_p()
    capi.check(capi.lib.dsinf_nccl_comm_create(uid, 1, 0, 0, C.byref(comm)))
    try:
        sym, first = C.c_int32(), C.c_float()
        capi.check(capi.lib.dsinf_nccl_window_check(comm, 12288, C.byref(sym), C.byref(first)))
        assert first.value == 1.0  # sum of ones over 1 rank
        print("symmetric windows:", bool(sym.value))
    finally:
        capi.check(capi.lib.dsinf_nccl_comm_destroy(comm))
