"""The Python mirror checks every buffer before a pointer reaches the C-ABI
(dtype, device, contiguity, operand and output sizes), so a wrong argument is
an InvalidArgument, never an out-of-bounds device read or write.  These run
without a GPU: validation happens before any launch."""
import numpy as np
import pytest
import torch


@pytest.fixture(scope="module")
def objs(qpk):
    # a PolymulPlan uploads its constants when created; here only its shape
    # matters (validation runs before any call into the library)
    pm = qpk.PolymulPlan.__new__(qpk.PolymulPlan)
    pm._h, pm.p, pm.q, pm.k, pm.m = None, 3, 32, 4, 53
    return dict(plan=qpk.RedqPlan(5, 128, 6, qpk.FLOAT_PREMUL), pm=pm, f=qpk.GfqField(3, 3, 1 << 10))


def test_device_path_rejects_cpu_tensors(qpk, objs):
    with pytest.raises(qpk.InvalidArgument, match="not a CUDA device"):
        objs["plan"].residues(torch.zeros(16, dtype=torch.float64))
    with pytest.raises(qpk.InvalidArgument, match="not a CUDA device"):
        objs["pm"](torch.zeros(16, dtype=torch.uint8), torch.zeros(16, dtype=torch.uint8))
    with pytest.raises(qpk.InvalidArgument, match="not a CUDA device"):
        objs["f"].mul_batch(torch.zeros(9, dtype=torch.uint8), torch.zeros(9, dtype=torch.uint8))


def test_device_path_rejects_wrong_dtypes(qpk, objs):
    with pytest.raises(qpk.InvalidArgument, match="dtype"):
        objs["plan"].residues(torch.zeros(16, dtype=torch.float32))  # 4-byte words on the 8-byte path
    with pytest.raises(qpk.InvalidArgument, match="dtype"):
        objs["f"].gemv(torch.zeros((2, 3), dtype=torch.float32), torch.zeros(3, dtype=torch.int32))


def test_device_path_rejects_non_contiguous_views(qpk, objs):
    with pytest.raises(qpk.InvalidArgument, match="contiguous"):
        objs["plan"].residues(torch.zeros(32, dtype=torch.float64)[::2])


def test_host_path_rejects_short_or_mistyped_outputs(qpk, objs):
    w = np.arange(10, dtype=np.float64)
    with pytest.raises(qpk.InvalidArgument, match="needs 70"):
        objs["plan"].residues(w, out=np.empty((9, 7), np.uint8))
    with pytest.raises(qpk.InvalidArgument, match="numpy uint8"):
        objs["plan"].residues(w, out=np.empty((10, 7), np.int32))
    with pytest.raises(qpk.InvalidArgument, match="C-contiguous"):
        objs["plan"].residues(w, out=np.empty((10, 14), np.uint8)[:, ::2])
    a = np.zeros((8, 4), np.uint8)
    with pytest.raises(qpk.InvalidArgument, match="needs 56"):
        objs["pm"](a, a, out=np.empty((7, 7), np.uint8))
    with pytest.raises(qpk.InvalidArgument, match="needs 14"):
        objs["pm"].fqt_mul(np.zeros(5, np.uint8), np.zeros(10, np.uint8), out=np.empty(13, np.uint8))
    f = objs["f"]
    with pytest.raises(qpk.InvalidArgument, match="needs 12"):
        f.matmul(np.zeros((2, 2, 3), np.uint8), np.zeros((2, 2, 3), np.uint8), 2, 2, 2, out=np.empty(11, np.uint8))
    with pytest.raises(qpk.InvalidArgument, match="needs 4"):
        f.matmul_rep(np.zeros((2, 2), np.uint32), np.zeros((2, 2), np.uint32), out=np.empty(3, np.uint32))


def test_operand_shapes_must_agree(qpk, objs):
    with pytest.raises(qpk.InvalidArgument, match="same n records"):
        objs["pm"](np.zeros((8, 4), np.uint8), np.zeros((7, 4), np.uint8))
    with pytest.raises(qpk.InvalidArgument, match="same n records"):
        objs["f"].mul_batch(np.zeros(9, np.uint8), np.zeros(10, np.uint8))
    with pytest.raises(qpk.InvalidArgument, match="inner dimensions"):
        objs["f"].matmul_rep(np.zeros((2, 3), np.uint32), np.zeros((2, 2), np.uint32))
    with pytest.raises(qpk.InvalidArgument, match="fewer than"):
        objs["f"].matmul(np.zeros(5, np.uint8), np.zeros(12, np.uint8), 2, 2, 2)
    with pytest.raises(qpk.InvalidArgument, match="re-pack"):
        objs["f"].matmul(np.zeros(12, np.uint8), np.zeros(12, np.uint8), 2, 2, 2, repack="nope")
