"""The drop-in's upload path: host arrays -> HBM as they are -> `lod_pack_points` on the device.

The device-packed records must equal the host packing rule (`device.pack_records`, the record
layout of include/lodb200.h): F32 records for float32 input or float64 input exact in float32,
F64 records otherwise (including NaN, which the split then reports like the reference)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _host(pos, col, fmt=None):
    from paper_2302_14801_b200.device import pack_records
    rec, f = pack_records(pos, col, fmt)
    return rec.view(np.uint8).reshape(-1), f


@pytest.mark.parametrize("case", ["f32", "f64_exact", "f64_inexact", "f64_nan", "f64_huge", "big_f32", "big_f64"])
def test_device_pack_equals_host_pack(case):
    from paper_2302_14801_b200.device import DeviceTree
    rng = np.random.default_rng(1)
    n = 3_000_003 if case.startswith("big") else 100_001
    pos = rng.random((n, 3)) * 100 - 50
    if case in ("f32", "big_f32"):
        pos = pos.astype(np.float32)
    elif case in ("f64_exact", "big_f64"):
        pos = pos.astype(np.float32).astype(np.float64)
    elif case == "f64_nan":
        pos = pos.astype(np.float32).astype(np.float64)
        pos[n // 2, 1] = np.nan
    elif case == "f64_huge":
        pos = pos.astype(np.float32).astype(np.float64)
        pos[7, 0] = 1e300
    col = rng.integers(0, 256, (n, 3)).astype(np.uint8)
    dev = DeviceTree()
    d, fmt = dev.upload(pos, col)[:2]
    exp, efmt = _host(pos, col)
    assert fmt == efmt
    got = d.cpu().numpy()
    if fmt == 0:   # the pad byte of an F32 record is 0 on both sides
        assert np.array_equal(got, exp)
    else:          # F64: compare the meaningful bytes (pad is unspecified)
        g, e = got.reshape(n, 32), exp.reshape(n, 32)
        assert np.array_equal(g[:, :27], e[:, :27])


def test_partition_of_float64_cloud_uses_f32_records_when_exact():
    from paper_2302_14801_b200 import BuildConfig, PointCloud, partition
    rng = np.random.default_rng(2)
    pos = rng.random((200_000, 3)).astype(np.float32).astype(np.float64)
    col = rng.integers(0, 256, (200_000, 3)).astype(np.uint8)
    tree = partition(PointCloud(pos, col), BuildConfig(T=5000))
    assert tree.device_tree.info().point_format == 0
    pos[5] += 1e-12   # no longer exact in float32
    tree = partition(PointCloud(pos, col), BuildConfig(T=5000))
    assert tree.device_tree.info().point_format == 1


def test_trees_allocate_through_torch_and_workspace_estimate():
    """lod_set_allocator routes the trees' buffers through torch's caching allocator (so torch
    sees the HBM they hold); lod_workspace_bytes bounds a surface-like build's need."""
    import torch
    from paper_2302_14801_b200 import BuildConfig, PointCloud, partition, build_lod
    from paper_2302_14801_b200.device import workspace_bytes
    from paper_2302_14801_b200.generators import synthetic_cloud
    pos, col = synthetic_cloud("sphere", 1_000_000, 1)
    before = torch.cuda.memory_allocated()
    tree = partition(PointCloud(pos.astype(np.float64), col), BuildConfig())
    build_lod(tree, "average", 0)
    held = tree.device_tree.device_bytes()
    assert held > 0 and torch.cuda.memory_allocated() - before >= held
    assert workspace_bytes(len(pos)) >= held
    tree.device_tree.close()
    assert torch.cuda.memory_allocated() - before < held
