"""Pipelined builds (the e2e pattern of bench.py): two trees on two streams, uploads from pinned
host memory on a third stream, downloads through lod_tree_copy_async while the other tree
builds.  Every downloaded tree must equal the same cloud built alone -- node table, leaf points
and every inner node's voxel run (the arena ORDER of the runs follows the per-depth work lists,
which are filled with atomics, so runs are compared per node) -- the build's host exchanges go
through mapped memory and its K4/K5 through a second stream, so this is the check that neither
leaks between concurrent trees."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _records(n, seed):
    from paper_2302_14801_b200 import _abi
    rng = np.random.default_rng(seed)
    rec = np.zeros((n, 4), np.uint32)
    xyz = rng.random((n, 3)).astype(np.float32)
    xyz[:, 2] = (0.3 * np.sin(6.0 * xyz[:, 0]) * np.cos(4.0 * xyz[:, 1]) + 0.5 + 0.01 * xyz[:, 2]).astype(np.float32)
    rec[:, :3] = xyz.view(np.uint32)
    rec[:, 3] = rng.integers(0, 1 << 24, n, dtype=np.uint32)
    assert _abi.LOD_POINTS_F32 == 0
    return rec.reshape(-1).view(np.uint8)


def _canonical(n_nodes, leaf, vox, nodes):
    """Per node: its fields except the arena offset, then its points (leaf) or voxels (inner)."""
    from paper_2302_14801_b200 import _abi
    tab = np.frombuffer(nodes, _abi.node_dtype(), count=n_nodes)
    leaf = leaf.reshape(-1, 16)
    vox = vox[: 8 * int(sum(tab["count"][tab["child"].max(1) >= 0]))].reshape(-1, 8) if n_nodes else vox
    out = []
    for nd in tab:
        inner = (nd["child"] >= 0).any()
        rows = (vox if inner else leaf)[nd["first"]: nd["first"] + nd["count"]]
        fields = (nd["min"].tobytes(), nd["size"], nd["count"], nd["parent"], nd["cell"].tobytes(), nd["depth"],
                  nd["flags"], nd["child"].tobytes())
        out.append((fields, rows.tobytes()))
    return out


def _download(torch, tree, lib, stream):
    info = tree.info()
    from paper_2302_14801_b200 import _abi
    leaf = torch.empty(info.n_points * 16, dtype=torch.uint8, pin_memory=True)
    vox = torch.empty(max(info.n_voxels * 8, 8), dtype=torch.uint8, pin_memory=True)
    nodes = torch.empty(max(info.n_nodes * _abi.node_dtype().itemsize, 8), dtype=torch.uint8, pin_memory=True)
    _abi.check(lib.lod_tree_copy_async(tree.h, C.c_void_p(leaf.data_ptr()), C.c_void_p(vox.data_ptr()),
                                       C.c_void_p(nodes.data_ptr()), C.c_void_p(stream.cuda_stream)))
    return info, leaf, vox, nodes


@pytest.mark.parametrize("mode", ["average", "first-come"])
def test_pipelined_builds_match_solo_builds(mode):
    import torch
    from paper_2302_14801_b200 import _abi
    from paper_2302_14801_b200.device import DeviceTree, make_config
    from paper_2302_14801_b200.sampling import _mode_code

    code = _mode_code(mode)
    cfg = make_config(2_000)
    clouds = [_records(300_000 + 50_000 * k, seed=k) for k in range(3)]
    lib = _abi.load()

    # reference: each cloud alone on the default stream
    solo = []
    ref_tree = DeviceTree(0)
    cur = torch.cuda.current_stream()
    for rec in clouds:
        d = torch.from_numpy(rec).cuda()
        ref_tree.build(d, len(rec) // 16, _abi.LOD_POINTS_F32, cfg, code, 7, stream=C.c_void_p(cur.cuda_stream))
        info, leaf, vox, nodes = _download(torch, ref_tree, lib, cur)
        torch.cuda.synchronize()
        solo.append((info.n_nodes, info.n_voxels,
                     _canonical(info.n_nodes, leaf.numpy().copy(), vox.numpy().copy(), nodes.numpy().copy())))

    # pipelined: step k builds cloud k % 3 on tree k % 2, upload of k+1 || build k || download k-1
    steps = 6
    trees = [DeviceTree(0), DeviceTree(0)]
    up = torch.cuda.Stream()
    cs = [torch.cuda.Stream(), torch.cuda.Stream()]
    h_in = [torch.from_numpy(c).pin_memory() for c in clouds]
    size = max(len(c) for c in clouds)
    d_stage = [torch.empty(size, dtype=torch.uint8, device="cuda") for _ in range(2)]
    uploaded = [torch.cuda.Event(), torch.cuda.Event()]
    built = [torch.cuda.Event(), torch.cuda.Event()]
    for b in range(2):
        built[b].record(cs[b])
    with torch.cuda.stream(up):
        d_stage[0][: len(clouds[0])].copy_(h_in[0], non_blocking=True)
        uploaded[0].record(up)
    outs = []
    for k in range(steps):
        b = k & 1
        if k + 1 < steps:
            nxt = (k + 1) % 3
            up.wait_event(built[1 - b])
            with torch.cuda.stream(up):
                d_stage[1 - b][: len(clouds[nxt])].copy_(h_in[nxt], non_blocking=True)
                uploaded[1 - b].record(up)
        cs[b].wait_event(uploaded[b])
        n = len(clouds[k % 3]) // 16
        trees[b].build(d_stage[b], n, _abi.LOD_POINTS_F32, cfg, code, 7, stream=C.c_void_p(cs[b].cuda_stream))
        built[b].record(cs[b])
        outs.append(_download(torch, trees[b], lib, cs[b]))
        # the host buffers of step k are only read after the sync below; the tree of step k
        # is rebuilt at step k + 2, after its download on the same stream
    torch.cuda.synchronize()
    for k, (info, leaf, vox, nodes) in enumerate(outs):
        n_nodes, n_vox, canon0 = solo[k % 3]
        assert (info.n_nodes, info.n_voxels) == (n_nodes, n_vox), k
        assert _canonical(info.n_nodes, leaf.numpy(), vox.numpy(), nodes.numpy()) == canon0, k


def test_one_tree_pipeline_with_output_wait():
    """The bench's one-tree e2e pattern: split k+1 runs its first stages while the leaf / node /
    voxel downloads of build k are still in flight (lod_tree_set_output_wait holds back only its
    skeleton and distribute; the caller orders voxelize k+1 after the voxel download).  Every
    download must equal the same cloud built alone."""
    import torch
    from paper_2302_14801_b200 import _abi
    from paper_2302_14801_b200.device import DeviceTree, make_config

    code = _abi.LOD_MODE_AVERAGE
    cfg = make_config(2_000)
    clouds = [_records(400_000 + 30_000 * k, seed=10 + k) for k in range(3)]
    lib = _abi.load()
    solo = []
    ref_tree = DeviceTree(0)
    cur = torch.cuda.current_stream()
    for rec in clouds:
        d = torch.from_numpy(rec).cuda()
        ref_tree.build(d, len(rec) // 16, _abi.LOD_POINTS_F32, cfg, code, 0, stream=C.c_void_p(cur.cuda_stream))
        info, leaf, vox, nodes = _download(torch, ref_tree, lib, cur)
        torch.cuda.synchronize()
        solo.append((info.n_nodes, info.n_voxels,
                     _canonical(info.n_nodes, leaf.numpy().copy(), vox.numpy().copy(), nodes.numpy().copy())))

    tree = DeviceTree(0)
    s, up, dl, dl2, jn = (torch.cuda.Stream() for _ in range(5))
    sp = C.c_void_p(s.cuda_stream)
    ev_split, ev_vox, ev_leaf, ev_voxdl, ev_out, ev_up = (torch.cuda.Event() for _ in range(6))
    h_in = [torch.from_numpy(c).pin_memory() for c in clouds]
    size = max(len(c) for c in clouds)
    d_stage = torch.empty(size, dtype=torch.uint8, device="cuda")
    with torch.cuda.stream(up):
        d_stage[: len(clouds[0])].copy_(h_in[0], non_blocking=True)
        ev_up.record(up)
    ev_voxdl.record(dl2)
    outs = []
    steps = 6
    for k in range(steps):
        n = len(clouds[k % 3]) // 16
        s.wait_event(ev_up)
        if k > 0:
            _abi.check(lib.lod_tree_set_output_wait(tree.h, C.c_void_p(ev_out.cuda_event)))
        tree.split(d_stage, n, _abi.LOD_POINTS_F32, cfg, stream=sp)
        ev_split.record(s)
        if k + 1 < steps:
            nxt = (k + 1) % 3
            up.wait_event(ev_split)
            with torch.cuda.stream(up):
                d_stage[: len(clouds[nxt])].copy_(h_in[nxt], non_blocking=True)
                ev_up.record(up)
        info = tree.info()
        leaf = torch.empty(info.n_points * 16, dtype=torch.uint8, pin_memory=True)
        dl.wait_event(ev_split)
        _abi.check(lib.lod_tree_copy_async(tree.h, C.c_void_p(leaf.data_ptr()), None, None, C.c_void_p(dl.cuda_stream)))
        ev_leaf.record(dl)
        s.wait_event(ev_voxdl)
        tree.voxelize(code, 0, stream=sp)
        ev_vox.record(s)
        info = tree.info()
        vox = torch.empty(max(info.n_voxels * 8, 8), dtype=torch.uint8, pin_memory=True)
        nodes = torch.empty(max(info.n_nodes * _abi.node_dtype().itemsize, 8), dtype=torch.uint8, pin_memory=True)
        dl2.wait_event(ev_vox)
        _abi.check(lib.lod_tree_copy_async(tree.h, None, C.c_void_p(vox.data_ptr()), C.c_void_p(nodes.data_ptr()),
                                           C.c_void_p(dl2.cuda_stream)))
        ev_voxdl.record(dl2)
        jn.wait_event(ev_leaf)
        jn.wait_event(ev_voxdl)
        ev_out.record(jn)
        outs.append((info, leaf, vox, nodes))
    torch.cuda.synchronize()
    for k, (info, leaf, vox, nodes) in enumerate(outs):
        n_nodes, n_vox, canon0 = solo[k % 3]
        assert (info.n_nodes, info.n_voxels) == (n_nodes, n_vox), k
        assert _canonical(info.n_nodes, leaf.numpy(), vox.numpy(), nodes.numpy()) == canon0, k
