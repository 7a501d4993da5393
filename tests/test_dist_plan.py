"""CPU tests of the multi-GPU host logic: subtree planning, the exchange layout, and the
real collective code path (TorchComm over gloo, world_size 2, CPU tensors)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2302_14801_b200.dist import TorchComm, exchange_layout, plan_subtrees

from oracle import lod_oracle as O


def toy_tree(seed=0, n=40_000, T=1500):
    """A real split (CPU oracle) in node-table form: depth, parent, is_leaf, leaf_node, leaf idx."""
    rng = np.random.default_rng(seed)
    pos = rng.random((n, 3))
    pos[::7] = 0.3 + 0.01 * pos[::7]          # a dense region -> uneven subtrees
    sp = O.split(pos, T=T)
    paths = sorted(sp.nodes, key=lambda p: (len(p), p))
    index = {p: i for i, p in enumerate(paths)}
    depth = np.array([len(p) for p in paths])
    parent = np.array([index[p[:-1]] if p else -1 for p in paths])
    is_leaf = np.array([sp.nodes[p].kind == "leaf" for p in paths])
    leaf_node = np.flatnonzero(is_leaf)
    leaf_idx = [sp.nodes[paths[k]].idx for k in leaf_node]
    return depth, parent, is_leaf, leaf_node, leaf_idx, n


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_plan_covers_every_node_once(world):
    depth, parent, is_leaf, leaf_node, leaf_idx, n = toy_tree()
    counts = np.array([len(i) for i in leaf_idx])
    plan = plan_subtrees(depth, parent, is_leaf, leaf_node, counts, world)
    assert plan.load.sum() == n
    # every node at or below the cut belongs to exactly the owner of its depth-cut ancestor
    for k in range(len(depth)):
        if depth[k] >= plan.cut and not (is_leaf[k] and depth[k] <= plan.cut):
            a = k
            while depth[a] > plan.cut:
                a = parent[a]
            assert plan.node_owner[k] == plan.node_owner[a]
        if is_leaf[k] and depth[k] <= plan.cut:
            assert plan.node_owner[k] == 0
    assert set(plan.leaf_owner.tolist()) <= set(range(world))
    if world > 1 and len(plan.roots) >= world:
        assert plan.load.max() <= 0.75 * n      # LPT spreads the points


def simulate_exchange(leaf_idx, n, world, leaf_owner):
    """Shards -> local leaf buffers (stable) -> layout -> all-to-all -> final buffers (numpy)."""
    bounds = [n * r // world for r in range(world + 1)]
    L = len(leaf_idx)
    all_counts = np.zeros((world, L), np.int64)
    local = []
    for r in range(world):
        segs = [np.asarray(i)[(np.asarray(i) >= bounds[r]) & (np.asarray(i) < bounds[r + 1])] for i in leaf_idx]
        all_counts[r] = [len(s) for s in segs]
        local.append(np.concatenate(segs) if segs else np.zeros(0, np.int64))
    lay = exchange_layout(leaf_owner, all_counts, world)
    send = []
    for r in range(world):
        buf = np.empty(len(local[r]), np.int64)
        for s, d, c in zip(*lay[r]["send"]):
            buf[d:d + c] = local[r][s:s + c]
        send.append(buf)
    finals = []
    for q in range(world):
        recv = np.concatenate([send[r][int(lay[r]["send_splits"][:q].sum()):
                                       int(lay[r]["send_splits"][:q + 1].sum())] for r in range(world)])
        assert len(recv) == lay[q]["recv_splits"].sum()
        final = np.empty(int(lay[q]["counts"].sum()), np.int64)
        for s, d, c in zip(*lay[q]["recv"]):
            final[d:d + c] = recv[s:s + c]
        finals.append((final, lay[q]["counts"]))
    return finals


@pytest.mark.parametrize("world", [2, 3, 4])
def test_exchange_keeps_global_input_order(world):
    depth, parent, is_leaf, leaf_node, leaf_idx, n = toy_tree(1)
    counts = np.array([len(i) for i in leaf_idx])
    plan = plan_subtrees(depth, parent, is_leaf, leaf_node, counts, world)
    finals = simulate_exchange(leaf_idx, n, world, plan.leaf_owner)
    for q, (final, cnt) in enumerate(finals):
        off = 0
        for j in np.flatnonzero(plan.leaf_owner == q):
            assert np.array_equal(final[off:off + cnt[j]], leaf_idx[j])  # = reference leaf content, input order
            off += cnt[j]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.distributed.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = TorchComm(device="cpu")
        depth, parent, is_leaf, leaf_node, leaf_idx, n = toy_tree(2, n=20_000, T=800)
        bounds = [n * r // world for r in range(world + 1)]
        segs = [np.asarray(i)[(np.asarray(i) >= bounds[rank]) & (np.asarray(i) < bounds[rank + 1])] for i in leaf_idx]
        local = np.concatenate(segs)
        local_counts = np.array([len(s) for s in segs], np.int64)
        all_counts = comm.all_gather_np(local_counts)                      # the real collective
        plan = plan_subtrees(depth, parent, is_leaf, leaf_node, all_counts.sum(axis=0), world)
        lay = exchange_layout(plan.leaf_owner, all_counts, world)[rank]
        send = np.empty(len(local), np.int64)
        for s, d, c in zip(*lay["send"]):
            send[d:d + c] = local[s:s + c]
        recv = comm.all_to_all_bytes(torch.from_numpy(send.view(np.uint8).copy()), lay["send_splits"] * 8,
                                     lay["recv_splits"] * 8)               # gloo send/recv path
        recv = recv[:int(lay["recv_splits"].sum()) * 8].numpy().view(np.int64)
        final = np.empty(int(lay["counts"].sum()), np.int64)
        for s, d, c in zip(*lay["recv"]):
            final[d:d + c] = recv[s:s + c]
        t = torch.tensor([float(rank)], dtype=torch.float64)
        comm.allreduce(t, "max")
        ok = t.item() == world - 1
        off = 0
        for j in np.flatnonzero(plan.leaf_owner == rank):
            ok &= bool(np.array_equal(final[off:off + lay["counts"][j]], leaf_idx[j]))
            off += int(lay["counts"][j])
        blobs = comm.gather_bytes(torch.from_numpy(np.full(rank + 3, rank, np.uint8)), rank + 3)
        if rank == 0:
            ok &= all(len(b) == r + 3 and int(b[0]) == r for r, b in enumerate(blobs))
        q.put((rank, ok))
    finally:
        torch.distributed.destroy_process_group()


def test_gloo_world2_exchange():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    res = dict(q.get(timeout=5) for _ in range(2))
    assert res == {0: True, 1: True}
