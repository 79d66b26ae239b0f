"""Multi-process (gloo, world_size 2, CPU) tests of the partition / halo plan of the
multi-GPU path (paper_2212_00964_b200.distributed).  The device kernels need a GPU; what
is verified here is the host logic every rank runs: node ranges, ghost layers, matching
send/recv lists, and that a halo-exchanged local SpMV on each rank's sub-mesh reproduces
the owned rows of the global SpMV (numpy stands in for the device operator)."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as orc
from paper_2212_00964_b200.distributed import node_ranges, plan_parts
from paper_2212_00964_b200.mesh import generate_box_mesh


def _value(rows, cols):
    """A deterministic pseudo-matrix entry for global DOF pairs."""
    return np.sin(0.37 * rows + 0.11 * cols) + 0.05 * (rows == cols)


def _global_spmv(mesh, vec, x):
    ip, ix, _ = orc.pattern(mesh.cells, mesh.n_nodes, vec)
    rows = np.repeat(np.arange(ip.size - 1), np.diff(ip))
    return orc.csr_matvec(ip, ix, _value(rows, ix), x, use_numba=False)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, dims, vec, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch

        mesh = generate_box_mesh(*dims, 1.0, 1.0, 1.0)
        plane = (dims[0] + 1) * (dims[1] + 1)
        ranges = node_ranges(mesh.n_nodes, world, plane)
        plan = plan_parts(mesh, ranges, [rank])[0]
        x = np.random.default_rng(7).standard_normal(mesh.n_nodes * vec)
        # local matrix on the sub-mesh, values from global ids
        sub_cells = plan.to_local(mesh.cells[plan.local_cells])
        ip, ix, _ = orc.pattern(sub_cells, plan.local_nodes.size, vec)
        g_dof = (plan.local_nodes[:, None] * vec + np.arange(vec)).ravel()
        rows = np.repeat(np.arange(ip.size - 1), np.diff(ip))
        data = _value(g_dof[rows], g_dof[ix])
        # local x: owned entries only, ghosts poisoned, then filled by the halo exchange
        lo, hi = plan.own_local
        xl = np.full(plan.local_nodes.size * vec, np.nan)
        xl[lo * vec:hi * vec] = x[plan.own[0] * vec:plan.own[1] * vec]
        reqs = []
        for q_, s_nodes in zip(plan.peers, plan.send_nodes):
            buf = torch.from_numpy(xl.reshape(-1, vec)[s_nodes].ravel().copy())
            reqs.append(dist.isend(buf, q_))
        for q_, r_nodes in zip(plan.peers, plan.recv_nodes):
            buf = torch.empty(r_nodes.size * vec, dtype=torch.float64)
            dist.recv(buf, q_)
            xl.reshape(-1, vec)[r_nodes] = buf.numpy().reshape(-1, vec)
        for r in reqs:
            r.wait()
        y_local = orc.csr_matvec(ip, ix, data, xl, use_numba=False)
        y_own = y_local[lo * vec:hi * vec]
        y_ref = _global_spmv(mesh, vec, x)[plan.own[0] * vec:plan.own[1] * vec]
        ok_spmv = bool(np.all(np.isfinite(y_own)) and np.allclose(y_own, y_ref, rtol=1e-13, atol=1e-13))
        # plan consistency: my send list to q (global ids) == q's recv list from me
        mine = {int(q_): plan.local_nodes[s].tolist() for q_, s in zip(plan.peers, plan.send_nodes)}
        recv = {int(q_): plan.local_nodes[r].tolist() for q_, r in zip(plan.peers, plan.recv_nodes)}
        gathered = [None] * world
        dist.all_gather_object(gathered, (mine, recv))
        ok_plan = all(gathered[q_][1].get(rank, []) == lst for q_, lst in mine.items())
        # owned ranges tile the mesh; distributed dot == global dot
        t = torch.tensor([float(np.dot(x[plan.own[0] * vec:plan.own[1] * vec], x[plan.own[0] * vec:plan.own[1] * vec]))],
                         dtype=torch.float64)
        dist.all_reduce(t)
        ok_dot = abs(t.item() - float(x @ x)) < 1e-9 * float(x @ x)
        q.put((rank, ok_spmv, ok_plan, ok_dot, len(plan.peers)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dims,vec", [((4, 3, 6), 3), ((5, 4, 7), 1)])
def test_two_rank_halo_spmv_matches_global(dims, vec):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, dims, vec, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for rank, ok_spmv, ok_plan, ok_dot, npeers in res:
        assert ok_spmv, f"rank {rank}: halo SpMV differs from the global SpMV"
        assert ok_plan, f"rank {rank}: send/recv lists do not match"
        assert ok_dot and npeers == 1


def test_plan_ghost_layers_single_process():
    mesh = generate_box_mesh(3, 2, 5, 1.0, 1.0, 1.0)
    plane = 4 * 3
    ranges = node_ranges(mesh.n_nodes, 3, plane)
    assert ranges[0][0] == 0 and ranges[-1][1] == mesh.n_nodes
    assert all(lo % plane == 0 for lo, _ in ranges)
    plans = plan_parts(mesh, ranges)
    for p in plans:
        lo, hi = p.own
        assert np.array_equal(p.local_nodes[p.own_local[0]:p.own_local[1]], np.arange(lo, hi))
        # every neighbour of an owned node is local (rows complete)
        ip, ix, _ = orc.pattern(mesh.cells, mesh.n_nodes, 1)
        for n in range(lo, hi):
            assert np.isin(ix[ip[n]:ip[n + 1]], p.local_nodes).all()
    # interior part talks to both neighbours, end parts to one
    assert [len(p.peers) for p in plans] == [1, 2, 1]


def test_rcb_order_compact_parts_on_shuffled_mesh():
    """Coordinate bisection (distributed.rcb_order) of a mesh with shuffled node ids: balanced
    contiguous parts after renumbering, and halos that are interfaces (far fewer ghost nodes
    than contiguous ranges of the shuffled ids)."""
    from paper_2212_00964_b200.distributed import rcb_order
    from paper_2212_00964_b200.mesh import Mesh

    box = generate_box_mesh(12, 10, 8, 1.2, 1.0, 0.8)
    perm0 = np.random.default_rng(1).permutation(box.n_nodes)
    inv0 = np.argsort(perm0)
    mesh = Mesh(nodes=box.nodes[perm0], cells=inv0[box.cells])
    for nparts in (2, 3, 4, 8):
        perm, ranges = rcb_order(mesh.nodes, nparts)
        assert np.array_equal(np.sort(perm), np.arange(mesh.n_nodes))
        sizes = [hi - lo for lo, hi in ranges]
        assert max(sizes) - min(sizes) <= 1 + mesh.n_nodes // 50
        inv = np.empty_like(perm)
        inv[perm] = np.arange(perm.size)
        m2 = Mesh(nodes=mesh.nodes[perm], cells=inv[mesh.cells])
        ghosts_rcb = sum(p.local_nodes.size - (p.own[1] - p.own[0]) for p in plan_parts(m2, ranges))
        ghosts_raw = sum(p.local_nodes.size - (p.own[1] - p.own[0])
                         for p in plan_parts(mesh, node_ranges(mesh.n_nodes, nparts)))
        assert ghosts_rcb < 0.25 * ghosts_raw
