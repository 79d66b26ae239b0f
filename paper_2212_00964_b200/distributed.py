"""Partitioned forward solve across GPUs (north_star multi-GPU).

Partitioning: contiguous node-id ranges.  For box meshes the node order is z-major, so a
range is a stack of node planes (a z-slab).  Part r owns the DOF rows of its nodes and keeps
every cell that touches an owned node (one ghost cell layer on each side).  Its owned rows
therefore assemble locally, with no communication and in the single-GPU cell order.  Only
two things are exchanged:

* a halo of the SpMV operand and of U: owned interface-node values are sent to the ghost
  entries of the neighbouring parts (csrc/krylov_dist.cu, ncclSend/ncclRecv);
* FP64 sum-allreduces of the Krylov dot groups and of the Newton residual norm.

Two communicators share this code:

* "nccl": one part per process (torchrun, one GPU per rank);
* "local": several parts in one process on one device.  This is the same algorithm with
  device copies and an in-order sum.  It is how the partitioning is verified on a single
  B200; there is no waiting kernel on one GPU.

The host-side plan (``plan_parts``) is plain numpy and is unit-tested with gloo on the CPU
(tests/test_dist_gloo.py).
"""

from __future__ import annotations

import copy
import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _device as D
from . import _lib
from .assembly import NeumannSpec, workspace
from .errors import NonConvergenceError, raise_for
from .materials import QuadPointState
from .mesh import FacetSet, Mesh
from .solvers import LinearSolveConfig, NewtonConfig, NewtonReport, SolveStats
from .sparse import CsrMatrix, GridOperator


# ------------------------------------------------------------------------------ plan
def node_ranges(n_nodes: int, nparts: int, plane: int | None = None):
    """Balanced contiguous node ranges; if `plane` (nodes per z-plane) is given, cut on planes."""
    if plane:
        n_planes = n_nodes // plane
        cuts = [round(k * n_planes / nparts) * plane for k in range(nparts + 1)]
    else:
        cuts = [round(k * n_nodes / nparts) for k in range(nparts + 1)]
    cuts[-1] = n_nodes
    return [(cuts[k], cuts[k + 1]) for k in range(nparts)]


def rcb_order(coords: np.ndarray, nparts: int):
    """Recursive coordinate bisection of the nodes into `nparts` spatially compact parts.

    Returns (perm, ranges): perm[new] = old node id with part 0's nodes first (original
    relative order kept inside a part), and the contiguous new-id range of every part.  Used
    for meshes whose numbering is not a z-major lattice (e.g. Gmsh files),
    where contiguous ranges of the original ids would be scattered node sets with halos
    spanning the whole mesh."""
    parts = []

    def split(ids, k):
        if k == 1:
            parts.append(np.sort(ids))
            return
        x = coords[ids]
        axis = int(np.argmax(x.max(axis=0) - x.min(axis=0)))
        k1 = k // 2
        order = ids[np.argsort(x[:, axis], kind="stable")]
        cut = int(round(ids.size * k1 / k))
        split(order[:cut], k1)
        split(order[cut:], k - k1)

    split(np.arange(coords.shape[0]), nparts)
    sizes = np.array([p.size for p in parts])
    cuts = np.concatenate([[0], np.cumsum(sizes)])
    return np.concatenate(parts), [(int(cuts[i]), int(cuts[i + 1])) for i in range(nparts)]


def renumbered(problem, perm):
    """The same problem with node n' = perm^-1 (the mesh nodes reordered, cells unchanged):
    geometric Dirichlet/Neumann/body data are re-located by the workspace; nodal designs are
    permuted."""
    mesh = problem.mesh
    inv = np.empty_like(perm)
    inv[perm] = np.arange(perm.size)
    p2 = copy.copy(problem)
    p2.mesh = Mesh(nodes=mesh.nodes[perm], cells=inv[mesh.cells])
    p2._ws = None
    if hasattr(p2, "_jac_cache"):
        delattr(p2, "_jac_cache")
    if getattr(problem, "design_layout", None) == "node":
        p2.theta = np.asarray(problem.theta)[perm]
        p2._theta_version = 0
    return p2


@dataclass
class PartPlan:
    rank: int
    own: tuple                      # (lo, hi) global node ids
    local_nodes: np.ndarray         # sorted global node ids (owned + ghosts)
    local_cells: np.ndarray         # sorted global cell ids touching owned nodes
    own_local: tuple                # owned range in local numbering
    peers: list = field(default_factory=list)
    send_nodes: list = field(default_factory=list)  # local ids, per peer
    recv_nodes: list = field(default_factory=list)  # local ids, per peer

    def to_local(self, global_ids):
        return np.searchsorted(self.local_nodes, global_ids)


def _touching(cells, lo, hi):
    return np.flatnonzero(((cells >= lo) & (cells < hi)).any(axis=1))


def plan_parts(mesh: Mesh, ranges, ranks=None):
    """Host plan for the given parts: ghost layers and matching send/recv node lists."""
    cells = mesh.cells
    touching = [_touching(cells, lo, hi) for lo, hi in ranges]
    ghost_sets = []
    for r, (lo, hi) in enumerate(ranges):
        nodes = np.unique(cells[touching[r]])
        ghost_sets.append(nodes[(nodes < lo) | (nodes >= hi)])
    starts = np.array([lo for lo, _ in ranges])
    plans = []
    for r in (range(len(ranges)) if ranks is None else ranks):
        lo, hi = ranges[r]
        local_nodes = np.unique(cells[touching[r]])
        p = PartPlan(rank=r, own=(lo, hi), local_nodes=local_nodes, local_cells=touching[r],
                     own_local=(int(np.searchsorted(local_nodes, lo)), int(np.searchsorted(local_nodes, hi))))
        owner = np.searchsorted(starts, ghost_sets[r], side="right") - 1
        for q in range(len(ranges)):
            if q == r:
                continue
            recv = ghost_sets[r][owner == q]                       # my ghosts owned by q
            send = ghost_sets[q][(ghost_sets[q] >= lo) & (ghost_sets[q] < hi)]  # q's ghosts I own
            if recv.size or send.size:
                p.peers.append(q)
                p.recv_nodes.append(p.to_local(recv).astype(np.int32))
                p.send_nodes.append(p.to_local(send).astype(np.int32))
        plans.append(p)
    return plans


def subproblem(problem, plan: PartPlan):
    """The same problem restricted to one part's cells (owned + ghost layer)."""
    mesh = problem.mesh
    sub_mesh = Mesh(nodes=mesh.nodes[plan.local_nodes], cells=plan.to_local(mesh.cells[plan.local_cells]))
    sub = copy.copy(problem)
    sub.mesh = sub_mesh
    sub._ws = None
    for attr in ("_jac_cache",):
        if hasattr(sub, attr):
            delattr(sub, attr)
    cell_map = -np.ones(mesh.n_cells, dtype=np.int64)
    cell_map[plan.local_cells] = np.arange(plan.local_cells.size)
    neu = []
    for spec in problem.neumann:
        f = spec.facet_set.facets
        keep = cell_map[f[:, 0]] >= 0 if f.size else np.zeros(0, dtype=bool)
        nf = f[keep].copy()
        if nf.size:
            nf[:, 0] = cell_map[nf[:, 0]]
        neu.append(NeumannSpec(FacetSet(nf), spec.traction_fn))
    sub.neumann = neu
    if problem.design_layout == "element":
        sub.theta = np.asarray(problem.theta)[plan.local_cells]
        sub._theta_version = 0
    elif problem.design_layout == "node":
        sub.theta = np.asarray(problem.theta)[plan.local_nodes]
        sub._theta_version = 0
    if hasattr(problem, "_host_state"):
        st = problem._current_state()
        sub._host_state = QuadPointState(st.eps_prev[plan.local_cells], st.sig_prev[plan.local_cells])
    return sub


# ------------------------------------------------------------------- communicator
class Communicator:
    """NCCL communicator created through libb200fem (one part per rank), or a local one."""

    def __init__(self, kind="local", rank=0, nranks=1):
        lib = _lib.lib()
        self.kind, self.rank, self.nranks = kind, rank, nranks
        h = C.c_void_p()
        if kind == "nccl":
            import torch.distributed as dist

            uid = (C.c_uint8 * 128)()
            if rank == 0:
                raise_for(lib.b200fem_comm_unique_id(uid), None, "nccl unique id")
            obj = [bytes(uid)]
            dist.broadcast_object_list(obj, src=0)
            uid = (C.c_uint8 * 128).from_buffer_copy(obj[0])
            raise_for(lib.b200fem_comm_create_nccl(C.byref(h), uid, nranks, rank), None, "ncclCommInitRank")
        else:
            raise_for(lib.b200fem_comm_create_local(C.byref(h)), None, "local comm")
        self.handle = h

    def allreduce_(self, t):
        """In-place sum of a CUDA float64 tensor over ranks (no-op for the local comm)."""
        raise_for(_lib.lib().b200fem_comm_allreduce(self.handle, D.ptr(t), t.numel(), D.stream()), None, "allreduce")

    def __del__(self):
        h = getattr(self, "handle", None)
        try:  # at interpreter exit the module globals may already be gone
            if h is not None and _lib._lib is not None:
                _lib._lib.b200fem_comm_destroy(h)
        except Exception:
            pass


# ---------------------------------------------------------------------- solver
class _Part:
    def __init__(self, problem, plan: PartPlan, operator="auto"):
        self.plan = plan
        self.problem = subproblem(problem, plan)
        self.ws = workspace(self.problem)
        n = self.problem.n_dofs
        self.vec = self.problem.vec
        # a plane-cut part of a box lattice is itself a lattice: same GRID3 operator as 1 GPU
        self.grid = operator in ("auto", "grid") and self.ws.has_grid
        self.K = GridOperator(self.ws) if self.grid else CsrMatrix._from_workspace(self.ws, D.empty(self.ws.nnz))
        h = self.K._device_handle()
        lib = _lib.lib()
        peers = np.array(plan.peers, dtype=np.int32)
        sc = np.array([s.size for s in plan.send_nodes], dtype=np.int64)
        rc = np.array([s.size for s in plan.recv_nodes], dtype=np.int32).astype(np.int64)
        sn = np.concatenate(plan.send_nodes).astype(np.int32) if plan.send_nodes else np.zeros(0, np.int32)
        rn = np.concatenate(plan.recv_nodes).astype(np.int32) if plan.recv_nodes else np.zeros(0, np.int32)
        ph = C.c_void_p()
        lo, hi = plan.own_local
        raise_for(lib.b200fem_part_create(C.byref(ph), h, lo, hi, len(plan.peers), D.hptr(peers), D.hptr(sc),
                                          D.hptr(sn), D.hptr(rc), D.hptr(rn)), None, "part_create")
        self.handle = ph
        self.U = D.zeros(n)
        self.R = D.empty(n)
        self.rhs = D.empty(n)
        self.dU = D.empty(n)
        self.own_dofs = (lo * self.vec, hi * self.vec)

    def assemble_tangent(self):
        if self.grid:
            self.ws.jacobian_grid(self.problem, self.U, self.K.device_data)
        else:
            self.ws.jacobian(self.problem, self.U, self.K.device_data)

    def __del__(self):
        h = getattr(self, "handle", None)
        try:  # at interpreter exit the module globals may already be gone
            if h is not None and _lib._lib is not None:
                _lib._lib.b200fem_part_destroy(h)
        except Exception:
            pass


class PartitionedSolver:
    """Newton / BiCGSTAB on a node-partitioned mesh (same semantics as solvers.newton_solve).

    nccl mode: call from every rank of an initialised torch.distributed NCCL group; this
    process solves part `rank` of `world_size`.  local mode: `nparts` parts in this process."""

    def __init__(self, problem, nparts=None, mode="auto", ranges=None, plane_cut=True, operator="auto",
                 reorder="auto"):
        import torch.distributed as dist

        if mode == "auto":
            mode = "nccl" if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1 else "local"
        mesh = problem.mesh
        if mode == "nccl":
            rank, world = dist.get_rank(), dist.get_world_size()
            nparts = world
        else:
            rank, world = 0, 1
            nparts = nparts or 2
        plane = self._plane_size(mesh) if plane_cut else None
        # a mesh that is not a z-major lattice is renumbered by coordinate bisection so that
        # every part is a compact node set (its halo is an interface, not the whole mesh)
        self.perm = None
        if ranges is None and (reorder is True or (reorder == "auto" and plane is None and nparts > 1)):
            self.perm, ranges = rcb_order(mesh.nodes, nparts)
            self.orig_problem = problem
            problem = renumbered(problem, self.perm)
            mesh = problem.mesh
        self.ranges = ranges or node_ranges(mesh.n_nodes, nparts, plane)
        self.mode = mode
        self.problem = problem
        self.comm = Communicator("nccl" if mode == "nccl" else "local", rank, world)
        ranks = [rank] if mode == "nccl" else list(range(nparts))
        self.plans = plan_parts(mesh, self.ranges, ranks)
        self.operator = operator
        self.parts = [_Part(problem, p, operator) for p in self.plans]
        self._ptrs = (C.c_void_p * len(self.parts))(*[p.handle.value for p in self.parts])

    @staticmethod
    def _plane_size(mesh):
        z = mesh.nodes[:, 2]
        if mesh.n_nodes > 1 and np.all(np.diff(z) >= 0):  # z-major numbering (box meshes)
            first = np.flatnonzero(z > z[0])
            if first.size and mesh.n_nodes % first[0] == 0:
                return int(first[0])
        return None

    # -- collectives over the parts
    def _vec_ptrs(self, attr):
        return (C.c_void_p * len(self.parts))(*[getattr(p, attr).data_ptr() for p in self.parts])

    def halo(self, attr):
        raise_for(_lib.lib().b200fem_dist_halo(self._ptrs, len(self.parts), self.comm.handle, self._vec_ptrs(attr)),
                  None, "halo")

    def dot(self, a, b) -> float:
        out = C.c_double()
        raise_for(_lib.lib().b200fem_dist_dot(self._ptrs, len(self.parts), self.comm.handle, self._vec_ptrs(a),
                                              self._vec_ptrs(b), C.byref(out)), None, "dist_dot")
        return out.value

    def residual_norm(self, apply_dirichlet=True) -> float:
        scale = (self.orig_problem if self.perm is not None else self.problem).bc_scale
        for p in self.parts:
            p.problem.bc_scale = scale
            p.ws.residual(p.problem, p.U, p.R, apply_dirichlet)
        return float(np.sqrt(self.dot("R", "R")))

    def _check_operator(self, cfg: LinearSolveConfig):
        """The parts' operators are built once (constructor ``operator``); a config asking for a
        storage the parts do not have is an error, not a silent substitution."""
        built = "grid" if all(p.grid for p in self.parts) else "csr"
        want = cfg.operator
        if want in ("auto", built):
            return
        raise ValueError(f'LinearSolveConfig(operator="{want}") is not available on this PartitionedSolver: '
                         f'its parts were built with the "{built}" operator (PartitionedSolver(..., operator=...))')

    def linear_solve(self, cfg: LinearSolveConfig) -> SolveStats:
        """rhs -> dU over all parts with cfg.method: "bicgstab" (reference) or "pcg"."""
        self._check_operator(cfg)
        if cfg.method not in ("bicgstab", "pcg"):
            raise ValueError(f"unknown linear method {cfg.method!r}")
        fn = _lib.lib().b200fem_dist_pcg if cfg.method == "pcg" else _lib.lib().b200fem_dist_bicgstab
        info = _lib.SolveInfo()
        err = _lib.Error()
        st = fn(self._ptrs, len(self.parts), self.comm.handle, self._vec_ptrs("rhs"), self._vec_ptrs("dU"), 0,
                float(cfg.rel_tol), float(cfg.abs_tol), int(cfg.max_iters), C.byref(info), C.byref(err))
        raise_for(st, err, f"dist_{cfg.method}")
        return SolveStats(info.iterations, info.matvecs, info.restarts, info.residual, info.tol)

    def bicgstab(self, cfg: LinearSolveConfig) -> SolveStats:
        """BiCGSTAB regardless of cfg.method (kept for callers of the round-1 API)."""
        from dataclasses import replace

        return self.linear_solve(replace(cfg, method="bicgstab"))

    def _dof_perm(self):
        vec = self.problem.vec
        return (self.perm[:, None] * vec + np.arange(vec)).ravel()  # new dof -> old dof

    def set_U(self, U):
        """Scatter a global U (host or device, length N, original numbering) into the parts."""
        Ug = D.to_device(U)
        if self.perm is not None:
            Ug = Ug[D.to_device(self._dof_perm(), D.torch().int64)]
        vec = self.problem.vec
        for p in self.parts:
            idx = (p.plan.local_nodes[:, None] * vec + np.arange(vec)).ravel()
            p.U.copy_(Ug[D.to_device(idx, D.torch().int64)])

    def gather_U(self) -> np.ndarray:
        """Global U on the host (owned blocks of all parts; all-gathered in nccl mode)."""
        vec = self.problem.vec
        U = np.zeros(self.problem.n_dofs)
        for p in self.parts:
            lo, hi = p.own_dofs
            glo = p.plan.own[0] * vec
            U[glo:glo + hi - lo] = D.to_host(p.U[lo:hi])
        if self.mode == "nccl":
            t = D.to_device(U)
            self.comm.allreduce_(t)  # disjoint owned blocks -> the sum is the concatenation
            U = D.to_host(t)
        if self.perm is not None:  # back to the original numbering
            Uo = np.empty_like(U)
            Uo[self._dof_perm()] = U
            U = Uo
        return U

    def newton_solve(self, U0=None, cfg: NewtonConfig = NewtonConfig(),
                     lin_cfg: LinearSolveConfig = LinearSolveConfig()):
        """Newton on the partitioned problem; returns (NewtonReport); U stays distributed."""
        lib = _lib.lib()
        stream = D.stream()
        if U0 is None:
            for p in self.parts:
                p.U.zero_()
        else:
            self.set_U(U0)
        norms = [self.residual_norm()]
        r0 = norms[0]
        lin = []
        for it in range(cfg.max_iters):
            if norms[-1] <= max(cfg.rel_tol * r0, cfg.abs_tol):
                return NewtonReport(norms, it, True, lin)
            for p in self.parts:
                if not (p.problem.jacobian_constant and getattr(p, "_k_done", False)):
                    p.assemble_tangent()
                    p._k_done = True
                lib.b200fem_scale(p.problem.n_dofs, -1.0, D.ptr(p.R), D.ptr(p.rhs), stream)
            lin.append(self.linear_solve(lin_cfg))
            for p in self.parts:
                lo, hi = p.own_dofs
                lib.b200fem_axpy(hi - lo, 1.0, D.ptr(p.dU[lo:]), D.ptr(p.U[lo:]), stream)
            self.halo("U")
            norms.append(self.residual_norm())
        if norms[-1] <= max(cfg.rel_tol * r0, cfg.abs_tol):
            return NewtonReport(norms, cfg.max_iters, True, lin)
        raise NonConvergenceError(f"Newton did not converge in {cfg.max_iters} iterations", residual_norms=norms)


def newton_solve_partitioned(problem, nparts=None, U0=None, cfg: NewtonConfig = NewtonConfig(),
                             lin_cfg: LinearSolveConfig = LinearSolveConfig(), mode="auto"):
    """Convenience: build a PartitionedSolver, solve, gather U -> (U, NewtonReport)."""
    s = PartitionedSolver(problem, nparts=nparts, mode=mode)
    rep = s.newton_solve(U0, cfg, lin_cfg)
    return s.gather_U(), rep
