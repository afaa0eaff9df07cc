"""Row-slab multi-GPU outer loop: one process per GPU over NCCL,
or every slab in one process ("local transport", the same kernels and
exchange pattern with device copies; used for single-GPU parity tests).

The reference has no distributed code; this shards the one grid of
`run()` (solvers.py:416-475) by element rows.  Rank r owns element rows
[e0, e1) of a balanced split and keeps a window of H = filter radius + 1 halo
rows on each side (`slab_rows`).  The scalars of every iteration (compliance,
residual_inf, sum of g, box sum, dv_inf, volume) are all-gathered per rank and
summed in rank order, so every rank takes identical decisions and runs are
bitwise reproducible.  Supported low-level steps: fbto, pfbto_jacobi, pcg_jacobi
(the CG dot products are all-gathered the same way; the search direction is
halo-exchanged before every matvec), mg_pcg (the same CG with a block-Jacobi
multigrid preconditioner: each rank runs a V-cycle on the principal submatrix
of K over its owned node rows; with one rank it is the single-GPU MG-PCG) and
cpfbto_krylov (each power is halo-exchanged and its norm all-gathered; every
rank reduces its owned rows to one TSQR factor, the factors are all-gathered
and merged in rank order).

Bootstrap: rank 0 creates the NCCL unique id in the library
(`bsp_nccl_unique_id`) and torch.distributed broadcasts it; the library then
owns its communicator and records the NCCL calls into the iteration's CUDA
graph.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _dev
from ._native import ALGO, call, load
from .filtering import gaussian_weights
from .problems import ProblemSpec

SUPPORTED = ("fbto", "pfbto_jacobi", "cpfbto_krylov", "pcg_jacobi", "mg_pcg")


def halo_rows(filter_size: int) -> int:
    """Window halo H (element rows) for a filter of `filter_size` taps."""
    return filter_size // 2 + 1


def slab_rows(ny: int, world: int, rank: int, halo: int) -> tuple[int, int, int, int]:
    """(e0, e1, w0, w1): owned element rows [e0, e1) and window [w0, w1) of `rank`.

    Balanced split e0 = floor(ny r / G); the window adds `halo` rows on each
    side, clipped to the grid.  Pure host logic (mirrors bsp_dist_slab_rows)."""
    if world < 1 or not 0 <= rank < world or ny < 1:
        raise ValueError(f"bad slab request (ny={ny}, world={world}, rank={rank})")
    e0, e1 = ny * rank // world, ny * (rank + 1) // world
    return e0, e1, max(0, e0 - halo), min(ny, e1 + halo)


def owned_node_rows(ny: int, world: int, rank: int) -> tuple[int, int]:
    """Global node rows [n0, n1) owned by `rank` (the last rank owns row ny)."""
    e0, e1, _, _ = slab_rows(ny, world, rank, 0)
    return e0, (e1 + 1 if rank == world - 1 else e1)


def halo_plan(e0: int, e1: int, w0: int, depth: int, node: bool) -> dict:
    """Local row ranges of one halo exchange (mirrors `halo_rows` in distributed.cu).

    Element fields exchange `depth` owned rows with each neighbour; node fields
    exchange one node row: the first owned node row goes up (it is rank-1's
    ghost row e0), the last owned node row e1-1 goes down (rank+1's ghost row
    e1 - 1 = its e0 - 1).  Returns {"send_up", "recv_up", "send_dn", "recv_dn"}
    as (start, stop) local row ranges."""
    own0, own1 = e0 - w0, e1 - w0
    if node:
        return {"send_up": (own0, own0 + 1), "recv_up": (own0 - 1, own0),
                "send_dn": (own1 - 1, own1), "recv_dn": (own1, own1 + 1)}
    return {"send_up": (own0, own0 + depth), "recv_up": (own0 - depth, own0),
            "send_dn": (own1 - depth, own1), "recv_dn": (own1, own1 + depth)}


def window_arrays(grid, v0, active, nx: int, ny: int, w0: int, w1: int):
    """Slices of the global host arrays covering window rows [w0, w1).  A
    SparseGridModel (large grids) is sliced from its index lists, so no rank
    materialises the global mask or load."""
    lo, hi = 2 * w0 * (nx + 1), 2 * (w1 + 1) * (nx + 1)  # DOFs of node rows [w0, w1]
    if hasattr(grid, "_fixed_idx") and grid._dense is None:
        fixed = np.zeros(hi - lo, dtype=np.uint8)
        f = grid._fixed_idx[(grid._fixed_idx >= lo) & (grid._fixed_idx < hi)]
        fixed[f - lo] = 1
        load_ = np.zeros(hi - lo)
        sel = (grid._load_idx >= lo) & (grid._load_idx < hi)
        load_[grid._load_idx[sel] - lo] = grid._load_vals[sel]
    else:
        fixed = np.asarray(grid.fixed_dofs, dtype=np.uint8)[lo:hi]
        load_ = np.asarray(grid.load, dtype=np.float64)[lo:hi]
    fixed = fixed.reshape(w1 - w0 + 1, nx + 1, 2)
    load_ = load_.reshape(w1 - w0 + 1, nx + 1, 2)
    v = np.asarray(v0, dtype=np.float64).reshape(ny, nx)[w0:w1]
    act = None if active is None else np.asarray(active, np.uint8).reshape(ny, nx)[w0:w1]
    c = np.ascontiguousarray
    return c(fixed), c(load_), c(v), (None if act is None else c(act))


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    nb = C.c_int()
    call("bsp_nccl_unique_id", C.addressof(buf), C.byref(nb))
    return bytes(buf[:nb.value])


class SlabLoop:
    """Owner of a `bsp_dist` (include/bisimp_b200.h, row slabs)."""

    FIELDS = {"u": 0, "v": 1, "v_phys": 2, "activation": 3}

    def __init__(self, problem: ProblemSpec, config, world: int = 1, rank: int = 0,
                 nccl_id: bytes | None = None, local: bool = True, max_batch: int = 256):
        from . import solvers as S
        _dev.require_cuda()
        config = S.as_solver_config(config)
        if config.algorithm not in SUPPORTED:
            raise NotImplementedError(f"row slabs support {SUPPORTED}, not {config.algorithm!r}")
        if not local and nccl_id is None:
            raise ValueError("the NCCL transport needs the rank-0 unique id")
        # beta of fbto / pfbto (a power iteration) is estimated on the slabs
        # below, not on the full grid by every rank
        ws = S._prepare(problem, config, with_beta=False)
        self.ws, self.config = ws, config
        self.world, self.rank, self.local = int(world), int(rank), bool(local)
        self.max_batch = int(max_batch)
        grid = ws.grid
        nx, ny = grid.nx, grid.ny
        self.nx, self.ny = nx, ny
        cfg = S.config_c(ws, config, self.max_batch)
        taps = gaussian_weights(ws.filter_spec)
        self.halo = halo_rows(int(taps.size))
        n_active = float(grid.num_elements if ws.active is None else int(np.count_nonzero(ws.active)))
        ke = np.ascontiguousarray(grid.ke, dtype=np.float64)
        if local:
            fixed = np.ascontiguousarray(grid.fixed_dofs, dtype=np.uint8)
            load_ = np.ascontiguousarray(grid.load, dtype=np.float64)
            v0 = np.ascontiguousarray(ws.v_init, dtype=np.float64)
            act = None if ws.active is None else np.ascontiguousarray(ws.active, dtype=np.uint8)
            idp = None
        else:
            _, _, w0, w1 = slab_rows(ny, world, rank, self.halo)
            fixed, load_, v0, act = window_arrays(grid, ws.v_init, ws.active, nx, ny, w0, w1)
            self._id = (C.c_uint8 * len(nccl_id)).from_buffer_copy(nccl_id)
            idp = C.addressof(self._id)
        h = C.c_void_p()
        call("bsp_dist_create", nx, ny, self.world, self.rank, idp, ke.ctypes.data, fixed.ctypes.data,
             load_.ctypes.data, C.byref(cfg), None if act is None else act.ctypes.data, n_active,
             v0.ctypes.data, C.byref(h))
        self._h = h.value
        self._rec = np.zeros((self.max_batch, 4))
        self._alphas = np.zeros(self.max_batch)
        if ws.beta is None:
            self.beta = self._estimate_beta(grid.num_dofs, config.seed)
            ws.beta = self.beta
        else:
            self.beta = float(ws.beta)

    def _estimate_beta(self, n: int, seed: int, iters: int = 50) -> float:
        """1/rho of the set-up power iteration on the slabs (solvers.py:334-364):
        the seeded normals of the global grid are generated on this device
        (fea.standard_normal, numpy's stream bit for bit); each slab masks and
        normalises its window of them."""
        from .fea import standard_normal
        normals = standard_normal(seed, n)
        rho = C.c_double()
        call("bsp_dist_estimate_beta", self._h, normals.data_ptr(), int(iters), C.byref(rho))
        del normals
        return 1.0 / float(rho.value)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                load().bsp_dist_destroy(h)
            except Exception:
                pass
            self._h = None

    def run(self, k_first: int, alphas):
        n = len(alphas)
        self._alphas[:n] = alphas
        done, status = C.c_int(), C.c_int()
        call("bsp_dist_run", self._h, int(k_first), n, self._alphas.ctypes.data,
             self._rec.ctypes.data, C.byref(done), C.byref(status))
        return done.value, status.value, self._rec[:n].copy()

    def read(self, name: str) -> np.ndarray:
        """Owned rows of a field (local transport: the global array)."""
        nx, ny = self.nx, self.ny
        if self.local:
            size = 2 * (nx + 1) * (ny + 1) if name == "u" else nx * ny
        elif name == "u":
            n0, n1 = owned_node_rows(ny, self.world, self.rank)
            size = 2 * (nx + 1) * (n1 - n0)
        else:
            e0, e1, _, _ = slab_rows(ny, self.world, self.rank, 0)
            size = nx * (e1 - e0)
        out = np.empty(size)
        call("bsp_dist_read", self._h, self.FIELDS[name], out.ctypes.data)
        return out

    def _global(self, name: str) -> np.ndarray:
        """A field as the global array on every rank (local transport: as read;
        NCCL: the ranks' owned rows all-gathered in rank order)."""
        own = self.read(name)
        if self.local or self.world == 1:
            return own
        import torch
        import torch.distributed as dist
        sizes = [None] * self.world
        dist.all_gather_object(sizes, int(own.size))
        m = max(sizes)
        # NCCL gathers device tensors; a gloo group (the bench's isolated
        # children) gathers host tensors
        dev = (torch.device("cuda", torch.cuda.current_device())
               if dist.get_backend() == "nccl" else torch.device("cpu"))
        t = torch.zeros(m, dtype=torch.float64, device=dev)
        t[:own.size] = torch.from_numpy(own).to(dev)
        parts = [torch.empty(m, dtype=torch.float64, device=dev) for _ in range(self.world)]
        dist.all_gather(parts, t)
        return np.concatenate([p[:sz].cpu().numpy() for p, sz in zip(parts, sizes)])

    def read_state(self):
        """(u, v, v_phys, activation) of the last completed iteration, global
        arrays on every rank (the sink's SolverState, solvers.py:367-378)."""
        return tuple(self._global(f) for f in ("u", "v", "v_phys", "activation"))

    def read_frame(self, kind: str = "f32") -> bytes:
        """The density frame of the last completed iteration (as
        DeviceLoop.read_frame), from the gathered v_phys."""
        from .outputs import density_pixels, frame_payload
        vp = self._global("v_phys")
        if kind == "f32":
            return frame_payload(vp)
        px = density_pixels(vp)
        return (px.cpu().numpy() if _dev.is_tensor(px) else np.asarray(px)).tobytes()

    def info(self) -> dict:
        out = np.zeros(5)
        call("bsp_dist_info", self._h, out.ctypes.data)
        return {"graphs": bool(out[0]), "host_lambda_iters": int(out[1]),
                "lambda_rounds": int(out[2]), "halo_rows": int(out[3]), "slabs_here": int(out[4])}

    def comm_ms(self, iters: int = 50) -> tuple[float, float]:
        """(halo exchange, all-gather) device ms per call."""
        out = np.zeros(2)
        call("bsp_dist_comm_bench", self._h, int(iters), out.ctypes.data)
        return float(out[0]), float(out[1])

    def stream(self) -> int:
        return load().bsp_dist_stream(self._h)


def broadcast_nccl_id(rank: int) -> bytes:
    """Rank 0's NCCL unique id, broadcast over the default torch.distributed group."""
    import torch.distributed as dist
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def slab_loop(problem: ProblemSpec, config, slabs) -> SlabLoop:
    """The SlabLoop behind run(..., slabs=...): "nccl" -> one slab per rank of
    the initialised torch.distributed group (rank 0's NCCL id broadcast);
    int G -> G slabs on this GPU (local transport)."""
    if slabs == "nccl":
        import torch.distributed as dist
        if not dist.is_available() or not dist.is_initialized():
            raise ValueError('slabs="nccl" needs an initialised torch.distributed group')
        world, rank = dist.get_world_size(), dist.get_rank()
        return SlabLoop(problem, config, world=world, rank=rank,
                        nccl_id=broadcast_nccl_id(rank), local=False)
    if isinstance(slabs, (int, np.integer)) and not isinstance(slabs, bool) and slabs >= 1:
        return SlabLoop(problem, config, world=int(slabs), local=True)
    raise ValueError(f'slabs must be None, "nccl" or a slab count >= 1, got {slabs!r}')
