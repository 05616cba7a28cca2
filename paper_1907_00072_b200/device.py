"""Device runtime: row-block shards, halo plans, communicators and the vector
engine the solver drives.

A *shard* is one contiguous block of rows ``[r0, r1)`` living on one GPU: its
slice of A as a SELL-C-sigma ``pg_matrix`` (columns renumbered: owned columns
first, then the ghost columns it reads from other shards, grouped by owner),
a reduction workspace and its device.  A distributed vector is a Python list
holding one float64 tensor per local shard, of length ``n_ext`` (owned rows +
ghost slots).  The solver is written once over that list:

* ``SoloComm``   -- every shard of the job lives in this process (1 shard on 1
  GPU for the default path; or P *virtual* shards on one GPU, which exercises
  the partition / halo / reduction logic with the real kernels on one device);
* ``DistComm``   -- one shard per process, ``torch.distributed`` (NCCL on GPUs):
  halo = batched point-to-point send/recv of boundary entries before each SpMV,
  and one all-reduce per batched-dot phase.

No reference CPU arithmetic lives here; every flop on the path is a libpgmres
kernel.  PyTorch provides device memory, streams and the collectives.
"""

from __future__ import annotations

import os
import threading
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .errors import DeviceError, DimensionMismatchError, ParameterError

F64 = torch.float64
KMAX = _lib.PG_KMAX  # columns per tall-skinny kernel call
MMAX = _lib.PG_MMAX  # widest basis (restart length + 1) of a solve
ROW_ALIGN = 64  # leading-dimension alignment of basis blocks (rows)


def _pad(n: int) -> int:
    return max(ROW_ALIGN, (n + ROW_ALIGN - 1) // ROW_ALIGN * ROW_ALIGN)


def ptr(t: torch.Tensor) -> int:
    return t.data_ptr()


def require_cuda():
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: the PP-GMRES device path has no CPU fallback")


# ---------------------------------------------------------------------------
# partition and halo plan
# ---------------------------------------------------------------------------
def balanced_offsets(row_ptr: np.ndarray, parts: int, align: int = 1) -> np.ndarray:
    """Row offsets of ``parts`` contiguous blocks with ~equal nnz, boundaries
    rounded to multiples of ``align`` rows (e.g. a grid plane)."""
    n = len(row_ptr) - 1
    if parts < 1:
        raise ParameterError("parts must be >= 1")
    nnz = int(row_ptr[-1])
    offs = [0]
    for p in range(1, parts):
        target = nnz * p / parts
        r = int(np.searchsorted(row_ptr, target, side="left"))
        r = int(round(r / align) * align) if align > 1 else r
        offs.append(min(max(r, offs[-1]), n))
    offs.append(n)
    return np.array(offs, dtype=np.int64)


@dataclass
class HaloPlan:
    """Ghost layout of one shard.  ``recv[q] = (offset, count)``: the ghost slots
    ``[offset, offset+count)`` of the local vector are filled from shard q (ghost
    columns sorted by global index, so each owner's ghosts are contiguous).
    ``send[q]``: local row indices this shard sends to shard q."""

    ghosts: np.ndarray
    recv: dict = field(default_factory=dict)
    send: dict = field(default_factory=dict)


def ghost_columns(cols: np.ndarray, r0: int, r1: int) -> np.ndarray:
    outside = cols[(cols < r0) | (cols >= r1)]
    return np.unique(outside)


def plan_recv(ghosts: np.ndarray, offsets: np.ndarray, n_local: int) -> dict:
    owners = np.searchsorted(offsets, ghosts, side="right") - 1
    recv = {}
    for q in np.unique(owners):
        idx = np.nonzero(owners == q)[0]
        recv[int(q)] = (n_local + int(idx[0]), int(len(idx)))
    return recv


def localize_columns(cols: np.ndarray, r0: int, r1: int, ghosts: np.ndarray) -> np.ndarray:
    """Global -> local column numbering; entry order (hence the per-row sum
    order of the SpMV) is untouched."""
    inside = (cols >= r0) & (cols < r1)
    return np.where(inside, cols - r0, (r1 - r0) + np.searchsorted(ghosts, cols)).astype(np.int64)


def choose_sigma(row_ptr: np.ndarray) -> int:
    """SELL sorting window: 1 (no reordering) unless slice padding with natural
    row order exceeds 15% of nnz (irregular rows, e.g. config 3)."""
    lens = np.diff(row_ptr)
    n = len(lens)
    if n == 0:
        return 1
    pad = (-n) % 32
    L = np.concatenate([lens, np.zeros(pad, lens.dtype)]).reshape(-1, 32)
    padded = int(L.max(axis=1).sum()) * 32
    return 1 if padded <= 1.15 * max(1, int(row_ptr[-1])) else 4096


# ---------------------------------------------------------------------------
# one shard
# ---------------------------------------------------------------------------
class Shard:
    def __init__(self, index: int, device: torch.device, r0: int, r1: int,
                 row_ptr: np.ndarray, cols_global: np.ndarray, values: np.ndarray,
                 offsets: np.ndarray, sigma: int | None = None):
        lib = _lib.load()
        self.index = index
        self.device = device
        self.dev_ord = device.index if device.index is not None else torch.cuda.current_device()
        self.r0, self.r1 = int(r0), int(r1)
        self.n = self.r1 - self.r0
        ghosts = ghost_columns(cols_global, self.r0, self.r1)
        self.plan = HaloPlan(ghosts, plan_recv(ghosts, offsets, self.n))
        self.n_ext = self.n + len(ghosts)
        self.ld = _pad(self.n_ext)
        self.offsets = np.asarray(offsets, dtype=np.int64)
        cols_local = localize_columns(cols_global, self.r0, self.r1, ghosts)
        self.sigma = choose_sigma(row_ptr) if sigma is None else int(sigma)
        rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        cl = np.ascontiguousarray(cols_local, dtype=np.int64)
        vl = np.ascontiguousarray(values, dtype=np.float64)
        h = _lib.C.c_void_p()
        _lib.call("pg_matrix_create", self.dev_ord, self.n, self.n_ext, rp.ctypes.data,
                  cl.ctypes.data, vl.ctypes.data, self.sigma, _lib.C.byref(h))
        self.mat = h
        w = _lib.C.c_void_p()
        _lib.call("pg_workspace_create", self.dev_ord, _lib.C.byref(w))
        self.ws = w
        self.nnz = int(row_ptr[-1])
        st = (_lib.C.c_int64 * 12)()
        _lib.call("pg_matrix_stats", self.mat, st)
        self.stats = dict(zip(("nrows", "ncols", "nnz", "padded_nnz", "n_slices",
                               "device_bytes", "max_width", "sigma", "col_bytes",
                               "val_bytes", "stream_bytes", "kernel"), list(st)))
        # bytes streamed per stored matrix entry (dictionary compression: 1+1)
        self.entry_bytes = int(st[10])
        pl = (_lib.C.c_int64 * 10)()
        _lib.call("pg_plane_plan", self.mat, pl)
        self.plane_plan = dict(zip(("kind", "Q", "Zc", "stages", "blocks", "H", "box",
                                    "stage_bytes", "sym", "vec"), list(pl)))
        # Arnoldi-step passes run as one dependency-driven kernel (chain.cu)
        fused = _lib.C.c_int(0)
        _lib.call("pg_chain_fused", h, _lib.C.byref(fused))
        self.chain_fused = bool(fused.value)
        # small per-shard device scratch: [c1 | c2 | nsq | spare]
        self.scal = torch.zeros(2 * KMAX + 8, dtype=F64, device=device)
        self.coef = torch.zeros(MMAX, dtype=F64, device=device)
        # two-slot ring of CGS2 scalars (one Arnoldi step of look-ahead), each
        # packed [c1 (k) | c2 (k) | nsq], and its pinned host mirror
        self.ring = [torch.zeros(2 * MMAX + 8, dtype=F64, device=device) for _ in range(2)]
        self.pinned = [torch.zeros(2 * MMAX + 1, dtype=F64).pin_memory() for _ in range(2)]
        self.send_idx: dict = {}
        self.send_buf: dict = {}
        self._lib = lib
        self._stream = None

    # send lists (local indices) are installed once every shard's ghost needs are known
    def set_send(self, q: int, local_idx: np.ndarray):
        local_idx = np.ascontiguousarray(local_idx, dtype=np.int32)
        self.plan.send[q] = local_idx
        contiguous = len(local_idx) > 0 and np.all(np.diff(local_idx) == 1)
        if contiguous:
            self.send_idx[q] = (int(local_idx[0]), int(len(local_idx)))
        else:
            self.send_idx[q] = torch.from_numpy(local_idx).to(self.device)
            self.send_buf[q] = torch.empty(len(local_idx), dtype=F64, device=self.device)

    @property
    def stream(self) -> int:
        """cudaStream_t of the device's current torch stream, cached by
        :meth:`Engine.bind_stream` at each public entry point."""
        st = self._stream
        if st is None:
            st = self._stream = torch.cuda.current_stream(self.device).cuda_stream
        return st

    def activate(self):
        _lib.call("pg_set_device", self.dev_ord)

    def vec(self) -> torch.Tensor:
        """Shard vector: owned rows, ghost slots, zero padding up to ``ld`` (the
        tile / ring kernels stream whole 16-byte pairs of rows)."""
        return torch.zeros(self.ld, dtype=F64, device=self.device)

    def block(self, cols: int) -> torch.Tensor:
        """Column-major n x cols block: row-major (cols, ld) tensor."""
        return torch.zeros((cols, self.ld), dtype=F64, device=self.device)

    def packed_send(self, x: torch.Tensor, q: int) -> torch.Tensor:
        sel = self.send_idx[q]
        if isinstance(sel, tuple):
            a, c = sel
            return x[a:a + c]
        buf = self.send_buf[q]
        _lib.call("pg_gather", ptr(x), ptr(sel), len(sel), ptr(buf), self.stream)
        return buf

    def pass_bytes(self, vec_bytes: int) -> int:
        """Algorithmic bytes of one SpMV pass over the stored format: the
        matrix stream (1 B per row for the row-pattern format -- none for the
        plane-ring kernel, whose interior planes read no pattern ids -- 8 B per entry
        + 1 B per row for the offset-pattern format; else the
        stored entry bytes + a 4-byte row length), the compulsory gather of x
        (8 B per row) and ``vec_bytes`` per row of epilogue vectors."""
        if self.stats["kernel"] == 9:  # plane ring: interior planes read no pattern ids
            return (8 + vec_bytes) * self.n
        if self.stats["kernel"] in (5, 6, 8):  # row patterns (gather, windowed, marching)
            return (1 + 8 + vec_bytes) * self.n
        if self.stats["kernel"] == 7:  # offset patterns: f64 values + 1 B per row
            return 8 * self.nnz + (1 + 8 + vec_bytes) * self.n
        return self.entry_bytes * self.nnz + (12 + vec_bytes) * self.n

    def close(self):
        if getattr(self, "mat", None):
            _lib.load().pg_matrix_destroy(self.mat)
            self.mat = None
        if getattr(self, "ws", None):
            _lib.load().pg_workspace_destroy(self.ws)
            self.ws = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------------------
# communicators
# ---------------------------------------------------------------------------
class SoloComm:
    """All shards of the job are in this process (1 GPU, or P virtual shards).
    Halo = device copies; all-reduce = fixed-order sum over shards."""

    distributed = False
    world = 1

    def __init__(self, shards):
        self.shards = shards

    def halo(self, xs):
        if len(self.shards) == 1:
            return
        for p, s in enumerate(self.shards):
            for q, (off, cnt) in s.plan.recv.items():
                src = self.shards[q].packed_send(xs[q], p)
                xs[p][off:off + cnt].copy_(src, non_blocking=True)

    def allreduce(self, bufs):
        if len(bufs) == 1:
            return
        total = bufs[0].clone()
        for b in bufs[1:]:
            total += b.to(total.device)
        for b in bufs:
            b.copy_(total)


class DistComm:
    """One shard per process; torch.distributed (NCCL for CUDA tensors, gloo
    for the CPU host-logic tests).  Halo: one batched send/recv round of
    boundary entries per SpMV.  Reductions: every rank's partials are
    all-gathered and summed in rank order -- the SoloComm order, identical on
    every rank, independent of NCCL's algorithm choice.

    With the NCCL backend the same exchanges also exist natively (``native``,
    a ``pg_dist`` communicator of csrc/dist.cu): the solver's Arnoldi steps,
    polynomial chains and power sequences then issue their halos and CGS2
    reductions from C between the kernels, one native call (or recorded
    graph) per step.  PG_DIST_NATIVE=0 keeps the torch-issued exchanges."""

    distributed = True

    def __init__(self, shards, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.shards = shards
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        # gloo moves CPU tensors only: device buffers are staged through the
        # host (host-logic tests, and several ranks sharing one GPU in the GPU
        # tests -- host-mediated, so no kernel ever waits on another rank)
        self.staged = dist.get_backend(group) == "gloo"
        self.native = None

    def open_native(self):
        """Create the pg_dist communicator (NCCL backend only) and install
        this shard's halo plan.  Collective: every rank calls it."""
        if self.staged or os.environ.get("PG_DIST_NATIVE", "1") == "0":
            return
        uid = _lib.C.create_string_buffer(128)
        if self.rank == 0:
            _lib.call("pg_nccl_unique_id", uid, 128)
        obj = [uid.raw if self.rank == 0 else None]
        self.dist.broadcast_object_list(obj, src=0, group=self.group)
        raw = _lib.C.create_string_buffer(obj[0], 128)
        s = self.shards[0]
        h = _lib.C.c_void_p()
        _lib.call("pg_dist_create", raw, self.world, self.rank, s.dev_ord, _lib.C.byref(h))
        self.native = h
        sp = sorted(s.plan.send)
        send_peer = np.asarray(sp, dtype=np.int32)
        send_cnt = np.asarray([len(s.plan.send[q]) for q in sp], dtype=np.int64)
        send_idx = (np.concatenate([s.plan.send[q] for q in sp]).astype(np.int32)
                    if sp else np.zeros(1, np.int32))
        rp = sorted(s.plan.recv)
        recv_peer = np.asarray(rp, dtype=np.int32)
        recv_off = np.asarray([s.plan.recv[q][0] for q in rp], dtype=np.int64)
        recv_cnt = np.asarray([s.plan.recv[q][1] for q in rp], dtype=np.int64)
        _lib.call("pg_dist_set_halo", h, len(sp), send_peer.ctypes.data, send_cnt.ctypes.data,
                  send_idx.ctypes.data, len(rp), recv_peer.ctypes.data, recv_off.ctypes.data,
                  recv_cnt.ctypes.data)

    def close(self):
        if self.native is not None:
            _lib.call("pg_dist_destroy", self.native)
            self.native = None

    def halo(self, xs):
        dist = self.dist
        s = self.shards[0]
        x = xs[0]
        ops, landing = [], []
        for q in sorted(s.plan.send):
            buf = s.packed_send(x, q)
            if self.staged and buf.is_cuda:
                buf = buf.cpu()
            ops.append(dist.P2POp(dist.isend, buf, q, self.group))
        for q, (off, cnt) in sorted(s.plan.recv.items()):
            dst = x[off:off + cnt]
            if self.staged and dst.is_cuda:
                tmp = torch.empty(cnt, dtype=dst.dtype)
                landing.append((dst, tmp))
                dst = tmp
            ops.append(dist.P2POp(dist.irecv, dst, q, self.group))
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()
        for dst, tmp in landing:
            dst.copy_(tmp)

    def any(self, flag: bool) -> bool:
        """Logical OR of a per-rank flag over the group."""
        dev = "cpu" if self.staged else self.shards[0].device
        t = torch.tensor([1 if flag else 0], dtype=torch.int32, device=dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return bool(t.item())

    def allreduce(self, bufs):
        """In-place sum over the ranks: all-gather, then ((b0 + b1) + b2) ..."""
        b = bufs[0]
        src = b.cpu() if (self.staged and b.is_cuda) else b
        parts = [torch.empty_like(src) for _ in range(self.world)]
        self.dist.all_gather(parts, src.contiguous(), group=self.group)
        total = parts[0].clone()
        for p in parts[1:]:
            total += p
        b.copy_(total)


def exchange_send_lists(shards, comm):
    """Turn every shard's ghost needs into the owners' send lists (the
    Epetra-Import construction).  In-process: direct; distributed: one
    all_gather_object of the per-rank needs at setup time."""
    if isinstance(comm, SoloComm):
        for p, s in enumerate(shards):
            for q, (off, cnt) in s.plan.recv.items():
                need = s.plan.ghosts[off - s.n: off - s.n + cnt]
                shards[q].set_send(p, need - shards[q].r0)
        return
    s = shards[0]
    needs = {q: s.plan.ghosts[off - s.n: off - s.n + cnt] for q, (off, cnt) in s.plan.recv.items()}
    gathered = [None] * comm.world
    comm.dist.all_gather_object(gathered, needs, group=comm.group)
    for p, nd in enumerate(gathered):
        if p != comm.rank and comm.rank in nd:
            s.set_send(p, np.asarray(nd[comm.rank]) - s.r0)


# ---------------------------------------------------------------------------
# the engine: every vector op of the solver, over the shard list
# ---------------------------------------------------------------------------
class PgEvent:
    """A libpgmres-owned CUDA event (pg_event_*), with the two methods the
    solver and bench.py use on torch events."""

    def __init__(self, device_ordinal: int):
        h = _lib.C.c_void_p()
        _lib.call("pg_event_create", int(device_ordinal), _lib.C.byref(h))
        self.h = h

    def record(self, stream):
        _lib.call("pg_event_record", self.h, stream)

    def synchronize(self):
        _lib.call("pg_event_wait", self.h)

    def elapsed_time(self, end) -> float:
        ms = _lib.C.c_float(0.0)
        _lib.call("pg_event_elapsed", self.h, end.h, _lib.C.byref(ms))
        return float(ms.value)

    def __del__(self):
        # (at interpreter shutdown the module globals may already be gone)
        h = getattr(self, "h", None)
        lib = getattr(_lib, "_lib", None) if _lib is not None else None
        if h is not None and lib is not None:
            lib.pg_event_destroy(h)
            self.h = None


def _fast_steps_enabled() -> bool:
    return os.environ.get("PG_FAST_STEP", "1") != "0"


def _step_graphs_enabled() -> bool:
    return os.environ.get("PG_STEP_GRAPHS", "1") != "0"


class _Elapsed:
    """A chain time already read back (ms), in the (start, end) slot of the
    bench timer: ``start.elapsed_time(end)`` returns it."""

    def __init__(self, ms: float):
        self.ms = ms

    def elapsed_time(self, _end=None) -> float:
        return self.ms


class _StepGraph:
    """One Arnoldi step recorded as a CUDA graph (pg_step_graph_create) with
    its own chain-timing events."""

    def __init__(self, h, c0, c1):
        self.h, self.c0, self.c1 = h, c0, c1

    def __del__(self):
        h = getattr(self, "h", None)
        lib = getattr(_lib, "_lib", None) if _lib is not None else None
        if h is not None and lib is not None:
            lib.pg_graph_destroy(h)
            self.h = None



class HostStage:
    """Two pinned staging buffers per device for numpy (pageable) vectors --
    the reference's call signature.  A large vector moves in chunks: the host
    copy of chunk i+1 into one pinned buffer overlaps the DMA of chunk i from
    the other (torch's pageable copy staged the whole vector synchronously,
    ~40 ms of the cfg4 e2e for b, v0 and x).  Chunks are ordered on the
    caller's stream; a buffer is refilled only after its previous DMA's event."""

    CHUNK = 1 << 20  # doubles (8 MB)
    MIN = 1 << 19    # smaller vectors take the plain copy

    _per_device: dict = {}

    def __init__(self):
        self.buf = [torch.empty(self.CHUNK, dtype=F64).pin_memory() for _ in range(2)]
        self.ev = [None, None]
        self.lock = threading.Lock()

    @classmethod
    def get(cls, device) -> "HostStage":
        key = torch.device(device).index
        st = cls._per_device.get(key)
        if st is None:
            st = cls._per_device[key] = HostStage()
        return st

    def _wait(self, i):
        if self.ev[i] is not None:
            self.ev[i].synchronize()
            self.ev[i] = None

    def h2d(self, src: np.ndarray, dst: torch.Tensor):
        """dst[:len(src)] <- src (numpy, contiguous f64)."""
        with self.lock, torch.cuda.device(dst.device):
            self._h2d(src, dst)

    def d2h(self, src: torch.Tensor, out: np.ndarray):
        """out <- src[:len(out)] (device)."""
        with self.lock, torch.cuda.device(src.device):
            self._d2h(src, out)

    def _h2d(self, src, dst):
        n = src.shape[0]
        stream = torch.cuda.current_stream(dst.device)
        for c, a in enumerate(range(0, n, self.CHUNK)):
            i = c & 1
            m = min(self.CHUNK, n - a)
            self._wait(i)
            self.buf[i][:m].copy_(torch.from_numpy(src[a:a + m]))
            dst[a:a + m].copy_(self.buf[i][:m], non_blocking=True)
            self.ev[i] = torch.cuda.Event()
            self.ev[i].record(stream)
        for i in range(2):
            self._wait(i)

    def _d2h(self, src, out):
        n = out.shape[0]
        stream = torch.cuda.current_stream(src.device)
        pend = []
        for c, a in enumerate(range(0, n, self.CHUNK)):
            i = c & 1
            m = min(self.CHUNK, n - a)
            if len(pend) == 2:  # drain the chunk that used this buffer
                ja, jm, ji = pend.pop(0)
                self._wait(ji)
                out[ja:ja + jm] = self.buf[ji][:jm].numpy()
            self.buf[i][:m].copy_(src[a:a + m], non_blocking=True)
            self.ev[i] = torch.cuda.Event()
            self.ev[i].record(stream)
            pend.append((a, m, i))
        for ja, jm, ji in pend:
            self._wait(ji)
            out[ja:ja + jm] = self.buf[ji][:jm].numpy()


class Engine:
    def __init__(self, shards, comm, n_global: int):
        self.shards = shards
        self.comm = comm
        self.N = int(n_global)
        self.P = len(shards)
        # optional list collecting (start_event, end_event, algorithmic_bytes)
        # per fused polynomial pass (bench.py's live roofline measurement)
        self.timer = None
        # ILU(0) left preconditioner (attach_ilu): when set, one operator
        # application is M^{-1} A v (IluPreconditionedOperator, gmres.py:63-95)
        self.ilu = None
        self._fast = _fast_steps_enabled()
        self._done_events = None
        # recorded Arnoldi steps, keyed by everything baked into the graph;
        # a step is recorded the second time its key is seen (repeated solves)
        self._graphs_on = _step_graphs_enabled()
        self._graphs: dict = {}
        self._graph_seen: set = set()

    # ---- construction -------------------------------------------------------
    @classmethod
    def build(cls, matrix, device=None, parts: int = 1, sigma=None, offsets=None):
        """All shards in this process.  ``matrix``: whole square CSR (reference
        CsrMatrix or CsrHost); ``parts`` > 1 splits it into virtual shards."""
        require_cuda()
        n = int(matrix.nrows)
        row_ptr = np.asarray(matrix.row_ptr, dtype=np.int64)
        cols = np.asarray(matrix.col_idx, dtype=np.int64)
        vals = np.asarray(matrix.values, dtype=np.float64)
        devs = device if isinstance(device, (list, tuple)) else [device] * parts
        devs = [torch.device("cuda", torch.cuda.current_device()) if d is None else torch.device(d)
                for d in devs]
        offs = balanced_offsets(row_ptr, parts) if offsets is None else np.asarray(offsets)
        shards = []
        for p in range(parts):
            a, b = int(offs[p]), int(offs[p + 1])
            q0, q1 = int(row_ptr[a]), int(row_ptr[b])
            shards.append(Shard(p, devs[p], a, b, row_ptr[a:b + 1] - q0, cols[q0:q1],
                                vals[q0:q1], offs, sigma))
        comm = SoloComm(shards)
        exchange_send_lists(shards, comm)
        return cls(shards, comm, n)

    @classmethod
    def build_distributed(cls, block, offsets, device, group=None, sigma=None):
        """One shard per process: ``block`` is this rank's row block (global
        column indices, ``block.row_offset == offsets[rank]``)."""
        require_cuda()
        import torch.distributed as dist
        rank = dist.get_rank(group)
        offs = np.asarray(offsets, dtype=np.int64)
        if int(block.row_offset) != int(offs[rank]) or int(block.nrows) != int(offs[rank + 1] - offs[rank]):
            raise DimensionMismatchError("row block does not match the partition offsets")
        s = Shard(rank, torch.device(device), int(offs[rank]), int(offs[rank + 1]),
                  np.asarray(block.row_ptr), np.asarray(block.col_idx),
                  np.asarray(block.values), offs, sigma)
        comm = DistComm([s], group)
        exchange_send_lists([s], comm)
        comm.open_native()
        return cls([s], comm, int(offs[-1]))

    def close(self):
        if self.ilu is not None:
            _lib.call("pg_ilu_destroy", self.ilu)
            self.ilu = None
        if self.comm.distributed:
            self.comm.close()
        for s in self.shards:
            s.close()

    # ---- ILU(0) left preconditioning ---------------------------
    def attach_ilu(self, factors):
        """Device copy of ILU(0) factors (ilu.Ilu0Factors); from now on every
        operator application of this engine is M^{-1} (A v).  Serial like the
        reference (ilu.py:1-7): a single shard only."""
        if self.P != 1 or self.comm.distributed:
            raise ParameterError("ILU(0) preconditioning needs a single shard")
        s = self.shards[0]
        if int(factors.n) != s.n:
            raise DimensionMismatchError("factors do not match the matrix")
        rp = np.ascontiguousarray(factors.row_ptr, dtype=np.int64)
        ci = np.ascontiguousarray(factors.col_idx, dtype=np.int64)
        va = np.ascontiguousarray(factors.values, dtype=np.float64)
        dp = np.ascontiguousarray(factors.diag_ptr, dtype=np.int64)
        h = _lib.C.c_void_p()
        _lib.call("pg_ilu_create", s.dev_ord, s.n, rp.ctypes.data, ci.ctypes.data, va.ctypes.data,
                  dp.ctypes.data, _lib.C.byref(h))
        if self.ilu is not None:
            _lib.call("pg_ilu_destroy", self.ilu)
        self.ilu = h

    def precondition(self, vs, outs):
        """outs = M^{-1} v (two sync-free triangular sweeps)."""
        s = self.shards[0]
        tmp = self.cached_vecs("ilu_y")
        _lib.call("pg_ilu_apply", self.ilu, ptr(vs[0]), ptr(tmp[0]), ptr(outs[0]), s.stream)

    def _op_generic(self, xs, ys):
        """ys = M^{-1} (A x) (ILU engines)."""
        t = self.cached_vecs("ilu_t")
        self.halo(xs)
        s = self.shards[0]
        _lib.call("pg_spmv", s.mat, ptr(xs[0]), ptr(t[0]), s.stream)
        self.precondition(t, ys)

    @property
    def fast_steps(self) -> bool:
        """Whole Arnoldi steps / polynomial chains as one native call
        (pg_arnoldi_step / pg_poly_chain): single shard, plain SpMV operator."""
        return (self._fast and self.P == 1 and self.ilu is None
                and (not self.comm.distributed or self.native_dist is not None))

    @property
    def native_dist(self):
        """The pg_dist communicator of a distributed engine, or None."""
        return getattr(self.comm, "native", None)

    def _chain_events(self):
        if self.timer is None:
            return None, None
        s0 = self.shards[0]
        return PgEvent(s0.dev_ord), PgEvent(s0.dev_ord)

    def _time_chain(self, ev0, ev1, s, d, pass_vec_bytes):
        """Record one chain of d fused passes in the bench timer (same byte
        accounting as Engine.poly)."""
        nbytes = nbytes12 = 0
        for k, vec in enumerate(pass_vec_bytes):
            nbytes += s.pass_bytes(vec)
            nbytes12 += 12 * s.nnz + (12 + vec) * s.n
        self.timer.append((ev0, ev1, nbytes, d, nbytes12))

    @staticmethod
    def _chain_vec_bytes(d, base):
        return [8 * (int(k > 1) + 1 + int(k < d) + int(base and k == d)) for k in range(1, d + 1)]

    def arnoldi_step(self, Vs, j: int, y, W, slot: int, plan=None):
        """One native call for Arnoldi step j (fast path of gmres._launch_step):
        z = A p(A) v_j, CGS2 into column j+1, scalars copied to the pinned ring
        slot behind a library event.  A step seen before with the same
        coefficients and buffers is replayed as a recorded CUDA graph.
        Returns a cgs2_fetch handle."""
        s = self.shards[0]
        if self._done_events is None:
            self._done_events = [PgEvent(s.dev_ord), PgEvent(s.dev_ord)]
        ev = self._done_events[slot]
        nroot, rmode, rc = 0, None, None
        if plan is not None:  # root-product chain (RootPlan.resid_steps)
            d, yarr = -1, None
            nroot = len(plan.resid_steps)
            rmode = np.ascontiguousarray([st[0] for st in plan.resid_steps], dtype=np.int32)
            rc = np.ascontiguousarray([v for st in plan.resid_steps for v in st[1:4]],
                                      dtype=np.float64)
        elif y is None:
            d, yarr = -1, None
        else:
            yarr = np.ascontiguousarray(y, dtype=np.float64)
            d = len(yarr) - 1
        host = s.pinned[slot]
        args = (s.mat, yarr.ctypes.data if yarr is not None else None, d, ptr(Vs[0]), s.ld, j,
                ptr(W.z[0]), ptr(W.t[0]), ptr(W.acc[0]), ptr(W.w0[0]), ptr(W.w1[0]),
                ptr(s.ring[slot]), host.data_ptr(), s.ws, ev.h)
        tail = (nroot, rmode.ctypes.data if rmode is not None else None,
                rc.ctypes.data if rc is not None else None)
        # the chain (d passes + wrapper SpMV, or the nroot root passes), 3 CGS2
        # phases, normalisation
        # one dependency-driven kernel for the whole chain on chain_fused
        # matrices (its timing events then also cover the wrapper SpMV)
        fused = s.chain_fused and (nroot > 1 or d > 0)
        if fused:
            nlaunch = 1 + 4
        else:
            nlaunch = (nroot if nroot else (max(d, 1) + 1 if d >= 0 else 1)) + 4
        chained = nroot > 0 or d > 0
        graph = None
        if self._graphs_on:
            key = (j, d, yarr.tobytes() if yarr is not None else b"",
                   (rmode.tobytes() + rc.tobytes()) if nroot else b"", args[3], args[6:12], s.ld,
                   id(s.mat))
            graph = self._graphs.get(key)
            if graph is None and key in self._graph_seen:
                if len(self._graphs) >= 512:  # bounded: drop the recorded set
                    self._graphs.clear()
                c0 = PgEvent(s.dev_ord) if chained else None
                c1 = PgEvent(s.dev_ord) if chained else None
                h = _lib.C.c_void_p()
                if self.native_dist is not None:
                    _lib.call("pg_step_graph_create_dist", *args, c0.h if c0 else None,
                              c1.h if c1 else None, *tail, self.native_dist, _lib.C.byref(h))
                else:
                    _lib.call("pg_step_graph_create", *args, c0.h if c0 else None,
                              c1.h if c1 else None, *tail, _lib.C.byref(h))
                graph = self._graphs[key] = _StepGraph(h, c0, c1)
            elif graph is None:
                self._graph_seen.add(key)
        if graph is not None:
            _lib.call("pg_graph_launch", graph.h, s.stream)
            c0, c1 = graph.c0, graph.c1
        else:
            c0, c1 = self._chain_events() if chained else (None, None)
            if self.native_dist is not None:
                _lib.call("pg_arnoldi_step_dist", *args, c0.h if c0 else None,
                          c1.h if c1 else None, *tail, self.native_dist, s.stream)
            else:
                _lib.call("pg_arnoldi_step", *args, c0.h if c0 else None, c1.h if c1 else None,
                          *tail, s.stream)
        _lib.add_launches("pg_arnoldi_step", nlaunch)
        timing = None
        if c0 is not None and self.timer is not None:
            if nroot:  # root passes: w write, [p read], [v read] (as wrapped_roots)
                vec = [8 * (1 + int((m & 3) == _lib.PG_ROOT_PAIR_B) +
                            int(bool(m & _lib.PG_ROOT_RESID))) for m in rmode]
                timing = (c0, c1, s, nroot, vec)
            elif fused:  # d passes + the wrapper SpMV (z write)
                timing = (c0, c1, s, d + 1, self._chain_vec_bytes(d, False) + [8])
            else:
                timing = (c0, c1, s, d, self._chain_vec_bytes(d, False))
        return ev, host, j + 1, timing

    def count_ops(self, counters, k: int):
        """Tally k operator applications (spmvs; prec_applies on ILU engines)."""
        counters.spmvs += k
        if self.ilu is not None:
            counters.prec_applies += k

    def bind_stream(self):
        """Re-read each device's current torch stream (call at every public
        entry point so `with torch.cuda.stream(...)` is honoured)."""
        for s in self.shards:
            s._stream = torch.cuda.current_stream(s.device).cuda_stream

    # ---- vectors --------------------------------------------------------------
    def vecs(self):
        return [s.vec() for s in self.shards]

    def blocks(self, cols):
        return [s.block(cols) for s in self.shards]

    def cached_blocks(self, key: str, cols: int):
        """Reusable zero-padded column blocks (>= cols columns) kept across
        calls: basis / power-sequence storage is allocated once per operator,
        not per solve.  Rows >= n of every column stay zero (kernels only
        write owned rows; halo fills rows n..n_ext before each SpMV)."""
        cache = self.__dict__.setdefault("_block_cache", {})
        blk = cache.get(key)
        if blk is None or blk[0].shape[0] < cols:
            blk = cache[key] = self.blocks(cols)
        return blk

    def cached_vecs(self, key: str):
        cache = self.__dict__.setdefault("_vec_cache", {})
        v = cache.get(key)
        if v is None:
            v = cache[key] = self.vecs()
        return v

    @property
    def local_n(self) -> int:
        return sum(s.n for s in self.shards)

    def from_host(self, v, pinned=False):
        """Global (or, distributed, rank-local) host vector -> shard vectors."""
        v = np.asarray(v, dtype=np.float64)
        out = self.vecs()
        if self.comm.distributed and v.shape == (self.local_n,):
            parts = [v]
        elif v.shape == (self.N,):
            parts = [v[s.r0:s.r1] for s in self.shards]
        else:
            raise DimensionMismatchError("vector length does not match operator")
        for s, t, part in zip(self.shards, out, parts):
            part = np.ascontiguousarray(part)
            if not pinned and part.shape[0] >= HostStage.MIN and t.is_cuda:
                HostStage.get(t.device).h2d(part, t)
                continue
            src = torch.from_numpy(part)
            if pinned:
                src = src.pin_memory()
            t[:s.n].copy_(src, non_blocking=pinned)
        return out

    def from_torch(self, v: torch.Tensor):
        if v.dtype != F64:
            v = v.to(F64)
        if v.dim() != 1:
            raise DimensionMismatchError("vector must be 1-d")
        out = self.vecs()
        if self.comm.distributed and v.shape[0] == self.local_n:
            for s, t in zip(self.shards, out):
                t[:s.n].copy_(v)
            return out
        if v.shape[0] != self.N:
            raise DimensionMismatchError("vector length does not match operator")
        # a pinned host source is copied in stream order (every public entry
        # point synchronises before it returns, so the caller's buffer is read
        # before control goes back)
        nb = (not v.is_cuda) and v.is_pinned()
        for s, t in zip(self.shards, out):
            t[:s.n].copy_(v[s.r0:s.r1], non_blocking=nb)
        return out

    def to_host(self, xs) -> np.ndarray:
        out = np.empty(self.local_n if self.comm.distributed else
                       sum(s.n for s in self.shards), dtype=np.float64)
        a = 0
        for s, t in zip(self.shards, xs):
            if s.n >= HostStage.MIN and t.is_cuda:
                HostStage.get(t.device).d2h(t[:s.n], out[a:a + s.n])
            else:
                out[a:a + s.n] = t[:s.n].cpu().numpy()
            a += s.n
        return out

    def to_torch(self, xs) -> torch.Tensor:
        if len(xs) == 1:
            return xs[0][:self.shards[0].n].clone()
        d = self.shards[0].device
        return torch.cat([t[:s.n].to(d) for s, t in zip(self.shards, xs)])

    def ingest(self, v):
        """Caller vector -> shard vectors; every public entry point starts here,
        so this is also where the launch stream is (re)bound."""
        self.bind_stream()
        if isinstance(v, torch.Tensor):
            return self.from_torch(v)
        return self.from_host(v)

    def emit(self, xs, like):
        """Result in the caller's vector type: CUDA tensor -> CUDA tensor, CPU
        tensor -> CPU tensor (one D2H copy), anything else -> numpy."""
        if isinstance(like, torch.Tensor):
            if like.is_cuda:
                return self.to_torch(xs)
            # straight into pinned memory (cached by torch's host allocator):
            # one direct DMA, no device-side clone, no pageable staging
            out = xs[0][:self.shards[0].n] if len(xs) == 1 else self.to_torch(xs)
            host = torch.empty(out.shape, dtype=out.dtype, pin_memory=True)
            host.copy_(out, non_blocking=True)
            torch.cuda.current_stream(out.device).synchronize()
            return host
        return self.to_host(xs)

    # ---- kernels ----------------------------------------------------------------
    def _each(self):
        for s in self.shards:
            if self.P > 1:
                s.activate()
            yield s

    def halo(self, xs):
        self.comm.halo(xs)

    def spmv(self, xs, ys):
        """One operator application: A x, or M^{-1} A x on an ILU engine."""
        if self.ilu is not None:
            return self._op_generic(xs, ys)
        self.halo(xs)
        for s, x, y in zip(self._each(), xs, ys):
            _lib.call("pg_spmv", s.mat, ptr(x), ptr(y), s.stream)

    def power_sequence(self, P, ncols: int):
        """P[:, k] = A P[:, k-1] for k = 1 .. ncols-1 (column 0 given): one
        native call on single-shard engines, operator applications otherwise
        (halo before each product; M^{-1} A on ILU engines)."""
        if self.fast_steps:
            s = self.shards[0]
            if self.native_dist is not None:
                _lib.call("pg_power_sequence_dist", s.mat, ptr(P[0]), s.ld, ncols,
                          self.native_dist, s.stream)
            else:
                _lib.call("pg_power_sequence", s.mat, ptr(P[0]), s.ld, ncols, s.stream)
            _lib.add_launches("pg_power_sequence", ncols - 1)
            return
        for k in range(ncols - 1):
            self.spmv([blk[k] for blk in P], [blk[k + 1] for blk in P])

    def poly(self, y, vs, out, acc, w0, w1, base=None):
        """out = (base +) p(A) v with p = sum_k y_k A^k (polyprec.py:193-212);
        d = len(y)-1 fused SpMV passes.  acc, w0, w1: scratch shard vectors."""
        y = [float(c) for c in y]
        d = len(y) - 1
        if self.ilu is not None and d > 0:
            return self._poly_generic(y, vs, out, acc, w0, w1, base)
        if self.fast_steps:
            s = self.shards[0]
            yarr = np.asarray(y, dtype=np.float64)
            c0, c1 = self._chain_events() if d > 0 else (None, None)
            b = base[0] if base is not None else None
            if self.native_dist is not None:
                _lib.call("pg_poly_chain_dist", s.mat, yarr.ctypes.data, d, ptr(vs[0]),
                          ptr(b) if b is not None else None, ptr(out[0]), ptr(acc[0]),
                          ptr(w0[0]), ptr(w1[0]), c0.h if c0 else None, c1.h if c1 else None,
                          self.native_dist, s.stream)
            else:
                _lib.call("pg_poly_chain", s.mat, yarr.ctypes.data, d, ptr(vs[0]),
                          ptr(b) if b is not None else None, ptr(out[0]), ptr(acc[0]),
                          ptr(w0[0]), ptr(w1[0]), c0.h if c0 else None, c1.h if c1 else None,
                          s.stream)
            _lib.add_launches("pg_poly_chain", max(d, 1))
            if c0 is not None:
                self._time_chain(c0, c1, s, d, self._chain_vec_bytes(d, base is not None))
            return
        if d == 0:
            for s, v, o, b in zip(self._each(), vs, out, base or [None] * self.P):
                _lib.call("pg_scale_add", ptr(b) if b is not None else None, y[0], ptr(v), s.n,
                          ptr(o), s.stream)
            return
        self.halo(vs)
        cur = vs
        ws = (w0, w1)
        timing = self.timer is not None and self.P == 1
        if timing:  # one event pair around the d back-to-back fused passes
            s0 = self.shards[0]
            ev0 = torch.cuda.Event(enable_timing=True)
            ev0.record(torch.cuda.current_stream(s0.device))
            nbytes = nbytes12 = 0
        for k in range(1, d + 1):
            last = k == d
            flags = (_lib.PG_PASS_FIRST if k == 1 else 0) | (0 if last else _lib.PG_PASS_WRITE_W)
            nxt = ws[k & 1]
            dst = out if last else acc
            for i, s in enumerate(self._each()):
                b = base[i] if (last and base is not None) else None
                _lib.call("pg_poly_pass", s.mat, ptr(cur[i]), ptr(acc[i]) if k > 1 else None,
                          ptr(b) if b is not None else None, ptr(dst[i]),
                          ptr(nxt[i]) if not last else None, y[0], y[k], flags, s.stream)
                if timing:
                    # algorithmic bytes: per nonzero the stored
                    # entry (12 B: f64 value + int32 index; 2 B with dictionary
                    # compression), 4 B row length, 8 B compulsory gather of x,
                    # then the epilogue's vector traffic
                    vec = 8 * (int(k > 1) + 1 + int(not last) + int(b is not None))
                    nbytes += s.pass_bytes(vec)
                    nbytes12 += 12 * s.nnz + (12 + vec) * s.n
            if not last:
                self.halo(nxt)
                cur = nxt
        if timing:
            ev1 = torch.cuda.Event(enable_timing=True)
            ev1.record(torch.cuda.current_stream(s0.device))
            self.timer.append((ev0, ev1, nbytes, d, nbytes12))

    def _poly_generic(self, y, vs, out, acc, w0, w1, base):
        """Running-power recurrence with a non-SpMV operator (ILU engines):
        acc = y0 v; w = op(w); acc = acc + yk w (polyprec.py:205-211), then
        out = base + acc.  Same rounding sequence as the reference."""
        s = self.shards[0]
        d = len(y) - 1
        _lib.call("pg_scale_add", None, y[0], ptr(vs[0]), s.n, ptr(acc[0]), s.stream)
        cur = vs
        ws = (w0, w1)
        for k in range(1, d + 1):
            nxt = ws[k & 1]
            self._op_generic(cur, nxt)
            last = k == d
            dst = out if (last and base is None) else acc
            _lib.call("pg_scale_add", ptr(acc[0]), y[k], ptr(nxt[0]), s.n, ptr(dst[0]), s.stream)
            cur = nxt
        if base is not None:
            _lib.call("pg_scale_add", ptr(base[0]), 1.0, ptr(acc[0]), s.n, ptr(out[0]), s.stream)

    def poly_roots(self, plan, vs, out, t, p0, p1, base=None):
        """out = (base +) p(A) v in root-product form (polyprec.RootPlan): one
        fused ``pg_root_pass`` per step, the running sum y in ``out`` (seeded
        with ``base``), the product in p0/p1 (ping-pong: every pass gathers
        it), the pair temporary in t.  vs is never written."""
        if self.ilu is not None:
            raise ParameterError("the root-product form needs the plain SpMV operator")
        if plan.degree == 0:
            for s, v, o, b in zip(self._each(), vs, out, base or [None] * self.P):
                _lib.call("pg_scale_add", ptr(b) if b is not None else None, plan.y0, ptr(v), s.n,
                          ptr(o), s.stream)
            return
        self.halo(vs)
        prod = vs
        bufs = (p0, p1)
        nb = 0
        timing = self.timer is not None and self.P == 1
        if timing:
            s0 = self.shards[0]
            ev0 = torch.cuda.Event(enable_timing=True)
            ev0.record(torch.cuda.current_stream(s0.device))
            nbytes = nbytes12 = 0
        first = True
        for mode, c1, c2, c3, keep in plan.steps:
            if mode == _lib.PG_ROOT_PAIR_B:
                x, p, w = t, prod, (bufs[nb] if keep else None)
            elif mode == _lib.PG_ROOT_PAIR_A:
                x, p, w = prod, None, (t if keep else None)
            else:
                x, p, w = prod, None, (bufs[nb] if keep else None)
            writes_y = mode != _lib.PG_ROOT_PAIR_B or c3 != 0.0
            for i, s in enumerate(self._each()):
                yin = (base[i] if base is not None else None) if first else out[i]
                _lib.call("pg_root_pass", s.mat, ptr(x[i]), ptr(p[i]) if p is not None else None,
                          ptr(yin) if (writes_y and yin is not None) else None,
                          ptr(out[i]) if writes_y else None, ptr(w[i]) if w is not None else None,
                          c1, c2, c3, mode, s.stream)
                if timing:
                    # entry stream + row lengths + x gather, then the epilogue:
                    # p read (PAIR_B), y read (unless seeded from zero), y/w writes
                    vec = 8 * (int(p is not None) + int(writes_y and yin is not None)
                               + int(writes_y) + int(w is not None))
                    nbytes += s.pass_bytes(vec)
                    nbytes12 += 12 * s.nnz + (12 + vec) * s.n
            if writes_y:
                first = False
            if w is not None:
                self.halo(w)
                if mode != _lib.PG_ROOT_PAIR_A:
                    prod = w
                    nb ^= 1
        if timing:
            ev1 = torch.cuda.Event(enable_timing=True)
            ev1.record(torch.cuda.current_stream(s0.device))
            self.timer.append((ev0, ev1, nbytes, plan.degree, nbytes12))

    def wrapped_roots(self, plan, vs, z, t, p0, p1):
        """z = A p(A) v = v - pi(A) v (RootPlan.resid_steps): d+1 fused passes
        that carry only the product -- no running sum is read or written, so
        each pass moves 16 B/row of vectors instead of the monomial's 32."""
        if self.ilu is not None:
            raise ParameterError("the root-product form needs the plain SpMV operator")
        if not plan.resid_steps:  # p == 0
            for s, v, o in zip(self._each(), vs, z):
                _lib.call("pg_scale_add", None, 0.0, ptr(v), s.n, ptr(o), s.stream)
            return
        self.halo(vs)
        prod = vs
        bufs = (p0, p1)
        nb = 0
        timing = self.timer is not None and self.P == 1
        if timing:
            s0 = self.shards[0]
            ev0 = torch.cuda.Event(enable_timing=True)
            ev0.record(torch.cuda.current_stream(s0.device))
            nbytes = nbytes12 = 0
        for mode, c1, c2, c3, _ in plan.resid_steps:
            m = mode & 3
            resid = bool(mode & _lib.PG_ROOT_RESID)
            x = t if m == _lib.PG_ROOT_PAIR_B else prod
            p = prod if m == _lib.PG_ROOT_PAIR_B else None
            w = z if resid else (t if m == _lib.PG_ROOT_PAIR_A else bufs[nb])
            for i, s in enumerate(self._each()):
                _lib.call("pg_root_pass", s.mat, ptr(x[i]), ptr(p[i]) if p is not None else None,
                          ptr(vs[i]) if resid else None, None, ptr(w[i]), c1, c2, c3, mode,
                          s.stream)
                if timing:
                    vec = 8 * (1 + int(p is not None) + int(resid))  # w, [p], [v]
                    nbytes += s.pass_bytes(vec)
                    nbytes12 += 12 * s.nnz + (12 + vec) * s.n
            if not resid:
                self.halo(w)
                if m != _lib.PG_ROOT_PAIR_A:
                    prod = w
                    nb ^= 1
        if timing:
            ev1 = torch.cuda.Event(enable_timing=True)
            ev1.record(torch.cuda.current_stream(s0.device))
            self.timer.append((ev0, ev1, nbytes, len(plan.resid_steps), nbytes12))

    def slot(self, i):
        """Per-shard 1-element device scalar slot i (0..7) after the coefficients."""
        return [s.scal[2 * KMAX + i:2 * KMAX + i + 1] for s in self.shards]

    def residual(self, xs, bs, rs, slot=4) -> float:
        """r = b - A x; returns the global sum of r^2 (host float), also left
        in device scalar slot ``slot``.  ILU engines: r = b - M^{-1} A x."""
        if self.ilu is not None:
            z = self.cached_vecs("ilu_z")
            self._op_generic(xs, z)
            s = self.shards[0]
            _lib.call("pg_scale_add", ptr(bs[0]), -1.0, ptr(z[0]), s.n, ptr(rs[0]), s.stream)
            return self.dot(rs, rs, slot=slot)
        self.halo(xs)
        nsq = self.slot(slot)
        for s, x, b, r, q in zip(self._each(), xs, bs, rs, nsq):
            _lib.call("pg_residual", s.mat, ptr(x), ptr(b), ptr(r), ptr(q), s.ws, s.stream)
        self.comm.allreduce(nsq)
        return float(nsq[0].item())

    def dot(self, xs, ys, slot=5, fetch=True):
        """Global x.y into device slot ``slot``; returns it as a host float
        unless ``fetch`` is False (then read later with :meth:`read_slot`)."""
        outs = self.slot(slot)
        for s, x, y, o in zip(self._each(), xs, ys, outs):
            _lib.call("pg_dot", ptr(x), ptr(y), s.n, ptr(o), s.ws, s.stream)
        self.comm.allreduce(outs)
        return float(outs[0].item()) if fetch else None

    def read_slot(self, slot) -> float:
        return float(self.slot(slot)[0].item())

    def normalize_dev(self, xs, nsq_slices, outs, n_rows=None):
        for s, x, q, o in zip(self._each(), xs, nsq_slices, outs):
            _lib.call("pg_normalize", ptr(x), ptr(q), s.n if n_rows is None else n_rows, ptr(o),
                      s.stream)

    def scale(self, xs, a, outs):
        for s, x, o in zip(self._each(), xs, outs):
            _lib.call("pg_scale_add", None, float(a), ptr(x), s.n, ptr(o), s.stream)

    def add(self, base, vs, outs):
        """out = base + v (x + update, gmres.py:330)."""
        for s, b, v, o in zip(self._each(), base, vs, outs):
            _lib.call("pg_scale_add", ptr(b), 1.0, ptr(v), s.n, ptr(o), s.stream)

    def cgs2(self, Vs, k, zs):
        """Two-pass CGS of z against columns 0..k-1 of V; writes w2/|w2| into
        column k.  Returns host (c1, c2, nsq) after the three batched
        all-reduces (one per phase)."""
        return self.cgs2_fetch(self.cgs2_launch(Vs, k, zs, 0))

    def cgs2_launch(self, Vs, k, zs, slot: int):
        """Asynchronous CGS2 (all three phases, their all-reduces and the
        normalisation of column k); the reduced scalars land in device ring
        slot ``slot`` (0/1), packed [c1 (k) | c2 (k) | nsq], and are copied to
        pinned host memory behind an event.  Returns a handle for
        :meth:`cgs2_fetch`."""
        bufs = [s.ring[slot] for s in self.shards]
        c1 = [b[0:k] for b in bufs]
        c2 = [b[k:2 * k] for b in bufs]
        nsq = [b[2 * k:2 * k + 1] for b in bufs]
        self._cgs2_phases(Vs, k, zs, c1, c2, nsq)
        s0 = self.shards[0]
        host = s0.pinned[slot]
        host[:2 * k + 1].copy_(bufs[0][:2 * k + 1], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(s0.device))
        return ev, host, k

    def cgs2_fetch(self, handle):
        ev, host, k = handle[:3]
        ev.synchronize()
        if len(handle) > 3 and handle[3] is not None and self.timer is not None:
            # the step's chain time, read now (a recorded step's events are
            # re-recorded by its next replay)
            c0, c1, s, d, vec = handle[3]
            self._time_chain(_Elapsed(c0.elapsed_time(c1)), None, s, d, vec)
        h = host.numpy()
        return h[:k].copy(), h[k:2 * k].copy(), float(h[2 * k])

    def _cgs2_phases(self, Vs, k, zs, c1, c2, nsq):
        if k > KMAX:
            return self._cgs2_wide(Vs, k, zs, c1, c2, nsq)
        if k > 0:
            for s, V, z, c in zip(self._each(), Vs, zs, c1):
                _lib.call("pg_cgs2_phase1", ptr(V), s.ld, k, ptr(z), s.n, ptr(c), s.ws, s.stream)
            self.comm.allreduce([c[:k] for c in c1])
            for s, V, z, a, c in zip(self._each(), Vs, zs, c1, c2):
                _lib.call("pg_cgs2_phase2", ptr(V), s.ld, k, ptr(z), s.n, ptr(a), ptr(c), s.ws,
                          s.stream)
            self.comm.allreduce([c[:k] for c in c2])
        for s, V, z, a, c, q in zip(self._each(), Vs, zs, c1, c2, nsq):
            col = V[k]
            _lib.call("pg_cgs2_phase3", ptr(V), s.ld, k, ptr(z), s.n, ptr(a), ptr(c), ptr(col),
                      ptr(q), s.ws, s.stream)
        self.comm.allreduce(nsq)
        # normalisation of column k is launched before the host looks at the
        # scalars; on breakdown the column is simply never used (ortho.py:67-70)
        self.normalize_dev([V[k] for V in Vs], nsq, [V[k] for V in Vs])

    def _cgs2_wide(self, Vs, k, zs, c1, c2, nsq):
        """CGS2 against more than KMAX columns, in column tiles (the C
        cgs2_wide with a reduction over the shards after each phase): c1 per
        tile, w1 = z - V c1 stored, c2 per tile, w2 = w1 - V c2 into column k."""
        tiles = [(t0, min(KMAX, k - t0)) for t0 in range(0, k, KMAX)]
        w1s = self.cached_vecs("cgs2_w1")
        for s, V, z, c in zip(self._each(), Vs, zs, c1):
            for t0, kt in tiles:
                _lib.call("pg_cgs2_phase1", ptr(V[t0]), s.ld, kt, ptr(z), s.n, ptr(c[t0:]), s.ws,
                          s.stream)
        self.comm.allreduce(c1)
        for s, V, z, c, w1 in zip(self._each(), Vs, zs, c1, w1s):
            for t0, kt in tiles:
                _lib.call("pg_gemv_acc", ptr(V[t0]), s.ld, kt, ptr(c[t0:]), s.n,
                          ptr(z if t0 == 0 else w1), -1.0, ptr(w1), s.stream)
        for s, V, c, w1 in zip(self._each(), Vs, c2, w1s):
            for t0, kt in tiles:
                _lib.call("pg_cgs2_phase1", ptr(V[t0]), s.ld, kt, ptr(w1), s.n, ptr(c[t0:]), s.ws,
                          s.stream)
        self.comm.allreduce(c2)
        for s, V, c, w1 in zip(self._each(), Vs, c2, w1s):
            col = V[k]
            for t0, kt in tiles:
                _lib.call("pg_gemv_acc", ptr(V[t0]), s.ld, kt, ptr(c[t0:]), s.n,
                          ptr(w1 if t0 == 0 else col), -1.0, ptr(col), s.stream)
        for s, V, q in zip(self._each(), Vs, nsq):
            _lib.call("pg_dot", ptr(V[k]), ptr(V[k]), s.n, ptr(q), s.ws, s.stream)
        self.comm.allreduce(nsq)
        self.normalize_dev([V[k] for V in Vs], nsq, [V[k] for V in Vs])

    def gemv(self, Vs, k, y_host, outs):
        """out = V[:, :k] y (gmres.py:326); KMAX-column tiles past KMAX."""
        yt = torch.from_numpy(np.ascontiguousarray(y_host, dtype=np.float64))
        for s, V, o in zip(self._each(), Vs, outs):
            s.coef[:k].copy_(yt)
            _lib.call("pg_gemv", ptr(V), s.ld, min(k, KMAX), ptr(s.coef), s.n, ptr(o), s.stream)
            for t0 in range(KMAX, k, KMAX):
                _lib.call("pg_gemv_acc", ptr(V[t0]), s.ld, min(KMAX, k - t0), ptr(s.coef[t0:]),
                          s.n, ptr(o), 1.0, ptr(o), s.stream)

    def gram(self, Ps, ncols) -> np.ndarray:
        """Global Gram matrix of the first ncols columns.  Each shard returns
        its double-double partial (hi | lo); partials are summed in
        double-double in shard order on the host (all_gather when distributed),
        so G -- and with it the Cholesky degree decision -- does not depend on
        the number of shards."""
        kk = ncols * ncols
        outs = [torch.zeros(2 * kk, dtype=F64, device=s.device) for s in self.shards]
        for s, P, o in zip(self._each(), Ps, outs):
            _lib.call("pg_gram", ptr(P), s.ld, ncols, s.n, ptr(o), s.ws, s.stream)
        parts = [o.cpu().numpy() for o in outs]
        if self.comm.distributed:
            src = torch.from_numpy(parts[0]) if self.comm.staged else outs[0]
            gathered = [torch.zeros_like(src) for _ in range(self.comm.world)]
            self.comm.dist.all_gather(gathered, src, group=self.comm.group)
            parts = [g.cpu().numpy() for g in gathered]
        hi = np.zeros(kk)
        lo = np.zeros(kk)
        for p in parts:  # TwoSum accumulation of every shard's (hi, lo)
            for x in (p[:kk], p[kk:]):
                s = hi + x
                bb = s - hi
                lo = lo + ((hi - (s - bb)) + (x - bb))
                hi = s
        return (hi + lo).reshape(ncols, ncols)

    # ---- reference-order reductions (csrc/blasorder.cu) -------------------------
    def dot_blas(self, xs, ys, slot: int, nthreads: int):
        """Global x.y in OpenBLAS ddot order (np.linalg.norm's squared sum,
        polyprec.py:46-51) into every shard's device slot ``slot``.  The order
        is defined on the global vector, so with several shards the vectors are
        first gathered onto shard 0's device (once per polynomial build)."""
        outs = self.slot(slot)
        s0 = self.shards[0]
        if self.P == 1 and not self.comm.distributed:
            _lib.call("pg_dot_blas", ptr(xs[0]), ptr(ys[0]), s0.n, nthreads, ptr(outs[0]),
                      s0.stream)
            return
        gx = self._gather_global(xs)
        gy = gx if ys is xs else self._gather_global(ys)
        s0.activate()
        _lib.call("pg_dot_blas", ptr(gx), ptr(gy), self.N, nthreads, ptr(outs[0]), s0.stream)
        for o in outs[1:]:
            o.copy_(outs[0].to(o.device))

    def _gather_global(self, xs) -> torch.Tensor:
        """The global vector on shard 0's device (rank-local device when
        distributed: an all_gather of the row blocks)."""
        s0 = self.shards[0]
        if not self.comm.distributed:
            return torch.cat([t[:s.n].to(s0.device) for s, t in zip(self.shards, xs)])
        comm = self.comm
        sizes = [int(v) for v in np.diff(s0.offsets)]
        m = max(sizes)
        src = torch.zeros(m, dtype=F64, device=s0.device)
        src[:s0.n].copy_(xs[0][:s0.n])
        if comm.staged:
            src = src.cpu()
        parts = [torch.zeros_like(src) for _ in range(comm.world)]
        comm.dist.all_gather(parts, src, group=comm.group)
        return torch.cat([p[:sz] for p, sz in zip(parts, sizes)]).to(s0.device)

    def gram_blas(self, Ps, ncols) -> np.ndarray:
        """Gram matrix of the first ncols columns in OpenBLAS syrk order
        (polyprec.py:115-122 through numpy's A.T @ A).  The shards run in row
        order, each continuing the previous one's open K-block chains and
        running sum (pg_gram_blas state), so G is bit-identical for any row
        partition.  Returns the full symmetric (ncols, ncols) host matrix."""
        npairs = ncols * (ncols + 1) // 2
        state = None
        comm = self.comm
        if comm.distributed and comm.rank > 0:
            dev = self.shards[0].device
            buf = torch.zeros(2 * npairs, dtype=F64, device="cpu" if comm.staged else dev)
            comm.dist.recv(buf, comm.rank - 1, group=comm.group)
            state = buf.to(dev)
        for s, P in zip(self._each(), Ps):
            need = _lib.C.c_int64(0)
            _lib.call("pg_gram_blas_scratch", s.n, s.r0, self.N, ncols, _lib.C.byref(need))
            scratch = torch.empty(max(int(need.value), 1), dtype=F64, device=s.device)
            out = torch.empty(2 * npairs, dtype=F64, device=s.device)
            sin = state.to(s.device) if state is not None else None
            _lib.call("pg_gram_blas", ptr(P), s.ld, ncols, s.n, s.r0, self.N,
                      ptr(sin) if sin is not None else None, ptr(out), ptr(scratch), s.stream)
            _lib.add_launches("pg_gram_blas", 2)
            state = out
        if comm.distributed:
            if comm.rank + 1 < comm.world:
                comm.dist.send(state.cpu() if comm.staged else state, comm.rank + 1,
                               group=comm.group)
            last = state.cpu() if comm.staged else state.clone()
            comm.dist.broadcast(last, comm.world - 1, group=comm.group)
            state = last
        packed = state[npairs:].cpu().numpy()
        G = np.zeros((ncols, ncols))
        iu = np.triu_indices(ncols)
        G[iu] = packed
        G.T[iu] = packed
        return G

    def copy(self, src, dst):
        for s, a, b in zip(self.shards, src, dst):
            b[:s.n].copy_(a[:s.n])
