"""Row-sharded SpMV over NVLink peer memory -- NON-PARITY extension.

The reference multiplies by the whole K with scipy's csr_matvec (linalg.py:27-32) and has no
distributed path (the paper's MPI runs are out of scope).  For operators beyond one
GPU this module cuts K into contiguous row blocks, one per rank (one process per GPU):

* `partition_rows`  -- row blocks balanced by stored entries (the bytes an SpMV streams);
* `ShardPlan`       -- rank p's rows with every column rewritten as `owner << 29 | offset`;
* `ShardedOperator` -- the device objects.  Each rank keeps its slice of x in an IPC-exported
  buffer (`dpp_peerbuf_*`); the handles are exchanged once through `torch.distributed`
  (all_gather_object, NCCL or gloo: plumbing only) and mapped by every peer.  `matvec` writes the
  local slice, crosses a barrier, and launches `k_shard_spmv`, which reads off-rank entries of x
  directly through the peer mappings -- there is no all-gather and no halo buffer.  A second
  barrier keeps a rank from overwriting its slice while peers still read it.

Row sums are lane-parallel, so results equal csr_matvec up to the order of additions (a few ulp):
outside the bit-exact contract, like any sharded preconditioner.  There is no CPU
path: without libdpp / a CUDA device every device call raises DeviceUnavailable.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from . import _native as N

MAX_RANKS = 8
OFF_BITS = 29


def partition_rows(indptr, world: int) -> np.ndarray:
    """starts[world + 1]: contiguous row blocks with (nearly) equal stored entries."""
    indptr = np.asarray(indptr, dtype=np.int64)
    n = len(indptr) - 1
    if not 1 <= world <= MAX_RANKS:
        raise ValueError(f"world size {world}: between 1 and {MAX_RANKS} ranks")
    if n < world:
        raise ValueError(f"{n} rows cannot be cut into {world} non-empty blocks")
    nnz = int(indptr[-1])
    targets = (np.arange(1, world, dtype=np.int64) * nnz) // world
    cuts = np.searchsorted(indptr, targets, side="left")
    starts = np.concatenate(([0], cuts, [n])).astype(np.int64)
    for p in range(1, world):            # keep every block non-empty
        starts[p] = min(max(starts[p], starts[p - 1] + 1), n - (world - p))
    return starts


def node_interleaved_order(sizes, per_node) -> np.ndarray:
    """perm[new] = old index: the DoFs of node v of every field next to each other.

    The reference orders K field by field, (u1, p1, u2, p2) (assembly.py:102-108), so a contiguous
    row block holds one field of the whole mesh and most of its columns belong to other ranks.
    For nodal formulations (CG-VMS: per_node = (dim, 1, dim, 1), velocity DoF = node * dim +
    component) this order makes a row block a slab of the mesh and only the slab faces couple
    ranks.  Apply it as K[perm][:, perm]; vectors permute the same way (x_new = x[perm]).
    """
    sizes = [int(n) for n in sizes]
    per_node = [int(k) for k in per_node]
    if len(sizes) != len(per_node) or any(k < 1 for k in per_node):
        raise ValueError("one positive DoF count per node for every field")
    nodes = {n // k for n, k in zip(sizes, per_node)}
    if len(nodes) != 1 or any(n % k for n, k in zip(sizes, per_node)):
        raise ValueError("fields do not share one node set (not a nodal formulation)")
    V = nodes.pop()
    off = np.concatenate(([0], np.cumsum(sizes)[:-1]))
    cols = [off[f] + np.arange(V)[:, None] * k + np.arange(k)[None, :] for f, k in enumerate(per_node)]
    return np.concatenate(cols, axis=1).ravel().astype(np.int64)


def encode_columns(indices, starts) -> np.ndarray:
    """uint32 codes `owner << 29 | offset in the owner's slice` for global column indices."""
    starts = np.asarray(starts, dtype=np.int64)
    idx = np.asarray(indices, dtype=np.int64)
    if len(starts) - 1 > MAX_RANKS:
        raise ValueError(f"more than {MAX_RANKS} ranks")
    if len(idx) and (idx.min() < 0 or idx.max() >= starts[-1]):
        raise ValueError("column index outside the partition")
    if np.diff(starts).max(initial=0) > 1 << OFF_BITS:
        raise ValueError("a rank's slice exceeds 2^29 rows")
    owner = np.searchsorted(starts, idx, side="right") - 1
    return ((owner << OFF_BITS) | (idx - starts[owner])).astype(np.uint32)


@dataclass
class ShardPlan:
    """Rank `rank`'s row block of a square CSR matrix, columns coded by owner."""
    rank: int
    world: int
    starts: np.ndarray          # (world + 1,)
    indptr: np.ndarray          # int32, local rows
    codes: np.ndarray           # uint32
    values: np.ndarray          # float64
    halo_entries: int           # stored entries whose column lives on another rank

    @classmethod
    def from_global(cls, A, rank: int, world: int, starts=None) -> "ShardPlan":
        A = sp.csr_matrix(A)
        if A.shape[0] != A.shape[1]:
            raise ValueError("sharded SpMV expects a square operator (x and y share the partition)")
        if not 0 <= rank < world:
            raise ValueError(f"rank {rank} outside world {world}")
        starts = partition_rows(A.indptr, world) if starts is None else np.asarray(starts, dtype=np.int64)
        if len(starts) != world + 1 or starts[0] != 0 or starts[-1] != A.shape[0] or np.any(np.diff(starts) < 0):
            raise ValueError("starts must be a monotone partition of the rows")
        r0, r1 = int(starts[rank]), int(starts[rank + 1])
        lo, hi = int(A.indptr[r0]), int(A.indptr[r1])
        codes = encode_columns(A.indices[lo:hi], starts)
        halo = int(np.count_nonzero((codes >> OFF_BITS) != rank))
        return cls(rank, world, starts, (A.indptr[r0:r1 + 1] - lo).astype(np.int32), codes,
                   np.ascontiguousarray(A.data[lo:hi], dtype=np.float64), halo)

    @property
    def rows(self) -> int:
        return len(self.indptr) - 1

    def seg_len(self) -> np.ndarray:
        return np.diff(self.starts).astype(np.int64)


class PeerBuffer:
    """An FP64 slice in HBM that other ranks can map over CUDA IPC."""

    def __init__(self, n=None, *, _handle=None, _n=None):
        if _handle is not None:
            self.h, self.n = _handle, _n
            return
        h = C.c_void_p()
        N.call("dpp_peerbuf_create", N.ctx(), int(n), C.byref(h))
        self.h, self.n = h, int(n)

    @classmethod
    def open(cls, ipc: bytes, n: int) -> "PeerBuffer":
        raw = (C.c_ubyte * 64).from_buffer_copy(ipc)
        h = C.c_void_p()
        N.call("dpp_peerbuf_open", N.ctx(), C.cast(raw, C.c_void_p), int(n), C.byref(h))
        return cls(_handle=h, _n=int(n))

    def export(self) -> bytes:
        raw = (C.c_ubyte * 64)()
        N.call("dpp_peerbuf_export", self.h, C.cast(raw, C.c_void_p))
        return bytes(raw)

    def write(self, x):
        x = N.f64(x)
        if x.ndim != 1 or len(x) > self.n:
            raise ValueError(f"slice of length {x.shape} does not fit a buffer of {self.n}")
        N.call("dpp_peerbuf_write", self.h, N.ptr(x), len(x))

    def read(self, n=None) -> np.ndarray:
        out = np.empty(self.n if n is None else int(n))
        N.call("dpp_peerbuf_read", self.h, N.ptr(out), len(out))
        return out

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and N._lib is not None:
            N.lib().dpp_peerbuf_destroy(h)
            self.h = None


class _DeviceShard:
    def __init__(self, plan: ShardPlan):
        self.plan = plan
        seg = plan.seg_len()
        h = C.c_void_p()
        N.call("dpp_shard_create", N.ctx(), plan.rows, len(plan.values), N.ptr(plan.indptr),
               N.ptr(plan.codes), N.ptr(plan.values), plan.world, N.ptr(seg), C.byref(h))
        self.h = h
        self.y = PeerBuffer(plan.rows)

    def _segs(self, xbufs):
        return (C.c_void_p * len(xbufs))(*[b.h for b in xbufs])

    def spmv(self, xbufs):
        N.call("dpp_shard_spmv", N.ctx(), self.h, self._segs(xbufs), self.y.h)
        return self.y

    def profile(self, xbufs, reps=20):
        ms, by = C.c_double(), C.c_double()
        N.call("dpp_shard_profile", N.ctx(), self.h, self._segs(xbufs), self.y.h, int(reps),
               C.byref(ms), C.byref(by))
        return ms.value, by.value

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and N._lib is not None:
            N.lib().dpp_shard_destroy(h)
            self.h = None


class ShardedOperator:
    """y_local = K[rows of this rank, :] @ x, x sharded by the same row partition.

    `ShardedOperator(A)` under an initialised `torch.distributed` group (one process per GPU)
    builds this rank's shard and maps every peer's x slice; without a group it is the
    single-rank operator.  Every rank passes the same global matrix (or one with at least its own
    rows filled: only rows [starts[rank], starts[rank+1]) are read when `starts` is given).
    With `perm` the operator is K[perm][:, perm] and every slice is in that ordering.
    """

    def __init__(self, A, group=None, starts=None, perm=None):
        self.group = group
        self.rank, self.world = _rank_world(group)
        if perm is not None:
            perm = np.asarray(perm, dtype=np.int64)
            A = sp.csr_matrix(sp.csr_matrix(A)[perm][:, perm])
            A.sort_indices()
        self.perm = perm
        self.plan = ShardPlan.from_global(A, self.rank, self.world, starts)
        self.shard = _DeviceShard(self.plan)
        seg = self.plan.seg_len()
        self.x = PeerBuffer(int(seg[self.rank]))
        self.xsegs = [None] * self.world
        self.xsegs[self.rank] = self.x
        if self.world > 1:
            import torch.distributed as dist
            handles = [None] * self.world
            dist.all_gather_object(handles, self.x.export(), group=group)
            for p in range(self.world):
                if p != self.rank:
                    self.xsegs[p] = PeerBuffer.open(handles[p], int(seg[p]))

    @property
    def shape(self):
        n = int(self.plan.starts[-1])
        return (n, n)

    @property
    def local_rows(self):
        return int(self.plan.starts[self.rank]), int(self.plan.starts[self.rank + 1])

    def _barrier(self):
        if self.world > 1:
            import torch.distributed as dist
            dist.barrier(group=self.group)

    def matvec(self, x_local) -> np.ndarray:
        """The local rows of K @ x; x_local is this rank's slice of x (collective call)."""
        r0, r1 = self.local_rows
        x_local = N.f64(x_local)
        if x_local.shape != (r1 - r0,):
            raise ValueError(f"expected this rank's slice of length {r1 - r0}, got {x_local.shape}")
        self.x.write(x_local)
        self._barrier()                      # every slice is in place before any peer reads it
        y = self.shard.spmv(self.xsegs).read(r1 - r0)
        self._barrier()                      # nobody rewrites a slice a peer may still be reading
        return y

    def profile(self, reps=20):
        """(ms per launch, algorithmic bytes per launch) of the local kernel, CUDA-event timed."""
        self._barrier()
        out = self.shard.profile(self.xsegs, reps)
        self._barrier()
        return out


class LocalShards:
    """All `world` shards of A in ONE process on one GPU (x slices are sibling buffers, no IPC).

    For checking the plan and the kernel where only one GPU is at hand, and for timing the kernel
    with its coded-column loads; launches run one after another and never wait on one another.
    `perm` (e.g. `node_interleaved_order`) reorders the operator first; `matvec` still takes and
    returns vectors in the caller's ordering.
    """

    def __init__(self, A, world: int, starts=None, perm=None):
        A = sp.csr_matrix(A)
        self.perm = None if perm is None else np.asarray(perm, dtype=np.int64)
        if self.perm is not None:
            A = sp.csr_matrix(A[self.perm][:, self.perm])
            A.sort_indices()
        self.world = world
        self.plans = [ShardPlan.from_global(A, p, world, starts) for p in range(world)]
        self.starts = self.plans[0].starts
        self.shards = [_DeviceShard(pl) for pl in self.plans]
        self.xsegs = [PeerBuffer(int(n)) for n in self.plans[0].seg_len()]

    def matvec(self, x) -> np.ndarray:
        x = N.f64(x)
        if x.shape != (int(self.starts[-1]),):
            raise ValueError(f"dimension mismatch: {x.shape}")
        if self.perm is not None:
            x = np.ascontiguousarray(x[self.perm])
        for p, b in enumerate(self.xsegs):
            b.write(x[self.starts[p]:self.starts[p + 1]])
        y = np.concatenate([s.spmv(self.xsegs).read(s.plan.rows) for s in self.shards])
        if self.perm is not None:
            out = np.empty_like(y)
            out[self.perm] = y
            return out
        return y

    def profile(self, reps=20):
        return [s.profile(self.xsegs, reps) for s in self.shards]


def _rank_world(group):
    try:
        import torch.distributed as dist
    except ImportError:
        return 0, 1
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1
