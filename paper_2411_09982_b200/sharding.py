"""Multi-GPU sharding of the two paths; one process per GPU.

* Magnus: contiguous interval blocks per rank.  Each rank computes its
  intervals' propagators and block product B_r = U_last ... U_first on its
  GPU, the ranks all-gather the B's (NCCL over NVLink; the ONLY collective),
  rank r applies B_{r-1} ... B_0 to psi0 and finishes its trajectory slice.
* NPAD sweeps: independent operators, contiguous point blocks per rank, no
  collective on the data path (results optionally gathered for reporting).
  A single NPAD solve is never split across GPUs (serial greedy chain).

The per-rank compute is injectable so the host logic (partition, exchange,
prefix order) is testable on CPU with the gloo backend; the default compute
is libqcheff on the rank's GPU.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import DimensionMismatch, GridMismatch, NormDrift


def shard_bounds(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [start, stop) block of ``total`` units for ``rank``; the
    first ``total % world`` ranks get one extra unit."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(int(total), int(world))
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


class DeviceMagnusCompute:
    """libqcheff on the current CUDA device (N <= 4): pass 1 = the fused
    single-pass kernel in prefix mode (qch_magnus_shard_prepare_c128), pass 2
    = one mat-vec chain per thread from the stored prefixes
    (qch_magnus_shard_finish_c128)."""

    def __init__(self):
        self.t = _lib.require_cuda()

    def prepare(self, ch, signals_slice, dt, dt_int, m_local, order, check):
        t = self.t
        from .magnus import _commutators

        h0, hk = ch.device_operators()
        comm = _commutators(ch) if order >= 2 and ch.num_controls else None
        sig = _lib.to_device(np.ascontiguousarray(signals_slice), t.float64)
        nbytes = int(_lib.load().qch_magnus_shard_workspace_bytes(ch.dim, m_local))
        work = t.empty(nbytes // 8 + 8, dtype=t.float64, device="cuda")
        block = t.empty((ch.dim, ch.dim), dtype=t.complex128, device="cuda")
        _lib.call(
            "qch_magnus_shard_prepare_c128", _lib.dptr(h0), _lib.dptr(hk), _lib.dptr(comm), ch.num_controls, ch.dim,
            _lib.dptr(sig), sig.shape[1], float(dt), float(dt_int), int(m_local), int(order), 1 if check else 0,
            _lib.dptr(work), _lib.dptr(block), _lib.stream_ptr(),
        )
        return block, (work, sig, comm, ch.dim, m_local, check)

    def apply_prefix(self, blocks, rank, psi0):
        t = self.t
        n = int(psi0.shape[0])
        out = t.empty(n, dtype=t.complex128, device="cuda")
        _lib.call("qch_magnus_apply_prefix_c128", _lib.dptr(blocks), n, int(rank), _lib.dptr(psi0), _lib.dptr(out),
                  _lib.stream_ptr())
        return out

    def finish(self, handle, psi_start):
        t = self.t
        work, _sig, _comm, n, m_local, check = handle
        traj = t.empty((m_local + 1, n), dtype=t.complex128, device="cuda")
        bad = ctypes.c_int64(-1)
        st = _lib.load().qch_magnus_shard_finish_c128(n, m_local, _lib.dptr(work), _lib.dptr(psi_start),
                                                     _lib.dptr(traj), 1 if check else 0, ctypes.byref(bad),
                                                     _lib.stream_ptr())
        if st == 9:
            raise NormDrift(f"state norm drifted after local interval {bad.value}")
        _lib.check(st)
        return traj

    def to_tensor(self, psi0):
        return _lib.to_device(np.asarray(psi0, dtype=np.complex128))


class ShardedEvolvePlan:
    """A sharded evolve set up once and run many times (new API; the
    multi-GPU counterpart of ``magnus.EvolvePlan``): this rank's signal slice,
    workspace and exchange buffers stay on the device, so a step is
    pass 1 (one fused launch) -> ONE NCCL all-gather of the N x N block
    products -> apply the rank's prefix -> pass 2 (one launch), with no host
    synchronisation (``check()`` reads the status words afterwards)."""

    def __init__(self, ch, grid, num_intervals: int, psi0, *, order: int = 1, check: bool = True, group=None):
        import torch.distributed as dist

        t = _lib.require_cuda()
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        m = int(num_intervals)
        if m < 1 or (grid.samples - 1) % m:
            raise GridMismatch(f"{m} intervals do not divide {grid.samples - 1} sample steps")
        if grid.num_controls != ch.num_controls:
            raise DimensionMismatch("grid / Hamiltonian control count mismatch")
        if m < self.world:
            raise ValueError("need at least one interval per rank")
        if ch.dim > 4:
            raise NotImplementedError("sharded evolve covers N <= 4 (the fused pipeline)")
        from .magnus import _as_state, _commutators

        self.sub = (grid.samples - 1) // m
        self.start, self.stop = shard_bounds(m, self.world, self.rank)
        self.m_local = self.stop - self.start
        self.n = ch.dim
        self.order, self.check_u = int(order), bool(check)
        self.dt, self.dt_int = float(grid.dt), (grid.t_end - grid.t_start) / m
        self.ch = ch
        self.h0, self.hk = ch.device_operators()
        self.comm = _commutators(ch) if order >= 2 and ch.num_controls else None
        sig = grid.signals if ch.num_controls else np.zeros((1, grid.samples))
        self.sig = _lib.to_device(np.ascontiguousarray(sig[:, self.start * self.sub: self.stop * self.sub + 1]),
                                  t.float64)
        self.psi0 = _lib.to_device(_as_state(psi0))
        nbytes = int(_lib.load().qch_magnus_shard_workspace_bytes(self.n, self.m_local))
        self.work = t.empty(nbytes // 8 + 8, dtype=t.float64, device="cuda")
        self.block = t.empty((self.n, self.n), dtype=t.complex128, device="cuda")
        self.blocks = t.empty((self.world, self.n, self.n), dtype=t.complex128, device="cuda")
        self.psi_start = t.empty(self.n, dtype=t.complex128, device="cuda")
        self.traj = t.empty((self.m_local + 1, self.n), dtype=t.complex128, device="cuda")
        self.flags = t.empty(2, dtype=t.int64, device="cuda")

    def run(self):
        import torch.distributed as dist

        lib, sp = _lib.load(), _lib.stream_ptr()
        _lib.check(lib.qch_magnus_shard_prepare_c128(
            _lib.dptr(self.h0), _lib.dptr(self.hk), _lib.dptr(self.comm), self.ch.num_controls, self.n,
            _lib.dptr(self.sig), self.sig.shape[1], self.dt, self.dt_int, self.m_local, self.order,
            1 if self.check_u else 0, _lib.dptr(self.work), _lib.dptr(self.block), sp))
        if self.world > 1:
            dist.all_gather_into_tensor(self.blocks, self.block, group=self.group)
        else:
            self.blocks[0].copy_(self.block)
        _lib.check(lib.qch_magnus_apply_prefix_c128(_lib.dptr(self.blocks), self.n, self.rank, _lib.dptr(self.psi0),
                                                    _lib.dptr(self.psi_start), sp))
        _lib.check(lib.qch_magnus_shard_finish_async_c128(self.n, self.m_local, _lib.dptr(self.work),
                                                          _lib.dptr(self.psi_start), _lib.dptr(self.traj),
                                                          _lib.dptr(self.flags), sp))
        return self.traj

    def check(self) -> None:
        a, b = (int(x) for x in _lib.to_host(self.flags).view(np.uint64))
        if self.check_u and a != (1 << 64) - 1:
            from .errors import NonFinite

            raise NonFinite(f"propagator not unitary (interval {self.start + a})")
        if b != (1 << 64) - 1:
            raise NormDrift(f"state norm drifted after interval {self.start + b}")


@dataclass
class ShardResult:
    start: int            # first interval owned by this rank
    stop: int             # one past the last
    trajectory: object    # (stop - start + 1, N): states at interval boundaries start..stop


def evolve_sharded(ch, grid, num_intervals: int, psi0, *, order: int = 1, check: bool = True, group=None,
                   compute=None) -> ShardResult:
    """Distributed ``evolve``: call on every rank of ``group`` (default: the
    WORLD process group).  Each rank returns its slice of the trajectory."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    m = int(num_intervals)
    if m < 1 or (grid.samples - 1) % m:
        raise GridMismatch(f"{m} intervals do not divide {grid.samples - 1} sample steps")
    if grid.num_controls != ch.num_controls:
        raise DimensionMismatch("grid / Hamiltonian control count mismatch")
    if m < world:
        raise ValueError("need at least one interval per rank")
    sub = (grid.samples - 1) // m
    start, stop = shard_bounds(m, world, rank)
    compute = compute or DeviceMagnusCompute()
    sig = grid.signals[:, start * sub: stop * sub + 1]
    dt_int = (grid.t_end - grid.t_start) / m
    block, handle = compute.prepare(ch, sig, grid.dt, dt_int, stop - start, order, check)
    blocks = [block.new_empty(block.shape) for _ in range(world)]
    dist.all_gather(blocks, block.contiguous(), group=group)
    import torch

    stacked = torch.stack(blocks).contiguous()
    psi_start = compute.apply_prefix(stacked, rank, compute.to_tensor(psi0))
    traj = compute.finish(handle, psi_start)
    return ShardResult(start, stop, traj)


def sweep_shard(points: np.ndarray, world: int, rank: int) -> np.ndarray:
    """The sweep points (rows) owned by ``rank`` (no collective needed)."""
    a, b = shard_bounds(points.shape[0], world, rank)
    return points[a:b]
