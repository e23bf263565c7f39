"""Multi-GPU sharding of the two paths; one process per GPU.

* Magnus, N <= 4: contiguous interval blocks per rank.  Each rank computes
  its intervals' propagators and block product B_r = U_last ... U_first on
  its GPU, the ranks all-gather the B's (NCCL over NVLink; the ONLY
  collective), rank r applies B_{r-1} ... B_0 to psi0 and finishes its
  trajectory slice.
* Magnus, N > 4 (config 5: N = 4096, 8 N^3 flop per block product would add a
  sixth to the work, and one rank cannot hold its intervals' propagators):
  chunks of c intervals dealt round-robin (chunk k -> rank k mod W).  Every
  rank computes its chunk's propagators (all ranks in parallel), then the
  state is RELAYED: rank r receives psi at the chunk start from rank r-1
  (NCCL send/recv, N complex = 64 KiB), applies its c propagators (the
  reference's sequential product, magnus.py:249-252) and sends psi on.  The
  relay of one wave of W chunks costs W chain steps (~0.3 ms each at
  N = 4096) against ~0.5 s of propagators per chunk, so the ranks stay busy.
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

    def _prepare(self):
        lib, sp = _lib.load(), _lib.stream_ptr()
        _lib.check(lib.qch_magnus_shard_prepare_c128(
            _lib.dptr(self.h0), _lib.dptr(self.hk), _lib.dptr(self.comm), self.ch.num_controls, self.n,
            _lib.dptr(self.sig), self.sig.shape[1], self.dt, self.dt_int, self.m_local, self.order,
            1 if self.check_u else 0, _lib.dptr(self.work), _lib.dptr(self.block), sp))

    def _finish(self):
        lib, sp = _lib.load(), _lib.stream_ptr()
        _lib.check(lib.qch_magnus_apply_prefix_c128(_lib.dptr(self.blocks), self.n, self.rank, _lib.dptr(self.psi0),
                                                    _lib.dptr(self.psi_start), sp))
        _lib.check(lib.qch_magnus_shard_finish_async_c128(self.n, self.m_local, _lib.dptr(self.work),
                                                          _lib.dptr(self.psi_start), _lib.dptr(self.traj),
                                                          _lib.dptr(self.flags), sp))

    def run(self):
        import torch.distributed as dist

        self._prepare()
        if self.world > 1:
            dist.all_gather_into_tensor(self.blocks.view(-1), self.block.view(-1), group=self.group)
        else:
            self.blocks[0].copy_(self.block)
        self._finish()
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


# -- Magnus N > 4: round-robin chunks + psi relay ---------------------------------

class DeviceRelayCompute:
    """libqcheff on the rank's GPU for N > 4: propagators of a chunk
    (qch_magnus_propagators_c128: coefficients, assembly incl. the second
    order, exp(-i Hbar) on the DMMA GEMMs, optional validate) and the ordered
    product over them (qch_magnus_chain_c128)."""

    def __init__(self):
        self.t = _lib.require_cuda()
        self._u = None

    def setup(self, ch, order):
        from .magnus import _commutators

        self.ch = ch
        self.h0, self.hk = ch.device_operators()
        self.comm = _commutators(ch) if order >= 2 and ch.num_controls else None

    def propagators(self, ch, signals_slice, dt, dt_int, m, order, check):
        t = self.t
        n = ch.dim
        if self._u is None or self._u.shape[0] < m:
            self._u = t.empty((m, n, n), dtype=t.complex128, device="cuda")
        sig = _lib.to_device(np.ascontiguousarray(signals_slice if ch.num_controls else np.zeros((1, signals_slice.shape[1]))),
                             t.float64)
        bad = ctypes.c_int64(-1)
        st = _lib.load().qch_magnus_propagators_c128(
            _lib.dptr(self.h0), _lib.dptr(self.hk), _lib.dptr(self.comm), ch.num_controls, n, _lib.dptr(sig),
            sig.shape[1], float(dt), float(dt_int), int(m), int(order), 1 if check else 0, _lib.dptr(self._u),
            ctypes.byref(bad), _lib.stream_ptr())
        if st != 0:
            return None, (st, int(bad.value), _lib.last_error())
        return self._u, None

    def chain(self, u, m, psi_in):
        t = self.t
        rows = t.empty((m, psi_in.shape[0]), dtype=t.complex128, device="cuda")
        bad = ctypes.c_int64(-1)
        st = _lib.load().qch_magnus_chain_c128(_lib.dptr(u), int(psi_in.shape[0]), int(m), _lib.dptr(psi_in),
                                              _lib.dptr(rows), ctypes.byref(bad), _lib.stream_ptr())
        if st != 0:
            return rows, (st, int(bad.value), _lib.last_error())
        return rows, None

    def to_tensor(self, psi):
        return _lib.to_device(np.asarray(psi, dtype=np.complex128))

    def empty(self, n):
        return self.t.empty(n, dtype=self.t.complex128, device="cuda")


_ERRCODE = {9: NormDrift}


def _p2p(op, tensor, peer, group):
    """send / recv of a device tensor; backends without device-memory
    point-to-point (gloo) go through a host copy."""
    import torch.distributed as dist

    if tensor.is_cuda and dist.get_backend(group) != "nccl":
        host = tensor.cpu()
        if op == "send":
            dist.send(host, dst=peer, group=group)
        else:
            dist.recv(host, src=peer, group=group)
            tensor.copy_(host)
        return
    if op == "send":
        dist.send(tensor, dst=peer, group=group)
    else:
        dist.recv(tensor, src=peer, group=group)


@dataclass
class RelayResult:
    num_intervals: int
    chunk: int
    world: int
    rank: int
    chunks: list          # [(start, stop, rows (stop-start, N) tensor)] owned by this rank
    psi0: object          # tensor (N,)

    def local_trajectory(self):
        """{interval index n: state after interval n} for this rank's chunks."""
        return {a: rows for a, _, rows in self.chunks}

    def gather(self, group=None):
        """The whole (M+1, N) trajectory on every rank (one all-gather)."""
        import torch
        import torch.distributed as dist

        n = int(self.psi0.shape[0])
        per = -(-self.num_intervals // self.chunk)  # chunks in total
        mine = -(-per // self.world)                 # chunk slots per rank
        buf = self.psi0.new_zeros((mine, self.chunk, n))
        for q, (a, b, rows) in enumerate(self.chunks):
            buf[q, : b - a].copy_(rows)
        if self.world > 1:
            parts = [buf.new_empty(buf.shape) for _ in range(self.world)]
            dist.all_gather(parts, buf, group=group)
            allb = torch.stack(parts)
        else:
            allb = buf.unsqueeze(0)
        out = self.psi0.new_empty((self.num_intervals + 1, n))
        out[0].copy_(self.psi0)
        for k in range(per):
            a, b = k * self.chunk, min(self.num_intervals, (k + 1) * self.chunk)
            out[a + 1: b + 1].copy_(allb[k % self.world, k // self.world, : b - a])
        return out


def relay_chunk(n: int, num_intervals: int, world: int, budget_bytes: float = 4 * 2**30) -> int:
    """Intervals per chunk: the chunk's propagators within ``budget_bytes``,
    and at least one chunk per rank."""
    per = 16 * n * n
    c = max(1, int(budget_bytes // per))
    return max(1, min(c, -(-num_intervals // world)))


def evolve_relay(ch, grid, num_intervals: int, psi0, *, order: int = 1, check: bool = True, chunk: int | None = None,
                 group=None, compute=None) -> RelayResult:
    """Distributed ``evolve`` for N > 4 (call on every rank of ``group``):
    chunk k of ``chunk`` intervals belongs to rank k mod W; each rank forms
    its chunks' propagators, receives the state at the chunk start from the
    rank before it, applies them in order and passes the state on.  Errors
    (NonFinite from check, NormDrift) travel with the relayed state so every
    rank raises the same exception (the first in interval order, as the
    reference's streamed path, magnus.py:254-260)."""
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    m = int(num_intervals)
    if m < 1 or (grid.samples - 1) % m:
        raise GridMismatch(f"{m} intervals do not divide {grid.samples - 1} sample steps")
    if grid.num_controls != ch.num_controls:
        raise DimensionMismatch("grid / Hamiltonian control count mismatch")
    from .magnus import _as_state

    psi0 = _as_state(psi0)
    if psi0.size != ch.dim:
        raise DimensionMismatch(f"state dim {psi0.size} does not match operator dim {ch.dim}")
    sub = (grid.samples - 1) // m
    c = int(chunk) if chunk else relay_chunk(ch.dim, m, world)
    n_chunks = -(-m // c)
    compute = compute or DeviceRelayCompute()
    compute.setup(ch, order)
    dt, dt_int = grid.dt, (grid.t_end - grid.t_start) / m
    n = ch.dim
    p0 = compute.to_tensor(psi0)
    msg = compute.empty(n + 1)  # psi + one status slot (code, interval)
    out = []
    err = None
    carry = None
    for k in range(rank, n_chunks, world):
        a, b = k * c, min(m, (k + 1) * c)
        u = None
        if err is None:
            u, e = compute.propagators(ch, grid.signals[:, a * sub: b * sub + 1], dt, dt_int, b - a, order, check)
            if e is not None:
                err = (e[0], a + e[1], e[2])
        # the state at the chunk start
        if k == 0:
            psi_in, in_err = p0, None
        elif world == 1:
            psi_in, in_err = carry
        else:
            _p2p("recv", msg, (k - 1) % world, group)
            st = complex(msg[n].item())
            psi_in = msg[:n].clone()
            in_err = None if st.real == 0 else (int(st.real), int(st.imag), "relayed")
        if in_err is not None:
            err = in_err  # an earlier interval failed: that is the error
        rows = None
        if err is None:
            rows, e = compute.chain(u, b - a, psi_in)
            if e is not None:
                err = (e[0], a + e[1], e[2])
        if rows is not None:
            out.append((a, b, rows))
        psi_out = rows[-1] if rows is not None and err is None else psi_in
        if k + 1 < n_chunks:
            if world == 1:
                carry = (psi_out, err)
            else:
                msg[:n].copy_(psi_out)
                msg[n] = complex(err[0], err[1]) if err is not None else 0j
                _p2p("send", msg, (k + 1) % world, group)
    if err is not None:
        from .errors import NonFinite

        exc = NormDrift if err[0] == 9 else NonFinite if err[0] == 6 else RuntimeError
        what = "state norm drifted after" if err[0] == 9 else "propagator not unitary at"
        raise exc(f"{what} interval {err[1]}")
    return RelayResult(m, c, world, rank, out, p0)


class RelayEvolvePlan:
    """``evolve_relay`` set up once (operators, commutators, signals on the
    device) and run many times; ``run()`` returns the RelayResult."""

    def __init__(self, ch, grid, num_intervals: int, psi0, *, order: int = 1, check: bool = True,
                 chunk: int | None = None, group=None, compute=None):
        self.args = (ch, grid, num_intervals, psi0)
        self.kw = dict(order=order, check=check, chunk=chunk, group=group)
        self.compute = compute or DeviceRelayCompute()
        self.compute.setup(ch, order)

    def run(self) -> RelayResult:
        return evolve_relay(*self.args, compute=self.compute, **self.kw)


def sweep_shard(points: np.ndarray, world: int, rank: int) -> np.ndarray:
    """The sweep points (rows) owned by ``rank`` (no collective needed)."""
    a, b = shard_bounds(points.shape[0], world, rank)
    return points[a:b]


# -- NPAD parameter sweep (config 4): independent points, no exchange ------------------

class DeviceSweepCompute:
    """libqcheff on the rank's GPU: build the shard's operators on the device
    and run the batched greedy NPAD (npad.npad_sweep_transmon)."""

    def run(self, points, n_q, n_r, target, tol, max_iter):
        from . import npad

        res = npad.npad_sweep_transmon(points, n_q, n_r, target, tol=tol, max_iter=max_iter)
        t = _lib.torch()
        return (t.from_numpy(res.applied.astype(np.int64)), t.from_numpy(res.converged.astype(np.int32)),
                t.from_numpy(res.diagonals()), res)


@dataclass
class SweepShardResult:
    start: int          # first sweep point of this rank
    stop: int
    applied: object     # (stop - start,) int64 (host tensor)
    converged: object   # (stop - start,) int32
    diagonals: object   # (stop - start, N) float64: the final diagonal of each point
    batch: object       # the rank's BatchResult (device-resident final operators)
    world: int
    total: int

    def gather(self, group=None):
        """(applied, converged, diagonals) of ALL points on every rank (one
        all-gather per field; results only — the data path has no collective)."""
        import torch
        import torch.distributed as dist

        if self.world == 1:
            return self.applied.numpy(), self.converged.numpy().astype(bool), self.diagonals.numpy()
        per = -(-self.total // self.world)
        out = []
        for x in (self.applied, self.converged, self.diagonals):
            buf = torch.zeros((per,) + tuple(x.shape[1:]), dtype=x.dtype)
            buf[: x.shape[0]] = x
            dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
            buf = buf.to(dev)
            parts = [torch.empty_like(buf) for _ in range(self.world)]
            dist.all_gather(parts, buf, group=group)
            rows = [parts[r][: shard_bounds(self.total, self.world, r)[1] - shard_bounds(self.total, self.world, r)[0]]
                    for r in range(self.world)]
            out.append(torch.cat(rows).cpu().numpy())
        return out[0], out[1].astype(bool), out[2]


def sweep_sharded(points: np.ndarray, n_q: int, n_r: int, target=None, *, tol: float, max_iter: int | None = None,
                  group=None, compute=None) -> SweepShardResult:
    """Config-4 parameter sweep over the ranks of ``group`` (call on every
    rank): contiguous blocks of (omega_q, alpha, omega_r, g) points per rank,
    each rank's block built and solved on its own GPU (npad_sweep_transmon);
    no collective during the solve.  ``SweepShardResult.gather`` collects the
    per-point results."""
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    points = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 4)
    if points.shape[0] < world:
        raise ValueError("need at least one sweep point per rank")
    a, b = shard_bounds(points.shape[0], world, rank)
    compute = compute or DeviceSweepCompute()
    ap, cv, dg, batch = compute.run(points[a:b], n_q, n_r, target, tol, max_iter)
    return SweepShardResult(a, b, ap, cv, dg, batch, world, points.shape[0])
