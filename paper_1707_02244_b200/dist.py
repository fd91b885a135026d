"""Sharded solves: one process per GPU, row/output-range sharding.

Shard g of G owns a contiguous, tile-aligned range of every product's outputs
(and, for ISTA, the residual rows of its position splits).  Between phases
each rank publishes its slice and all-gathers the others' slices -- the only
cross-GPU traffic, n (or m) floats per phase.  No reduction crosses ranks, so
the iterate is bitwise identical for every G.

The collective is pluggable: ``TorchGather`` uses torch.distributed (NCCL
over NVLink on GPUs, gloo on CPU tensors in the tests); the phase logic in
``ShardedRunner`` is backend-agnostic and is exercised on CPU by
tests/test_dist_gloo.py with a CPU backend defined in the tests.
"""
from __future__ import annotations

import ctypes as C
from typing import Protocol, Sequence

from ._native import lib
from .api import _check


class ShardBackend(Protocol):
    """What ShardedRunner needs from a solver shard."""

    def phases(self) -> Sequence[int]: ...

    def run_phase(self, phase: int) -> None: ...

    def phase_output(self, phase: int):
        """-> (full-length tensor view of the produced vector, begin, end)."""
        ...


class TorchGather:
    """All-gather of unequal contiguous slices via torch.distributed.

    Each rank copies its slice into a padded staging row, one
    all_gather_into_tensor exchanges the rows, and the slices are copied back
    into the full vector at their offsets.  Offsets are exchanged once per
    phase (they are static) and cached.
    """

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self._ranges = {}
        self._stage = {}

    def ranges(self, key, begin, end, device):
        import torch
        if key not in self._ranges:
            mine = torch.tensor([begin, end], dtype=torch.int64, device=device)
            allr = torch.zeros(2 * self.world, dtype=torch.int64, device=device)
            self.dist.all_gather_into_tensor(allr, mine, group=self.group)
            rr = allr.view(self.world, 2).cpu().tolist()
            self._ranges[key] = [(int(a), int(b)) for a, b in rr]
        return self._ranges[key]

    def __call__(self, key, full, begin, end):
        import torch
        rr = self.ranges(key, begin, end, full.device)
        width = max(b - a for a, b in rr)
        if width == 0:
            return
        st = self._stage.get((key, full.device))
        if st is None or st.numel() != width * (self.world + 1):
            st = torch.zeros(width * (self.world + 1), dtype=full.dtype, device=full.device)
            self._stage[(key, full.device)] = st
        mine = st[self.world * width:(self.world + 1) * width]
        mine[: end - begin].copy_(full[begin:end])
        allrows = st[: self.world * width]
        self.dist.all_gather_into_tensor(allrows, mine, group=self.group)
        rows = allrows.view(self.world, width)
        for g, (a, b) in enumerate(rr):
            if g != self.rank and b > a:
                full[a:b].copy_(rows[g, : b - a])


class ShardedRunner:
    """Drives one iteration as phase -> all-gather -> phase ...."""

    def __init__(self, backend: ShardBackend, gather):
        self.b = backend
        self.gather = gather

    def step(self, iters: int = 1):
        for _ in range(iters):
            for ph in self.b.phases():
                self.b.run_phase(ph)
                full, begin, end = self.b.phase_output(ph)
                self.gather(ph, full, begin, end)


class _CudaArray:
    """__cuda_array_interface__ view of a library-owned device buffer."""

    def __init__(self, ptr: int, length: int):
        self.__cuda_array_interface__ = {"shape": (length,), "typestr": "<f4", "data": (ptr, False),
                                         "version": 3, "strides": None}


class CudaShard:
    """ShardBackend over a cl_solver handle (ISTA or cADMM) on one GPU."""

    def __init__(self, state, rank: int, world: int):
        import torch
        self.state = state
        self.kind = state.KIND
        _check(lib.cl_solver_shard(state.handle, rank, world))
        sp = C.c_void_p()
        _check(lib.cl_solver_stream(state.handle, C.byref(sp)))
        self.stream = torch.cuda.ExternalStream(sp.value)
        self._views = {}

    def phases(self):
        return (0, 1) if self.kind == 0 else (0, 1, 2)

    def run_phase(self, phase: int):
        _check(lib.cl_solver_run_phase(self.state.handle, phase))

    def phase_output(self, phase: int):
        import torch
        ptr = C.c_void_p()
        b, e, tot = C.c_int64(), C.c_int64(), C.c_int64()
        _check(lib.cl_solver_phase_output(self.state.handle, phase, C.byref(ptr), C.byref(b), C.byref(e),
                                          C.byref(tot)))
        key = (ptr.value, tot.value)
        if key not in self._views:
            self._views[key] = torch.as_tensor(_CudaArray(ptr.value, tot.value), device="cuda")
        return self._views[key], b.value, e.value


class NativeComm:
    """A library-owned NCCL communicator (cl_comm_*): the exchange runs inside cl_solver_step /
    cl_solver_run once a solver is attached -- no Python, no staging copies."""

    def __init__(self, uid: bytes, world: int, rank: int, device: int):
        if len(uid) != 128:
            raise ValueError("NativeComm: the NCCL unique id is 128 bytes")
        self.rank, self.world, self.device = rank, world, device
        h = C.c_void_p()
        _check(lib.cl_comm_init_rank(uid, world, rank, device, C.byref(h)))
        self._h = h

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(lib.cl_comm_unique_id(buf))
        return buf.raw

    @classmethod
    def from_torch(cls, device: int, group=None):
        """Every rank of a torch.distributed group: rank 0's id is broadcast over the group."""
        import torch.distributed as dist
        obj = [cls.unique_id() if dist.get_rank(group) == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        return cls(obj[0], dist.get_world_size(group), dist.get_rank(group), device)

    def attach(self, state):
        """Shards `state` as (rank, world); its steps and run loop then exchange through this communicator."""
        _check(lib.cl_solver_attach_comm(state.handle, self._h))
        state._comm = self  # the communicator outlives the solver's use of it

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.cl_comm_destroy(h)
            self._h = None


PEER_BLOB_BYTES = 512  # CL_PEER_BLOB_BYTES


class IpcPeers:
    """One process per GPU with no NCCL: CUDA IPC peer stores (cl_solver_peer_export / _attach).  Each rank
    exports its solver's exchange vectors, the blobs travel over any channel (``exchange``: a callable that
    maps this rank's blob to the list of every rank's blob, e.g. ``torch.distributed.all_gather_object``),
    and from then on the solver's steps and run loop store each phase's slice straight into every rank's
    copy and order the phases through device flags.  Destroying the attached solvers is collective."""

    @staticmethod
    def export(state, rank: int, world: int) -> bytes:
        buf = C.create_string_buffer(PEER_BLOB_BYTES)
        _check(lib.cl_solver_peer_export(state.handle, rank, world, buf))
        return buf.raw

    @staticmethod
    def attach(state, blobs) -> None:
        if any(len(b) != PEER_BLOB_BYTES for b in blobs):
            raise ValueError("IpcPeers.attach: every blob is PEER_BLOB_BYTES long")
        _check(lib.cl_solver_peer_attach(state.handle, b"".join(blobs)))

    @classmethod
    def connect(cls, state, rank: int, world: int, exchange) -> None:
        cls.attach(state, exchange(cls.export(state, rank, world)))

    @classmethod
    def from_torch(cls, state, group=None) -> None:
        """Every rank of a torch.distributed group (any backend): the blobs are all-gathered as objects."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)

        def exchange(blob):
            out = [None] * world
            dist.all_gather_object(out, blob, group=group)
            return out
        cls.connect(state, rank, world, exchange)


class TorchIpc:
    """The ``comm=`` of ista_run / cadmm_run for the CUDA IPC peer-store transport over a torch.distributed
    group: attach(state) exports, all-gathers and attaches every rank's blob (IpcPeers.from_torch)."""

    def __init__(self, group=None):
        self.group = group

    def attach(self, state) -> None:
        IpcPeers.from_torch(state, self.group)


def sharded_step(shard: CudaShard, gather: TorchGather, iters: int = 1):
    """Advance a CudaShard `iters` iterations; collectives run on the solver's stream."""
    import torch
    runner = ShardedRunner(shard, gather)
    with torch.cuda.stream(shard.stream):
        runner.step(iters)
