"""World-size-2 gloo test of the sharded solve orchestration (CPU only).

The product's ShardedRunner + TorchGather (paper_1707_02244_b200/dist.py) and
its shard-range logic (cl_shard_ranges, the same function the CUDA solver
uses) drive a CPU test backend that evaluates each phase with fp64 numpy for
the rank's own rows/outputs only.  After the all-gathers every rank must hold
exactly the single-process iterate (bitwise: every output entry is computed
by the same arithmetic whatever the sharding), for ISTA and cADMM.
"""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as orc


def cmv(row_hat, x, transpose=False):
    """C x (C[i, j] = row[(j - i) mod n]) or C^T x through numpy's FFT: deterministic and
    independent of any shard shape or thread count."""
    xh = np.fft.fft(x)
    return np.fft.ifft((row_hat if transpose else np.conj(row_hat)) * xh).real


class CpuIstaShard:
    """ShardBackend over fp64 numpy: phase 0 = residual rows, phase 1 = gradient + update.

    Each phase evaluates the full product (FFT, deterministic) and keeps only its
    own slice; everything else must arrive through the all-gather."""

    def __init__(self, p, rng, shard_rows, shard_out):
        s = orc.spectral_norm(p.row)
        self.ch = np.fft.fft(p.row / s)
        self.om, self.n = p.omega, p.n
        self.y = p.y / s
        self.tau, self.g = 0.9, 1e-4
        self.x = torch.zeros(p.n, dtype=torch.float64)
        self.r = torch.zeros(p.m, dtype=torch.float64)
        self.rows, self.outs = shard_rows, shard_out

    def phases(self):
        return (0, 1)

    def run_phase(self, ph):
        x = self.x.numpy()
        if ph == 0:
            a, b = self.rows
            self.r[a:b] = torch.from_numpy((self.y - cmv(self.ch, x)[self.om])[a:b])
        else:
            a, b = self.outs
            emb = np.zeros(self.n)
            emb[self.om] = self.r.numpy()
            d = cmv(self.ch, emb, transpose=True)[a:b]
            v = x[a:b] + self.tau * d
            self.x[a:b] = torch.from_numpy(np.sign(v) * np.maximum(np.abs(v) - self.g, 0.0))

    def phase_output(self, ph):
        return (self.r, *self.rows) if ph == 0 else (self.x, *self.outs)


class CpuCadmmShard:
    """Phases 0 beta, 1 x, 2 duals (reference parallel.hpp:178-228) on the rank's outputs."""

    def __init__(self, p, outs):
        s = orc.spectral_norm(p.row)
        c = p.row / s
        self.ch = np.fft.fft(c)
        self.bh = np.fft.fft(orc.regularized_gram_inverse(c, 0.1, 0.1))
        self.d = orc.mask_gram_inverse(p.omega, p.n, 0.1)
        self.pty = np.zeros(p.n)
        self.pty[p.omega] = p.y / s
        self.rho = self.sigma = 0.1
        self.thr = 1e-4 / 0.1
        z = lambda: torch.zeros(p.n, dtype=torch.float64)
        self.x, self.z, self.nu, self.mu, self.v, self.beta = z(), z(), z(), z(), z(), z()
        self.outs = outs

    def phases(self):
        return (0, 1, 2)

    def run_phase(self, ph):
        a, b = self.outs
        if ph == 0:
            ctv = cmv(self.ch, self.v.numpy(), transpose=True)[a:b]
            self.beta[a:b] = torch.from_numpy(self.rho * ctv + self.sigma * (self.z[a:b] - self.nu[a:b]).numpy())
        elif ph == 1:
            self.x[a:b] = torch.from_numpy(cmv(self.bh, self.beta.numpy())[a:b])
        else:
            cx = cmv(self.ch, self.x.numpy())[a:b]
            x, nu, mu = self.x[a:b].numpy(), self.nu[a:b].numpy(), self.mu[a:b].numpy()
            vn = self.d[a:b] * (self.rho * (cx - mu) + self.pty[a:b])
            v = x + nu
            zn = np.sign(v) * np.maximum(np.abs(v) - self.thr, 0.0)
            mun = mu + 1.0 * (vn - cx)
            self.z[a:b] = torch.from_numpy(zn)
            self.mu[a:b] = torch.from_numpy(mun)
            self.nu[a:b] = torch.from_numpy(nu + 1.0 * (x - zn))
            self.v[a:b] = torch.from_numpy(vn + mun)

    def phase_output(self, ph):
        full = (self.beta, self.x, self.v)[ph]
        return (full, *self.outs)


def shard_ranges(kind, p, rank, world):
    from paper_1707_02244_b200._native import lib
    from paper_1707_02244_b200.api import _check
    om = np.ascontiguousarray(p.omega, dtype=np.int64)
    v = [C.c_int64() for _ in range(4)]
    _check(lib.cl_shard_ranges(kind, p.n, p.m, om.ctypes.data_as(C.POINTER(C.c_int64)), rank, world,
                               *[C.byref(t) for t in v]))
    return (v[2].value, v[3].value), (v[0].value, v[1].value)


def _worker(rank, world, port, n, m, k, iters, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1707_02244_b200.dist import ShardedRunner, TorchGather
    p = orc.make_problem(n, m, k, 7)
    rows, outs = shard_ranges(0, p, rank, world)
    ista = CpuIstaShard(p, None, rows, outs)
    ShardedRunner(ista, TorchGather()).step(iters)
    _, outs_c = shard_ranges(1, p, rank, world)
    admm = CpuCadmmShard(p, outs_c)
    ShardedRunner(admm, TorchGather()).step(iters)
    out[rank] = (ista.x.numpy().copy(), admm.z.numpy().copy(), admm.v.numpy().copy(), admm.x.numpy().copy(),
                 rows, outs, outs_c)
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_iterations_match_single_process(world):
    n, m, k, iters = 20000, 5000, 40, 6  # 5 gradient / 3 dense tiles: ragged shards
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), n, m, k, iters, out), nprocs=world, join=True,
                       start_method="spawn")
    p = orc.make_problem(n, m, k, 7)
    single = CpuIstaShard(p, None, (0, m), (0, n))
    for _ in range(iters):
        single.run_phase(0)
        single.run_phase(1)
    single_c = CpuCadmmShard(p, (0, n))
    for _ in range(iters):
        for ph in (0, 1, 2):
            single_c.run_phase(ph)
    rows_cover, outs_cover = [], []
    for r in range(world):
        xi, zc, vc, xc, rows, outs, outs_c = out[r]
        assert np.array_equal(xi, single.x.numpy()), f"rank {r} ISTA iterate differs"
        a, b = outs_c  # z, mu, nu stay slice-local; v and x are all-gathered
        assert np.array_equal(zc[a:b], single_c.z.numpy()[a:b]), f"rank {r} cADMM iterate differs"
        assert np.array_equal(vc, single_c.v.numpy()) and np.array_equal(xc, single_c.x.numpy())
        rows_cover.append(rows)
        outs_cover.append(outs)
    # shards tile [0, m) and [0, n) contiguously
    assert rows_cover[0][0] == 0 and rows_cover[-1][1] == m
    assert outs_cover[0][0] == 0 and outs_cover[-1][1] == n
    for a, b in zip(rows_cover, rows_cover[1:]):
        assert a[1] == b[0]
    for a, b in zip(outs_cover, outs_cover[1:]):
        assert a[1] == b[0]
    assert np.count_nonzero(single.x.numpy()) > 0


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_tensor_core_shard_ranges(world):
    """Shard ranges when the direct products run on the tensor cores (power-of-two n >= 2^17 for
    ISTA, >= 2^15 for cADMM; host logic only): outputs split by 128 x 256-output tiles, and an ISTA
    rank's residual rows are exactly Omega within its outputs."""
    for lg, kind in ((17, 0), (20, 0), (16, 1), (20, 1)):
        n = 1 << lg
        m = n // 4
        rng = np.random.default_rng(lg)
        omega = np.sort(rng.choice(n, m, replace=False)).astype(np.int64)

        class P:
            pass
        p = P()
        p.n, p.m, p.omega = n, m, omega
        prev_o, prev_r = 0, 0
        for r in range(world):
            rows, outs = shard_ranges(kind, p, r, world)
            assert outs[0] == prev_o and outs[0] % (128 * 256) == 0
            prev_o = outs[1]
            if kind == 0:
                assert rows[0] == prev_r
                assert rows == (np.searchsorted(omega, outs[0]), np.searchsorted(omega, outs[1]))
                prev_r = rows[1]
        assert prev_o == n
        if kind == 0:
            assert prev_r == m


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_tensor_core_shards_are_whole_cta_pairs(world):
    """At the bench sizes (n = 2^20, 2^24) every rank's tile range of the tcgen05 plan starts and ends on an even
    tile, so every rank runs the CTA-pair kernel (cta_group::2: two adjacent 128 x 256-output tiles per pair);
    host logic only (cl_shard_ranges)."""
    tile = 128 * 256
    for lg in (20, 24):
        n = 1 << lg

        class P:
            pass
        p = P()
        p.n, p.m, p.omega = n, n // 4, np.arange(0, n, 4, dtype=np.int64)
        for r in range(world):
            _, outs = shard_ranges(1, p, r, world)
            assert outs[0] % (2 * tile) == 0 and outs[1] % (2 * tile) == 0, (lg, r, outs)
