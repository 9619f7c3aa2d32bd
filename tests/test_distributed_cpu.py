"""Multi-GPU host logic on CPU with gloo, world size 2 (no GPU needed):
LPT shard placement, exact M assembly by all-gather + column permutation, and the sharded ALS phase
sequence (ShardedALS + 3 allreduces per iteration) against the single-process
oracle, with the per-phase compute emulated in NumPy on each rank's slices."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import dpar2_oracle as orc
from paper_2203_12798_b200 import distributed as D_
from paper_2203_12798_b200 import synth


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def run_world(fn, world=2, *args):
    port = free_port()
    mp.spawn(_entry, args=(world, port, fn, args), nprocs=world, join=True)


def _entry(rank, world, port, fn, args):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fn(rank, world, *args)
    finally:
        dist.destroy_process_group()


def test_shard_slices_cover_and_balance():
    rng = np.random.default_rng(0)
    for world in (1, 2, 4, 8):
        rows = [int(r) for r in rng.integers(50, 6000, size=300)]
        shards, loads = D_.shard_slices(rows, world)
        assert sorted(k for s in shards for k in s) == list(range(300))
        assert all(s == sorted(s) for s in shards)
        assert max(loads) - min(loads) <= max(rows)
        assert [sum(rows[k] for k in s) for s in shards] == loads


def _assemble(rank, world):
    K, J, R = 13, 7, 3
    M = np.random.default_rng(5).standard_normal((J, K * R))
    shards, _ = D_.shard_slices([int(r) for r in np.random.default_rng(6).integers(1, 100, K)], world)
    ids = shards[rank]
    local = np.concatenate([M[:, k * R:(k + 1) * R] for k in ids], axis=1) if ids else np.zeros((J, 0))
    full = D_.assemble_m(torch.from_numpy(local), ids, K, R, shards=shards)
    assert full.numpy().tobytes() == M.tobytes()


def test_assemble_m_exact_gloo():
    run_world(_assemble)


class NumpyAlsOps:
    """CPU emulation of the dp2_als_phase phases on one rank's slices."""

    def __init__(self, comp, local_ids, h, v, w_local, normalize=True, tol=0.0):
        self.c, self.ids, self.R = comp, local_ids, comp.rank
        self.H, self.V, self.W = h.copy(), v.copy(), w_local.copy()
        self.normalize, self.tol, self.trace = normalize, tol, []
        self.stop = False

    def phase(self, ph, it=0, red_in=None):
        c, R = self.c, self.R
        if ph == 0:
            self.cc = orc.core_cols(c, self.V)
            return None
        if self.stop:
            return torch.zeros(2 * R * R if ph in (1, 3) else 1, dtype=torch.float64)
        if ph == 1:
            self.theta = {}
            g1, wtw = np.zeros((R, R)), np.zeros((R, R))
            for j, k in enumerate(self.ids):
                t = ((c.block(k) @ self.cc) * self.W[j]) @ self.H.T
                z, _, p = orc.truncated_svd(t, R)
                th = (p @ z.T) @ c.block(k)
                self.theta[k] = th
                g1 += (th @ self.cc) * self.W[j]
                wtw += np.outer(self.W[j], self.W[j])
            return torch.from_numpy(np.concatenate([g1.ravel(), wtw.ravel()]))
        if ph == 2:
            red = red_in.numpy()
            g1, wtw = red[:R * R].reshape(R, R), red[R * R:].reshape(R, R)
            h = g1 @ orc.pinv_small(wtw * (self.V.T @ self.V))
            self.nh = np.ones(R)
            if self.normalize:
                n = np.linalg.norm(h, axis=0)
                self.nh = np.where(n < 1e-300, 1.0, n)
                h = h / self.nh
            self.H = h
            return None
        if ph == 3:
            summed, wtw2 = np.zeros((R, R)), np.zeros((R, R))
            for j, k in enumerate(self.ids):
                w = self.W[j] * self.nh
                summed += w * (self.theta[k].T @ self.H)
                wtw2 += np.outer(w, w)
            return torch.from_numpy(np.concatenate([summed.ravel(), wtw2.ravel()]))
        if ph == 4:
            red = red_in.numpy()
            summed, wtw2 = red[:R * R].reshape(R, R), red[R * R:].reshape(R, R)
            v = (c.D @ (c.E[:, None] * summed)) @ orc.pinv_small(wtw2 * (self.H.T @ self.H))
            if self.normalize:
                n = np.linalg.norm(v, axis=0)
                v = v / np.where(n < 1e-300, 1.0, n)
            self.V = v
            self.cc = orc.core_cols(c, v)
            return None
        if ph == 5:
            pinv3 = orc.pinv_small((self.V.T @ self.V) * (self.H.T @ self.H))
            e = 0.0
            for j, k in enumerate(self.ids):
                g3 = np.einsum("ir,ir->r", self.H, self.theta[k] @ self.cc)
                self.W[j] = g3 @ pinv3
                buf = (self.theta[k] * c.E) @ c.D.T - (self.H * self.W[j]) @ self.V.T
                e += float(np.dot(buf.ravel(), buf.ravel()))
            return torch.tensor([e], dtype=torch.float64)
        if ph == 6:
            e = float(red_in[0])
            self.trace.append(e)
            if len(self.trace) > 1:
                prev = self.trace[-2]
                self.stop = prev == 0.0 or abs(prev - e) <= self.tol * prev
            return None


def _sharded_als(rank, world, tol):
    cfg = synth.scaled(synth.CONFIGS["c1"], num_slices=14, cols=30, rows=("uniform", 30, 80), rank=4)
    xs = synth.generate(cfg, 2)
    comp = orc.compress(xs, 4)
    shards, _ = D_.shard_slices([x.shape[0] for x in xs], world)
    ids = shards[rank]
    h, v, w = orc.initial_factors(cfg.cols, len(xs), 4)
    ops = NumpyAlsOps(comp, ids, h, v, w[ids], tol=tol)

    def allreduce(t):
        dist.all_reduce(t)
        return t

    D_.ShardedALS(ops, allreduce).run(12)
    ref = orc.fit_dpar2(xs, 4, 12, tol, 0, comp=comp)
    n = len(ref["objective"])
    assert ops.trace[:n] == pytest.approx(ref["objective"], rel=1e-10)
    assert np.abs(ops.H - ref["H"]).max() <= 1e-9 * np.abs(ref["H"]).max()
    assert np.abs(ops.V - ref["V"]).max() <= 1e-9 * np.abs(ref["V"]).max()
    assert np.abs(ops.W - ref["W"][ids]).max() <= 1e-9 * np.abs(ref["W"]).max()


@pytest.mark.parametrize("tol", [0.0, 1e-3])
def test_sharded_als_matches_oracle_gloo(tol):
    run_world(_sharded_als, 2, tol)


def _assemble_uneven(rank, world):
    K, J, R = 29, 5, 4
    rows = [int(r) for r in np.random.default_rng(8).integers(1, 5000, K)]
    M = np.random.default_rng(9).standard_normal((J, K * R))
    shards, _ = D_.shard_slices(rows, world)
    ids = shards[rank]
    local = np.concatenate([M[:, k * R:(k + 1) * R] for k in ids], axis=1)
    plan = D_.gather_plan(shards, R, "cpu")
    full = D_.assemble_m(torch.from_numpy(local), ids, K, R, shards=shards, plan=plan)
    assert full.numpy().tobytes() == M.tobytes()


@pytest.mark.parametrize("world", [3, 4])
def test_assemble_m_allgather_uneven_shards(world):
    """All-gather of padded per-rank blocks + column permutation == M, bit
    for bit, for shards of different sizes (LPT over heavy-tailed rows)."""
    run_world(_assemble_uneven, world)


def test_als_policy_cost_model():
    """The default ALS split (DistributedFit(als="auto")): replicated on one
    GPU and for c2 (K = 1000) at any world size; sharded for c5 (K = 20 000)
    from 4 GPUs; sharded whenever R > 16 (no persistent loop there)."""
    assert D_.als_policy(1000, 1, 512, 10) == "replicated"
    assert all(D_.als_policy(1000, w, 512, 10) == "replicated" for w in (2, 4, 8))
    assert D_.als_policy(20000, 8, 1000, 10) == "sharded"
    assert D_.als_policy(20000, 4, 1000, 10) == "sharded"
    assert D_.als_policy(20000, 2, 1000, 10) == "replicated"
    assert D_.als_policy(1000, 2, 512, 50) == "sharded"
