"""Generate tests/golden/ fixtures from the REAL reference and pin the oracle.

Run in the build container (where /root/reference exists):

    python oracle/make_golden.py

It imports the reference package ``dpar2`` from /root/reference/pkg/src,
runs it on small seeded inputs, writes the outputs as fixtures, and checks
that ``oracle/dpar2_oracle.py`` reproduces every one of them (the oracle is
pinned against the reference here; the fixtures pin it on the GPU box where
the reference is absent).  Test infrastructure only.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
from pathlib import Path

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
REF = Path("/root/reference/pkg/src")
OUT = ROOT / "tests" / "golden"
sys.path.insert(0, str(REF))
sys.path.insert(0, str(ROOT))

import dpar2  # noqa: E402  (the reference)
from dpar2.compress import compress as ref_compress  # noqa: E402
from dpar2.linalg import RsvdParams, derived_seed as ref_derived_seed, randomized_svd  # noqa: E402
from dpar2 import solver as ref_solver  # noqa: E402
from dpar2.factors import initial_factors as ref_init  # noqa: E402

from oracle import dpar2_oracle as orc  # noqa: E402
from paper_2203_12798_b200 import synth  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


def relerr(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


# ---------------------------------------------------------------- inputs
def tiny_instances(seed, count):
    """Reference-test-style random instances (R 1-4, J 4-16, I_k in [R, 20])."""
    rng = np.random.Generator(np.random.PCG64(seed))
    out = []
    for _ in range(count):
        rank = int(rng.integers(1, 5))
        cols = int(rng.integers(max(rank, 4), 17))
        num = int(rng.integers(1, 13))
        counts = rng.integers(rank, 21, size=num)
        out.append(([rng.random((int(c), cols)) for c in counts], rank))
    return out


def planted(K, J, lo, hi, R, noise, seed, dtype="f64"):
    cfg = synth.SynthConfig("g", K, J, ("uniform", lo, hi), rank=R, noise=noise, dtype=dtype)
    xs = synth.generate(cfg, seed)
    return [x.astype(np.float64) for x in xs]


def fit_cases():
    cases = {}
    for i, (xs, r) in enumerate(tiny_instances(101, 6)):
        cases[f"tiny{i}"] = dict(xs=xs, rank=r, max_iters=8, tol=0.0, seed=0, normalize=True)
    cases["planted"] = dict(xs=planted(12, 40, 30, 90, 5, 0.1, 3), rank=5, max_iters=32,
                            tol=0.0, seed=0, normalize=True)
    cases["planted_tol"] = dict(xs=planted(10, 30, 20, 60, 4, 0.2, 5), rank=4, max_iters=50,
                                tol=1e-6, seed=7, normalize=True)
    cases["planted_nonorm"] = dict(xs=planted(8, 24, 20, 50, 3, 0.1, 6), rank=3, max_iters=10,
                                   tol=0.0, seed=0, normalize=False)
    cases["f32vals"] = dict(xs=planted(16, 64, 40, 120, 6, 0.1, 8, dtype="f32"), rank=6,
                            max_iters=32, tol=0.0, seed=0, normalize=True)
    cases["wide"] = dict(xs=planted(6, 300, 20, 40, 4, 0.1, 9), rank=4, max_iters=16,
                         tol=0.0, seed=3, normalize=True)
    return cases


def run_ref_fit(c):
    t = dpar2.IrregularTensor(c["xs"])
    opts = dpar2.SolverOptions(max_iters=c["max_iters"], tol=c["tol"], seed=c["seed"],
                               threads=1, normalize=c["normalize"])
    f, tr = dpar2.fit_dpar2(t, c["rank"], opts)
    comp = ref_compress(t, c["rank"], rsvd=RsvdParams(rank=c["rank"], seed=c["seed"]), threads=1)
    fit = dpar2.fitness(t, f, threads=1)
    return f, tr, comp, fit


def save_fit_case(name, c):
    f, tr, comp, fit = run_ref_fit(c)
    xs = c["xs"]
    rows = np.array([x.shape[0] for x in xs], dtype=np.int64)
    data = dict(
        X=np.concatenate([x.ravel() for x in xs]), rows=rows, J=xs[0].shape[1],
        rank=c["rank"], max_iters=c["max_iters"], tol=c["tol"], seed=c["seed"],
        normalize=c["normalize"],
        H=f.H, V=f.V, W=f.W, Q=np.concatenate(f.Q), objective=np.array(tr.objective),
        converged=tr.converged, float_count=tr.compressed_float_count, fitness=fit,
        A=np.concatenate(comp.slice_bases), D=comp.col_basis, E=comp.weights, F=comp.cores,
    )
    np.savez_compressed(OUT / f"fit_{name}.npz", **data)
    # pin the oracle against the reference on this case
    o = orc.fit_dpar2(xs, c["rank"], c["max_iters"], c["tol"], c["seed"], c["normalize"])
    ofit = orc.fitness(xs, o["H"], o["V"], o["W"], o["Q"])
    errs = dict(H=relerr(o["H"], f.H), V=relerr(o["V"], f.V), W=relerr(o["W"], f.W),
                Q=relerr(np.concatenate(o["Q"]), np.concatenate(f.Q)),
                obj=relerr(o["objective"], tr.objective), fit=abs(ofit - fit),
                A=relerr(np.concatenate(o["comp"].bases), np.concatenate(comp.slice_bases)))
    assert o["converged"] == tr.converged and len(o["objective"]) == len(tr.objective), name
    assert max(errs.values()) <= 1e-12, (name, errs)
    return errs


def save_c1():
    """c1 (K=100, J=100, I_k~U{200..1000}, R=10, 32 iterations): inputs are
    regenerated from the seed; the fixture holds the reference's outputs."""
    cfg = synth.CONFIGS["c1"]
    xs = synth.generate(cfg, 0)
    t = dpar2.IrregularTensor(xs)
    f, tr = dpar2.fit_dpar2(t, 10, dpar2.SolverOptions(max_iters=32, tol=0.0, seed=0, threads=1))
    fit = dpar2.fitness(t, f, threads=1)
    comp = ref_compress(t, 10, rsvd=RsvdParams(rank=10, seed=0), threads=1)
    q = np.concatenate(f.Q)
    np.savez_compressed(
        OUT / "c1.npz", rows=np.array([x.shape[0] for x in xs]), H=f.H, V=f.V, W=f.W,
        objective=np.array(tr.objective), fitness=fit, Q_head=np.concatenate(f.Q[:4]),
        Q_colsum=q.sum(axis=0), Q_abssum=np.abs(q).sum(axis=0), D=comp.col_basis,
        E=comp.weights, F=comp.cores, A_head=np.concatenate(comp.slice_bases[:4]),
        x_sum=float(sum(float(x.sum()) for x in xs)),
        x_sq=float(sum(float(np.dot(x.ravel(), x.ravel())) for x in xs)))
    return fit


def save_kernels():
    """ALS kernels on hand-built compressed tensors (reference test style)."""
    out = {}
    rng = np.random.Generator(np.random.PCG64(4))
    for tag, (rank, cols, num, rows) in dict(a=(3, 9, 5, 8), b=(5, 20, 7, 12), c=(10, 40, 9, 30)).items():
        def ortho(m, n):
            q, _ = np.linalg.qr(rng.standard_normal((m, max(m, n))))
            return np.ascontiguousarray(q[:, :n])
        bases = [ortho(rows, rank) for _ in range(num)]
        d = ortho(cols, rank)
        e = np.sort(rng.uniform(1.0, 5.0, rank))[::-1].copy()
        f = np.concatenate([ortho(rank, rank) for _ in range(num)])
        comp = dpar2.CompressedTensor(rank=rank, slice_bases=bases, col_basis=d, weights=e, cores=f)
        h = rng.standard_normal((rank, rank))
        v = rng.standard_normal((cols, rank))
        w = rng.standard_normal((num, rank))
        rots = ref_solver.update_rotations(comp, h, v, w, threads=1)
        polar = np.stack([r.Z @ r.P.T for r in rots])
        g1 = ref_solver.mttkrp_mode1(comp, rots, w, v, threads=1)
        g2 = ref_solver.mttkrp_mode2(comp, rots, w, h, threads=1)
        g3 = ref_solver.mttkrp_mode3(comp, rots, v, h, threads=1)
        met = ref_solver.convergence_metric(comp, rots, h, v, w, threads=1)
        sweep_n = ref_solver.update_factors(comp, rots, h, v, w, normalize=True, threads=1)
        sweep_p = ref_solver.update_factors(comp, rots, h, v, w, normalize=False, threads=1)
        np.savez_compressed(OUT / f"kernels_{tag}.npz", rank=rank, A=np.concatenate(bases), rows=rows,
                            D=d, E=e, F=f, H=h, V=v, W=w, polar=polar, g1=g1, g2=g2, g3=g3, metric=met,
                            Hn=sweep_n[0], Vn=sweep_n[1], Wn=sweep_n[2],
                            Hp=sweep_p[0], Vp=sweep_p[1], Wp=sweep_p[2])
        # oracle pin
        oc = orc.Compressed(rank, bases, d, e, f)
        orots = orc.update_rotations(oc, h, v, w)
        assert relerr(np.stack([z @ p.T for z, p, _ in orots]), polar) <= 1e-12
        assert relerr(orc.mttkrp_mode1(oc, orots, w, v), g1) <= 1e-12
        assert relerr(orc.mttkrp_mode2(oc, orots, w, h), g2) <= 1e-12
        assert relerr(orc.mttkrp_mode3(oc, orots, v, h), g3) <= 1e-12
        assert abs(orc.convergence_metric(oc, orots, h, v, w) - met) <= 1e-12 * met
        out[tag] = met
    return out


def save_stage1():
    """Per-slice rSVD triples and the stage-2 input M for a small tensor,
    including slices narrower than R + 10 (per-slice sketch width) and a
    config-4 style oversampling = R case."""
    xs = planted(9, 36, 12, 70, 4, 0.1, 11)
    xs[3] = xs[3][:9]            # I_k < R + 10 -> s_k = 9 for this slice
    trips = [randomized_svd(x, RsvdParams(rank=4, seed=ref_derived_seed(0, k))) for k, x in enumerate(xs)]
    comp_over = ref_compress(dpar2.IrregularTensor(xs), 4, rsvd=RsvdParams(rank=4, oversampling=4, seed=2),
                             threads=1)
    np.savez_compressed(OUT / "stage1.npz", X=np.concatenate([x.ravel() for x in xs]),
                        rows=np.array([x.shape[0] for x in xs]), J=36, rank=4,
                        A=np.concatenate([t.U for t in trips]), S=np.stack([t.S for t in trips]),
                        V=np.stack([t.V for t in trips]),
                        over_A=np.concatenate(comp_over.slice_bases), over_D=comp_over.col_basis,
                        over_E=comp_over.weights, over_F=comp_over.cores)
    oc = orc.compress(xs, 4, seed=0, keep_stage1=True)
    assert relerr(np.concatenate(oc.bases), np.concatenate([t.U for t in trips])) <= 1e-12
    oo = orc.compress(xs, 4, seed=2, oversampling=4)
    assert relerr(oo.F, comp_over.cores) <= 1e-12 and relerr(oo.D, comp_over.col_basis) <= 1e-12


def save_scalars():
    rng = np.random.Generator(np.random.PCG64(17))
    parts = []
    for _ in range(300):
        k = int(rng.integers(1, 60))
        counts = [int(c) for c in rng.integers(1, 5000, size=k)]
        if rng.random() < 0.3:
            counts = [int(c) for c in rng.integers(1, 4, size=k)]  # many ties
        t = int(rng.integers(1, 10))
        p = dpar2.greedy_partition(counts, t)
        osets, oloads = orc.greedy_partition(counts, t)
        assert osets == p.sets and oloads == p.loads
        parts.append(dict(counts=counts, workers=t, sets=p.sets, loads=p.loads))
    p = dpar2.greedy_partition([5, 4, 3, 3, 2], 2)
    parts.append(dict(counts=[5, 4, 3, 3, 2], workers=2, sets=p.sets, loads=p.loads))
    seeds = []
    for s in (0, 1, 12345, 2**63 + 5, 2**64 - 1, -1):
        for k in (0, 1, 2, 99, 1000, 2**32 + 7):
            v = ref_derived_seed(s, k)
            assert v == orc.derived_seed(s, k)
            seeds.append(dict(seed=s, index=k, value=str(v)))
    omegas = []
    for k in range(6):
        sd = ref_derived_seed(0, k)
        om = np.random.Generator(np.random.PCG64(sd)).standard_normal((100, 20))
        omegas.append(dict(seed=str(sd), n=100, s=20, sha256=sha(om), head=om.ravel()[:8].tolist()))
    (OUT / "scalars.json").write_text(json.dumps(dict(partitions=parts, derived_seeds=seeds,
                                                      omegas=omegas), indent=0))


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    save_scalars()
    save_stage1()
    kern = save_kernels()
    worst = {}
    for name, c in fit_cases().items():
        worst[name] = max(save_fit_case(name, c).values())
    fit = save_c1()
    manifest = dict(numpy=np.__version__, openblas_threads=os.environ.get("OPENBLAS_NUM_THREADS"),
                    reference="/root/reference/pkg (dpar2 0.1.0)", oracle_vs_reference_max_rel=worst,
                    c1_fitness=fit, kernel_metrics=kern)
    (OUT / "MANIFEST.json").write_text(json.dumps(manifest, indent=1))
    print(json.dumps(manifest, indent=1))


if __name__ == "__main__":
    main()
