"""Host logic of the native library: the LPT partition (bit-exact with the
reference), the piece planner, and the exported C ABI."""
import ctypes as C
import json
import re

import numpy as np
import pytest

from paper_2203_12798_b200 import _lib, greedy_partition


def test_library_exports_every_header_symbol():
    header = (_lib.lib_path().parents[1] / "include" / "dpar2_b200.h").read_text()
    declared = set(re.findall(r"\b(dp2_[a-z0-9_]+)\s*\(", header))
    handle = _lib.lib()
    missing = [name for name in sorted(declared) if not hasattr(handle, name)]
    assert not missing, missing
    assert declared == set(_lib.EXPORTS)
    assert handle.dp2_abi_version() == 1


def test_partition_matches_reference_golden(golden):
    data = json.loads((golden / "scalars.json").read_text())
    for p in data["partitions"]:
        plan = greedy_partition(p["counts"], p["workers"])
        assert plan.sets == p["sets"] and plan.loads == p["loads"]


def test_partition_hand_traced_and_errors():
    plan = greedy_partition([5, 4, 3, 3, 2], 2)
    assert plan.loads == [8, 9] and plan.sets == [[0, 3], [1, 2, 4]]
    assert greedy_partition([7], 3).sets == [[0], [], []]
    for bad in (([], 1), ([1, 2], 0), ([1, 0], 2)):
        with pytest.raises(ValueError):
            greedy_partition(*bad)


def test_partition_spread_bound_random():
    rng = np.random.default_rng(3)
    for _ in range(1000):
        counts = rng.integers(1, 10000, size=int(rng.integers(1, 80)))
        t = int(rng.integers(1, 9))
        plan = greedy_partition(counts, t)
        assert sorted(k for s in plan.sets for k in s) == list(range(len(counts)))
        assert max(plan.loads) - min(plan.loads) <= counts.max()


def plan(rows, nseg):
    lib = _lib.lib()
    off = np.zeros(len(rows) + 1, np.int64)
    np.cumsum(rows, out=off[1:])
    K = len(rows)
    cap = lib.dp2_piece_capacity(K, nseg)
    ps, pr0, prs = np.empty(cap, np.int32), np.empty(cap, np.int64), np.empty(cap, np.int32)
    sb, sl = np.empty(nseg + 1, np.int32), np.empty(K + 1, np.int32)
    n = C.c_int64()
    P = C.POINTER
    st = lib.dp2_plan_pieces(off.ctypes.data_as(P(C.c_int64)), K, nseg, ps.ctypes.data_as(P(C.c_int32)),
                             pr0.ctypes.data_as(P(C.c_int64)), prs.ctypes.data_as(P(C.c_int32)),
                             sb.ctypes.data_as(P(C.c_int32)), sl.ctypes.data_as(P(C.c_int32)), C.byref(n))
    assert st == 0
    n = n.value
    return off, ps[:n], pr0[:n], prs[:n], sb, sl


@pytest.mark.parametrize("seed", range(20))
def test_piece_plan_invariants(seed):
    rng = np.random.default_rng(seed)
    rows = rng.integers(1, 5000, size=int(rng.integers(1, 300)))
    nseg = int(rng.integers(1, 400))
    off, ps, pr0, prs, sb, sl = plan(rows, nseg)
    N = off[-1]
    # pieces tile [0, N) in order, each inside one slice
    assert pr0[0] == 0 and (pr0[1:] == pr0[:-1] + prs[:-1]).all() and pr0[-1] + prs[-1] == N
    assert (prs > 0).all()
    assert (off[ps] <= pr0).all() and (pr0 + prs <= off[ps + 1]).all()
    # segments: equal split of rows, contiguous piece ranges
    for g in range(nseg):
        a, b = N * g // nseg, N * (g + 1) // nseg
        seg = range(sb[g], sb[g + 1])
        assert sum(int(prs[p]) for p in seg) == b - a
    # slice -> piece index ranges
    for k in range(len(rows)):
        assert all(ps[p] == k for p in range(sl[k], sl[k + 1]))
        assert sum(int(prs[p]) for p in range(sl[k], sl[k + 1])) == rows[k]


def test_omega_tail_replay_matches_python_log1p():
    """dp2_omega_replay (host C, libm log1p) == the Python restatement of the
    reference's layer-0 tail branch (math.log1p is libm's log1p too)."""
    import ctypes as C
    import math

    from paper_2203_12798_b200 import _lib
    from paper_2203_12798_b200.rng import _REC, _ZIG_INV_R, _ZIG_R

    rng = np.random.default_rng(11)
    n = 4000
    r = np.zeros(n, dtype=_REC)
    r["slice"] = rng.integers(0, 50, n)
    r["index"] = rng.integers(0, 10000, n)
    r["negative"] = rng.integers(0, 2, n)
    r["u"] = rng.random((n, 8))
    want_v, want_ok = np.zeros(n), np.zeros(n, dtype=np.int32)
    for i in range(n):
        # the acceptance sequence decides the attempt count the device saw
        a_acc = None
        for a in range(4):
            xx = -_ZIG_INV_R * math.log1p(-r["u"][i, 2 * a])
            yy = -math.log1p(-r["u"][i, 2 * a + 1])
            if yy + yy > xx * xx:
                a_acc = a
                break
        r["attempts"][i] = (a_acc + 1) if a_acc is not None else 4
        if i % 7 == 0:  # a device that disagreed: claims a different attempt
            r["attempts"][i] = 1 + (r["attempts"][i] % 4)
        ok = 1
        v = 0.0
        for a in range(r["attempts"][i]):
            xx = -_ZIG_INV_R * math.log1p(-r["u"][i, 2 * a])
            yy = -math.log1p(-r["u"][i, 2 * a + 1])
            acc = (yy + yy) > (xx * xx)
            last = a + 1 == r["attempts"][i]
            if acc != last:
                ok = 0
            if last:
                v = -(_ZIG_R + xx) if r["negative"][i] else _ZIG_R + xx
        want_v[i], want_ok[i] = v, ok
    vals = np.empty(n)
    okv = np.empty(n, dtype=np.int32)
    assert _lib.lib().dp2_omega_replay(C.c_void_p(r.ctypes.data), n, vals.ctypes.data_as(C.POINTER(C.c_double)),
                                       okv.ctypes.data_as(C.POINTER(C.c_int32))) == 0
    assert np.array_equal(okv, want_ok)
    good = want_ok == 1  # values of rejected records are never used
    assert np.array_equal(vals[good].view(np.uint64), want_v[good].view(np.uint64))
    assert 0 < want_ok.sum() < n
