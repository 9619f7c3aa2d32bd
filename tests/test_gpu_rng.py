"""Device sketch matrices are byte-identical to the reference's NumPy draws
(P/linalg.py:122-123, derived seeds P/linalg.py:187-194)."""
import hashlib
import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_golden_omega_digests(golden):
    import torch
    from paper_2203_12798_b200.rng import omega_device
    data = json.loads((golden / "scalars.json").read_text())
    # the golden draws are PCG64(derived_seed(0, k)) for k = 0..5 with n=100, s=20
    out = omega_device(0, 100, [20] * 6, 24, torch.device("cuda")).cpu().numpy()
    for k, o in enumerate(data["omegas"]):
        om = np.ascontiguousarray(out[k, :, :20])
        assert hashlib.sha256(om.astype("<f8").tobytes()).hexdigest() == o["sha256"], k


@pytest.mark.parametrize("seed,K,J,smax", [(0, 1000, 512, 20), (7, 300, 100, 20), ((1 << 64) - 1, 64, 37, 13),
                                           (2**63 + 5, 200, 256, 32), (12345, 50, 1000, 20), (99, 2, 4000, 16)])
def test_device_omega_matches_numpy_bytes(seed, K, J, smax):
    import torch
    from paper_2203_12798_b200.linalg import padded_width
    from paper_2203_12798_b200.rng import omega_device, omega_host
    rng = np.random.default_rng(seed % 1000)
    widths = [int(w) for w in rng.integers(max(1, smax - 6), smax + 1, size=K)]
    sp = padded_width(max(widths))
    stats = {}
    dev = omega_device(seed, J, widths, sp, torch.device("cuda"), stats=stats).cpu().numpy()
    host = omega_host(seed, J, widths, sp).numpy()
    assert dev.tobytes() == host.tobytes(), stats
    if K * J * smax > 5e6:
        assert stats["omega_tail_events"] > 100  # the tail replay path was exercised


def test_device_omega_slice_ids():
    import torch
    from paper_2203_12798_b200.rng import omega_device, omega_host
    ids = [5, 17, 0, 999]
    dev = omega_device(3, 40, [12] * 4, 16, torch.device("cuda"), slice_ids=ids).cpu().numpy()
    host = omega_host(3, 40, [12] * 4, 16, slice_ids=ids).numpy()
    assert dev.tobytes() == host.tobytes()


@pytest.mark.parametrize("seed,rows,width", [(0, 10000, 20), (2**64 - 3, 333, 7), (77, 50000, 40), (5, 1, 1),
                                             (123456789, 4096, 13)])
def test_device_stage2_omega_matches_numpy_bytes(seed, rows, width):
    """The stage-2 sketch matrix (one stream, P/compress.py:109-111) generated
    by segments on the device, tail draws replayed and patched: byte-exact."""
    import torch
    from paper_2203_12798_b200.rng import stage2_omega, stage2_omega_finish, stage2_omega_launch
    stats = {}
    h = stage2_omega_launch(seed, rows, width, torch.device("cuda"))
    dev = stage2_omega_finish(h, stats).cpu().numpy()
    assert dev.tobytes() == stage2_omega(seed, rows, width).tobytes(), stats
    if rows * width >= 1e6:
        assert stats["omega2_tail_events"] > 50 and stats["omega2_host_regenerated"] == 0
