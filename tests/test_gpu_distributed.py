"""The multi-GPU phase API (dp2_als_phase) on one GPU with virtual ranks: the
slices are split into LPT shards, each shard runs the phases on its own
slices, and the R x R partials are summed in rank order between phases --
exactly what the NCCL allreduce does on N GPUs.  Must agree with the
single-GPU graph path (fit_dpar2) to rounding."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 3])
def test_virtual_ranks_match_single_gpu(world):
    import paper_2203_12798_b200 as dp
    from paper_2203_12798_b200 import distributed as D_, synth
    from paper_2203_12798_b200.factors import initial_factors
    from paper_2203_12798_b200.solver import run_als
    cfg = synth.scaled(synth.CONFIGS["c1"], num_slices=40)
    xs = synth.generate(cfg, 3)
    t = dp.IrregularTensor(xs)
    comp = dp.compress(t, 10)
    K, J, R = t.num_slices, t.num_cols, 10
    h, v, w = initial_factors(J, K, R)
    H1, V1, W1, _, tr1, _ = run_als(comp, h, v, w, 16, 0.0, True)
    shards, _ = D_.shard_slices(t.row_counts, world)
    dev = comp.cores.device
    ops = []
    for ids in shards:
        H = torch.from_numpy(h).to(dev)
        V = torch.from_numpy(v).to(dev)
        W = torch.from_numpy(w[ids]).to(dev)
        ops.append(D_.GpuAlsOps(D_.local_rows(comp.cores, ids, R), comp.col_basis, comp.weights, H, V, W, J, R,
                                16, 0.0, True))

    class Virtual:
        def phase(self, ph, it=0, red_in=None):
            outs = [o.phase(ph, it=it, red_in=red_in) for o in ops]
            return outs[0] if outs[0] is None else sum(outs[1:], outs[0].clone())

    class Driver:
        def __init__(self):
            self.pending = None

        def run(self, iters):
            v = Virtual()
            v.phase(0)
            for it in range(iters):
                for a, b in ((1, 2), (3, 4), (5, 6)):
                    v.phase(b, it=it, red_in=v.phase(a, it=it))

    Driver().run(16)
    tr = ops[0].trace.cpu().numpy()
    assert np.allclose(tr, tr1, rtol=1e-10, atol=0)
    assert torch.allclose(ops[0].H, H1, rtol=0, atol=1e-9 * float(H1.abs().max()))
    assert torch.allclose(ops[0].V, V1, rtol=0, atol=1e-9 * float(V1.abs().max()))
    for o, ids in zip(ops, shards):
        assert torch.allclose(o.W, W1[ids], rtol=0, atol=1e-9 * float(W1.abs().max()))
        assert torch.equal(o.trace, ops[0].trace)


def test_distributed_fit_replicated_als_world1_matches_fit():
    """bench.py's N > 1 path (DistributedFit: sharded stage 1, M assembled,
    stage 2 + the persistent ALS replicated, Q for the local slices) at world
    size 1 must reproduce fit_dpar2 on the same tensor."""
    import paper_2203_12798_b200 as dp
    from paper_2203_12798_b200 import distributed as D_, synth
    cfg = synth.scaled(synth.CONFIGS["c1"], num_slices=30)
    runner = D_.DistributedFit(cfg, 4, 0, 1)
    opts = dp.SolverOptions(max_iters=12, tol=0.0, seed=0)
    f, tr = runner.fit(cfg.rank, opts)
    g, tr2 = dp.fit_dpar2(runner.tensor, cfg.rank, opts, output="device")
    for key in ("H", "V", "W"):
        a, b = getattr(f, key).cpu().numpy(), getattr(g, key).cpu().numpy()
        assert np.abs(a - b).max() <= 1e-10 * max(np.abs(b).max(), 1.0), key
    assert np.allclose(tr.objective, tr2.objective, rtol=1e-12, atol=0)
    q1, q2 = f.Q_packed.cpu().numpy(), g.Q_packed.cpu().numpy()
    assert np.abs(q1 - q2).max() <= 1e-10


def _nccl_world1():
    import socket
    import torch.distributed as dist
    if not dist.is_initialized():
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
    return dist


@pytest.mark.parametrize("als", ["sharded", "replicated", "auto"])
def test_distributed_fit_nccl_world1_matches_fit(als):
    """DistributedFit over a real NCCL process group (world size 1 on this
    box): the all-gather M assembly, and the sharded ALS captured with its
    allreduces in a CUDA graph (replayed on the second fit) or the replicated
    loop, reproduce fit_dpar2."""
    import paper_2203_12798_b200 as dp
    from paper_2203_12798_b200 import distributed as D_, synth
    _nccl_world1()
    cfg = synth.scaled(synth.CONFIGS["c1"], num_slices=30)
    runner = D_.DistributedFit(cfg, 4, 0, 1, host_slices=synth.generate(cfg, 4))
    opts = dp.SolverOptions(max_iters=12, tol=0.0, seed=0)
    g, tr2 = dp.fit_dpar2(runner.tensor, cfg.rank, opts, output="device")
    for rep in range(2):  # second fit replays the captured graph
        f, tr = runner.fit(cfg.rank, opts, als=als)
        for key in ("H", "V", "W"):
            a, b = getattr(f, key).cpu().numpy(), getattr(g, key).cpu().numpy()
            assert np.abs(a - b).max() <= 1e-9 * max(np.abs(b).max(), 1.0), (als, rep, key)
        assert np.allclose(tr.objective, tr2.objective, rtol=1e-10, atol=0)
        q1, q2 = f.Q_packed.cpu().numpy(), g.Q_packed.cpu().numpy()
        assert np.abs(q1 - q2).max() <= 1e-9
    if als == "sharded":
        assert runner._als_graph[1].captured, "the sharded loop was not captured in a CUDA graph"
