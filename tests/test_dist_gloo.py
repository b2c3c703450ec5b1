"""The K-sharded multi-rank path on CPU (gloo, world_size 2 and 3): partition, packing and the single
SUM all-reduce of [grad | f] reproduce the full evaluation. The per-rank evaluator here is the oracle
(tests may call it); the product passes the CUDA evaluator through the same ShardedEvaluator."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_eval_fn(d, T, w, f, g):
    import oracle
    I, J, K, R, Kt, k0 = d.I, d.J, d.K, d.R, d.K_total, d.k_begin
    wn = w.numpy()
    A = wn[:I * R]
    B = wn[I * R:(I + J) * R]
    C = wn[(I + J) * R:].reshape(R, Kt)[:, k0:k0 + K].reshape(-1)
    fl, gl = oracle.cpd_eval(T.numpy().reshape(-1), np.concatenate([A, B, C]), I, J, K, R)
    out = np.zeros(R * (I + J + Kt))
    out[:(I + J) * R] = gl[:(I + J) * R]
    out[(I + J) * R:].reshape(R, Kt)[:, k0:k0 + K] = gl[(I + J) * R:].reshape(R, K)
    g.copy_(torch.from_numpy(out))
    f.fill_(fl)


def _worker(rank, world, port, dims, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import synth
        from paper_2110_05997_b200.dist import ShardedEvaluator, shard_range
        I, J, K, R = dims
        k0, k1 = shard_range(K, rank, world)
        P = synth.make_problem("c2", "cpu", dims=dims, k_range=(k0, k1))
        ev = ShardedEvaluator(I, J, K, R, eval_fn=_oracle_eval_fn)
        assert (ev.k0, ev.k1) == (k0, k1)
        f, g = ev(P.T, P.w("random"))
        q.put((rank, float(f.item()), g.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,dims", [(2, (13, 11, 7, 3)), (3, (9, 10, 8, 4))])
def test_k_sharded_allreduce_gloo(world, dims):
    pytest.importorskip("paper_2110_05997_b200")
    import oracle
    import synth
    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    port = _free_port()
    procs = [ctxm.Process(target=_worker, args=(r, world, port, dims, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    I, J, K, R = dims
    P = synth.make_problem("c2", "cpu", dims=dims)
    fr, gr = oracle.cpd_eval(P.T.numpy().reshape(-1), P.w("random").numpy(), I, J, K, R)
    for rank, f, g in res:
        assert abs(f - fr) <= 1e-12 * abs(fr)
        np.testing.assert_allclose(g, gr, rtol=1e-11, atol=1e-12 * np.abs(gr).max())
    # every rank holds the identical reduced result
    for _, f, g in res[1:]:
        assert f == res[0][1] and np.array_equal(g, res[0][2])


def test_shard_ranges_cover_and_balance():
    from paper_2110_05997_b200.dist import shard_range
    import synth
    for K in (1, 7, 400, 500, 1200):
        for world in (1, 2, 3, 4, 8):
            rs = [shard_range(K, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == K
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1
            assert rs == [synth.shard_range(K, r, world) for r in range(world)]


def test_sharded_generation_is_bit_identical():
    """A K-shard generated alone equals the same slices of the full tensor (synth counter-based noise)."""
    import synth
    full = synth.make_problem("c3", "cpu", dims=(12, 9, 10, 3))
    part = synth.make_problem("c3", "cpu", dims=(12, 9, 10, 3), k_range=(4, 7))
    assert torch.equal(full.T[4:7], part.T)
    assert torch.equal(full.w("random"), part.w("random"))


def _hook_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2110_05997_b200.dist import allreduce_hook
        import synth
        # the exchange of the sharded dGN loop: partial [grad | F] of each rank's slices (here: the oracle's
        # per-shard values packed like the library packs them) summed in place by the hook
        I, J, K, R = 9, 8, 10, 3
        from paper_2110_05997_b200.dist import shard_range
        k0, k1 = shard_range(K, rank, world)
        P = synth.make_problem("c2", "cpu", dims=(I, J, K, R), k_range=(k0, k1))
        g = torch.zeros(R * (I + J + K) + 1, dtype=torch.float64)
        _oracle_eval_fn(type("D", (), dict(I=I, J=J, K=k1 - k0, R=R, K_total=K, k_begin=k0))(), P.T,
                        P.w("random"), g[-1:], g[:-1])
        sums = torch.tensor([float(P.T.abs().sum()), float((P.T * P.T).sum())], dtype=torch.float64)
        hook = allreduce_hook()
        hook(g)
        hook(sums)
        q.put((rank, g.numpy().copy(), sums.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_dgn_exchange_gloo(world):
    """The all-reduce hook of tf_cpd_dgn_sharded (dist.allreduce_hook) on gloo: the summed partial [grad | F]
    of the ranks' K-shards is the full evaluation, the summed tensor sums are the full ||T||^2 and sum|t|, and
    every rank holds the identical buffer (so the replicated CG/damping/stopping run identically)."""
    pytest.importorskip("paper_2110_05997_b200")
    import oracle
    import synth
    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    port = _free_port()
    procs = [ctxm.Process(target=_hook_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    I, J, K, R = 9, 8, 10, 3
    P = synth.make_problem("c2", "cpu", dims=(I, J, K, R))
    fr, gr = oracle.cpd_eval(P.T.numpy().reshape(-1), P.w("random").numpy(), I, J, K, R)
    for _, g, sums in res:
        np.testing.assert_allclose(g[:-1], gr, rtol=1e-11, atol=1e-12 * np.abs(gr).max())
        assert abs(g[-1] - fr) <= 1e-12 * fr
        assert abs(sums[1] - float((P.T * P.T).sum())) <= 1e-12 * sums[1]
        assert abs(sums[0] - float(P.T.abs().sum())) <= 1e-12 * sums[0]
    for _, g, sums in res[1:]:
        assert np.array_equal(g, res[0][1]) and np.array_equal(sums, res[0][2])


def test_bench_multi_rank_control_path_under_torchrun():
    """bench.py's multi-rank control path end to end, launched the way the driver launches N > 1 (torchrun, one
    process per rank, 127.0.0.1 rendezvous), on CPU with gloo (`--mock`: the same rank set-up, K-sharding,
    ShardedEvaluator all-reduce, barriers and max-over-ranks timing, with a stand-in evaluator whose all-reduced
    output is exactly checkable): both ranks exit 0, rank 0 alone prints one JSON line, the shards partition K,
    f = sum of all of T and row k of the dF/dC block is the sum of slice k for every k (each rank contributed its
    own slices and zeros elsewhere)."""
    import json
    import subprocess
    import sys
    import synth
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2", "--mock", "--config", "c1", "--steps",
           "2", "--warmup", "3"]
    out = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, out.stdout
    b = json.loads(lines[0])
    assert b["mock"] is True and b["value"] is None and b["n_gpus"] == 2
    assert b["config"]["parallelism"].startswith("K-sharded x2")
    P = synth.make_problem("c1", "cpu")
    K = P.cfg.K
    assert b["check"]["shards"] == [[0, K // 2], [K // 2, K]]
    T = P.T.numpy()
    assert abs(b["check"]["f"] - float(T.sum())) <= 1e-12 * abs(T).sum()
    np.testing.assert_allclose(b["check"]["gC_row0"], T.reshape(K, -1).sum(axis=1), rtol=1e-13, atol=1e-13)
