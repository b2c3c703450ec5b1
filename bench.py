#!/usr/bin/env python
"""Benchmark of the dGN evaluation hot path (BASELINE.json metric: CPD gradient evals/s).

One step = one full pass of the hot path over the workload:
  tf_cpd_eval (residual, F, three fused MTTKRPs, Grams)  [+ one SUM all-reduce of [grad|f] when N>1]
  + tf_cg_solve (Hadamard chains, Jacobi-free CG on (J^T J + lambda I) x = -grad, fixed iterations)
The evaluation uses the library's default guarded Pi form (reading R31 of DESIGN.md): the three MTTKRPs of T
in one pass (4IJKR flops) with F by the Gram expansion, rerun in the residual form (6IJKR) on the device when
cancellation makes the expansion unsafe; the JSON line reports which one the timed steps used.
Default workload: c5 (1200^3, R=100, 13.8 GB fp64 T, 20 CG iterations) — the largest BASELINE
config, the one the north star's scaling target is quoted on, and it fits one GPU.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1..c5] [--impl reference]

N>1 is launched by torchrun (one rank per GPU, NCCL); T is sharded along K (strong scaling of one
problem: total work fixed). Timing: W untimed warm-up steps, then K steps bracketed by a barrier and
cuda synchronize, CUDA events on the evaluation stream, max over ranks. T (13.8 GB) exceeds the
126 MB L2, so no flush is needed between steps; for configs whose T would fit in L2 (c1, c2) every timed
step is preceded by a 256 MB L2-flushing write and timed by its own CUDA-event pair (the flush outside it). `--impl reference` times the CPU oracle (the
"reference arm" of this tier) on a bounded sample of the same workload.
"""
from __future__ import annotations

L2_BYTES = 126 * 1024 * 1024        # B200 L2
L2_FLUSH_BYTES = 256 * 1024 * 1024  # written between timed steps when T could stay in L2

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "CPD gradient evals/s (fused 3-mode MTTKRP+f); % of FP64/HBM roofline"
UNIT = "evals/s"


def load_json(path, default=None):
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return default


def fp64_peak():
    """Measured FP64 tensor-core (DMMA) peak on this pool's B200 (tools/peaks.cu, profiles/peaks_r01.json)."""
    p = load_json(os.path.join(ROOT, "profiles", "peaks_r01.json"), {}) or {}
    return float(p.get("best_dmma_tflops", 37.07)), float(p.get("read_hbm_gbs", 6914.0))


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 50 ms during the timed region (short configs need enough
    steps for the region to span several samples: c1-c3 are run with --steps in the thousands)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- CPU oracle timing
def host_cpu():
    """The host CPU model and core count (lscpu), recorded beside every oracle timing."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                model = ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return {"model": model, "nproc": os.cpu_count()}


def oracle_shard_sample(cfg, T_shard, w_np, k_s, threads):
    """Time the oracle (as it stands, never tuned) on one K-shard of the workload plus the step's whole CG.

    The sample is a real unit of the method's sharded form: F + grad over the contiguous shard of
    the first k_s frontal slices (oracle_eval, OpenMP over slices; the evaluation is a sum over slices, so a
    shard costs exactly k_s/K of the evaluation), then ALL cfg.cg_iters iterations of Alg. CG-dGN with Thm-Hv
    matvecs on the full parameter vector (not scaled). Returns (evals/s of one full step on this host, seconds
    actually spent, description): evals/s = 1 / (t_shard * K / k_s + t_cg).
    """
    import numpy as np

    import oracle
    I, J, K, R = cfg.I, cfg.J, cfg.K, cfg.R
    A = w_np[:I * R]
    B = w_np[I * R:(I + J) * R]
    C = w_np[(I + J) * R:].reshape(R, K)[:, :k_s].reshape(-1)
    ws = np.concatenate([A, B, C])
    t0 = time.perf_counter()
    f, g = oracle.cpd_eval(T_shard, ws, I, J, k_s, R, nthreads=threads)
    t_eval = time.perf_counter() - t0
    t_cg = 0.0
    if cfg.cg_iters:
        rhs = -np.concatenate([g[:(I + J) * R], np.zeros(K * R)])
        rhs[(I + J) * R:] = -np.pad(g[(I + J) * R:].reshape(R, k_s), ((0, 0), (0, K - k_s))).reshape(-1)
        t0 = time.perf_counter()
        oracle.cg(w_np, rhs, cfg.lam, cfg.cg_iters, I, J, K, R)
        t_cg = time.perf_counter() - t0
    step_s = t_eval * K / k_s + t_cg
    sample = (f"oracle_eval on the K-shard of frontal slices 0..{k_s - 1} of {K} ({t_eval:.2f} s, {threads} OpenMP "
              f"threads, 80-bit accumulation; the evaluation is a sum over slices, so one shard is {k_s}/{K} of it)")
    if cfg.cg_iters:
        sample += f" + all {cfg.cg_iters} CG iterations on the full vector ({t_cg:.2f} s, one thread)"
    sample += f"; one step = {t_eval:.2f} s x {K}/{k_s} + {t_cg:.2f} s"
    return 1.0 / step_s, t_eval + t_cg, sample


def pick_k_slices(cfg, T_first_slice, w_np, budget_s=12.0, threads=16):
    """Shard size (frontal slices) for ~budget_s of CPU work: time one slice on one thread, then scale."""
    import numpy as np

    import oracle
    I, J, K, R = cfg.I, cfg.J, cfg.K, cfg.R
    C = w_np[(I + J) * R:].reshape(R, K)[:, :1].reshape(-1)
    ws = np.concatenate([w_np[:(I + J) * R], C])
    t0 = time.perf_counter()
    oracle.cpd_eval(T_first_slice, ws, I, J, 1, R, nthreads=1)
    t1 = time.perf_counter() - t0          # one slice on one thread
    per_slice = t1 / max(1, threads)
    return int(max(1, min(cfg.K, budget_s / max(per_slice, 1e-9))))


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    import synth
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg = synth.CONFIGS[args.config]
    threads = os.cpu_count() or 1
    P1 = synth.make_problem(args.config, "cpu", k_range=(0, 1))
    k_sl = pick_k_slices(cfg, P1.T.numpy().reshape(-1), P1.w(cfg.points[-1]).numpy(), 6.0, threads)
    P = synth.make_problem(args.config, "cpu", k_range=(0, k_sl))
    w = P.w(cfg.points[-1]).numpy()
    T = P.T.numpy().reshape(-1)
    # the oracle has no warm-up state: the W warm-up steps would only repeat the CPU work, so none are run
    vals, secs, sample = [], [], ""
    t_run = time.perf_counter()
    for _ in range(max(1, args.steps)):
        v, s, sample = oracle_shard_sample(cfg, T, w, k_sl, threads)
        vals.append(v)
        secs.append(s)
    t_run = time.perf_counter() - t_run
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": len(vals), "warmup": 0, "ms_per_step": 1000.0 * statistics.median(secs), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64 (80-bit long double accumulation)",
        "data": "synthetic (seeded, BASELINE.json recipe)",
        "config": {"workload": f"{cfg.name}: {cfg.desc}", "I": cfg.I, "J": cfg.J, "K": cfg.K, "R": cfg.R,
                   "cg_iters": cfg.cg_iters, "lambda": cfg.lam},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample,
                         "host": host_cpu()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": t_run,
        "note": ("the reference arm of this tier is the CPU oracle on the box's host cores. Each step is one "
                 "bounded sample (a K-shard evaluation + the whole CG); ms_per_step is the wall time a sample "
                 "step actually took, value the evals/s of one full step that the sample implies"),
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- multi-rank control path
def init_ranks(backend: str, cuda: bool):
    """One process per GPU (torchrun env: RANK / LOCAL_RANK / WORLD_SIZE / MASTER_*): the process group and
    this rank's device. NCCL's communicator set-up lines (nranks, NVLS / P2P over NVLink) go to stderr."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if cuda and backend != "nccl":
        local = local % max(1, torch.cuda.device_count())
    if world > 1:
        if cuda:
            torch.cuda.set_device(local)
        if backend == "nccl":
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return world, rank, local


def max_over_ranks(x: float, dev, world: int) -> float:
    """The timed-region length as the max over ranks (a MAX all-reduce), the value every rank reports."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_mock(args):
    """TEST-ONLY check of the multi-rank control path on CPU (gloo; tests/test_dist_gloo.py runs it under
    torchrun with 2 ranks): the same rank set-up, K-sharding (shard_range), ShardedEvaluator with its single SUM
    all-reduce of [grad | f], barriers, timed loop and max-over-ranks reduction as the CUDA arm, with a stand-in
    evaluator that is NOT the method (f_local = sum of the local slices, dF/dC row k = sum of slice k, dF/dA =
    dF/dB = 0) so that the all-reduced result is checkable exactly. It measures nothing; its JSON line says
    "mock": true and carries no throughput."""
    import torch
    import torch.distributed as dist

    import synth
    from paper_2110_05997_b200.dist import ShardedEvaluator, shard_range

    world, rank, _ = init_ranks("gloo", cuda=False)
    cfg = synth.CONFIGS[args.config]
    I, J, K, R = cfg.I, cfg.J, cfg.K, cfg.R
    k0, k1 = shard_range(K, rank, world)
    P = synth.make_problem(args.config, "cpu", k_range=(k0, k1))

    def stand_in(d, T, w, f, g, grams=None):
        g.zero_()
        f.fill_(float(T.sum()))
        gC = g[(d.I + d.J) * d.R:].view(d.R, d.K_total)
        gC[:, d.k_begin:d.k_begin + d.K] = T.reshape(d.K, -1).sum(dim=1)[None, :]

    ev = ShardedEvaluator(I, J, K, R, rank=rank, world=world, eval_fn=stand_in)
    assert (ev.k0, ev.k1) == (k0, k1)
    w = P.w(cfg.points[-1])

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        ev(P.T, w)
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        f, g = ev(P.T, w)
    barrier()
    sec = max_over_ranks(time.perf_counter() - t0, "cpu", world)
    if rank == 0:
        gC = g[(I + J) * R:].view(R, K)[0]
        print(json.dumps({"mock": True, "impl": "ours-mock", "n_gpus": world, "steps": args.steps,
                          "warmup": args.warmup, "max_rank_seconds": sec, "value": None,
                          "config": {"workload": f"{cfg.name}: {cfg.desc}",
                                     "parallelism": f"K-sharded x{world} + 1 GLOO all-reduce of [grad|f]"},
                          "check": {"f": float(f.item()), "gC_row0": gC.tolist(),
                                    "shards": [list(shard_range(K, r, world)) for r in range(world)]}}),
              flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


# ----------------------------------------------------------------------------- our arm
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2110_05997_b200 as tf
    import synth
    from paper_2110_05997_b200.dist import ShardedEvaluator, shard_range

    # TF_BENCH_BACKEND=gloo (development only): a functional check of the multi-rank path on a box with fewer
    # GPUs than ranks (ranks share a device; the all-reduce goes through the host, so no kernel waits on another
    # rank). Numbers from such a run are not scaling measurements.
    backend = os.environ.get("TF_BENCH_BACKEND", "nccl")
    world, rank, local = init_ranks(backend, cuda=True)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    cfg = synth.CONFIGS[args.config]
    I, J, K, R = cfg.I, cfg.J, cfg.K, cfg.R
    k0, k1 = shard_range(K, rank, world)
    P = synth.make_problem(args.config, dev, k_range=(k0, k1))
    point = cfg.points[-1]
    w = P.w(point).contiguous()
    n = cfg.n
    stream = torch.cuda.current_stream(dev)
    ctx = tf.Context(local, stream)
    ev = ShardedEvaluator(I, J, K, R, rank=rank, world=world, ctx=ctx)
    grams = torch.empty(3 * R * R, dtype=torch.float64, device=dev)
    x = torch.empty(n, dtype=torch.float64, device=dev)
    rhs = torch.empty(n, dtype=torch.float64, device=dev)
    dglob = tf.Dims(I, J, K, R)

    f1 = torch.empty(1, dtype=torch.float64, device=dev)
    g1 = torch.empty(n, dtype=torch.float64, device=dev)

    def step():
        if world == 1:   # one call: F, grad and the Grams (which the evaluation forms anyway)
            f, g = ctx.tf_cpd_eval(dglob, P.T, w, f1, g1, grams=grams)
        else:            # local partials + one all-reduce of [grad | f]; the Grams of the full factors
            f, g = ev(P.T, w, grams=grams)
        torch.neg(g, out=rhs)
        if cfg.cg_iters:
            ctx.tf_cg_solve(dglob, grams, w, rhs, cfg.lam, cfg.cg_iters, 0.0, False, x)
        return f

    def barrier():
        if world > 1:
            if backend == "nccl":
                dist.barrier(device_ids=[local])
            else:
                dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        step()
    barrier()
    ctx.set_timing(True)
    ctx.kernel_stats(reset=True)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    flush_l2 = cfg.t_bytes < 2 * L2_BYTES   # T (and the factors) could stay in L2 from one step to the next
    scratch = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev) if flush_l2 else None
    with ClockSampler(local) as clk:
        barrier()
        if flush_l2:
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(args.steps)]
            for i in range(args.steps):
                scratch.fill_(i)           # evicts T, the factors and the workspaces from L2
                evs[i][0].record(stream)
                step()
                evs[i][1].record(stream)
        else:
            e0.record(stream)
            for _ in range(args.steps):
                step()
            e1.record(stream)
        barrier()
    ms_local = sum(a.elapsed_time(b) for a, b in evs) if flush_l2 else e0.elapsed_time(e1)
    eval_ms, eval_n, launches = ctx.kernel_stats(reset=True)
    ctx.set_timing(False)
    ms_total = max_over_ranks(ms_local, dev, world)
    ms_per_step = ms_total / args.steps
    value = 1000.0 / ms_per_step          # whole-job evaluations of the full problem per second

    # roofline of the dominant kernel (the fused evaluation kernel), on this rank. The evaluation runs in the
    # guarded Pi form (two DMMA slice contractions: 4*I*J*K*R flops) unless its cancellation guard fell back to
    # the residual form (three contractions: 6*I*J*K*R) — ask the library which one the timed steps used.
    kernel_ms = eval_ms / max(1, eval_n)
    fell_back = ctx.eval_fell_back()
    form = "residual" if fell_back != 0 else "pi"
    nctr = 6.0 if form == "residual" else 4.0
    flops = nctr * I * J * (k1 - k0) * R
    peak_tf, peak_bw = fp64_peak()
    achieved_tf = flops / (kernel_ms * 1e-3) / 1e12
    prof, prof_src = {}, None
    for tag in ("r02", "r01"):
        src = os.path.join("profiles", f"ncu_eval_{cfg.name}_{tag}.json")
        prof = load_json(os.path.join(ROOT, src), {}) or {}
        if prof.get("dram_bytes_per_launch"):
            prof_src = src
            break
    traffic = prof.get("dram_bytes_per_launch") if world == 1 else None
    roofline = {"bound": "tensor", "achieved": achieved_tf, "peak": peak_tf, "unit": "TFLOP/s",
                "frac": achieved_tf / peak_tf, "traffic": traffic,
                "traffic_source": (f"{prof_src}: dram__bytes_read.sum + dram__bytes_write.sum of one launch from a "
                                   "stored ncu --set full capture of this kernel at this config (not measured in "
                                   "this run)") if traffic else None,
                "kernel": "k_eval_fused", "kernel_ms": kernel_ms, "eval_form": form,
                "algorithmic": (f"{int(nctr)}*I*J*K_local*R = {flops:.4e} flop per evaluation "
                                + ("(Pi form: T_k B and T_k^T A diag(c_k) per slice, PAPER.md:2641; kernel_ms spans "
                                   "the MTTKRP pass through the guard)" if form == "pi" else
                                   "(residual form: 3 DMMA contractions per slice)")),
                "peak_source": "measured FP64 DMMA (mma.sync.m8n8k4.f64) peak, tools/peaks.cu, profiles/peaks_r01.json",
                "hbm": {"bytes": 8.0 * I * J * (k1 - k0), "achieved_gbs": 8.0 * I * J * (k1 - k0) / (kernel_ms * 1e-3) / 1e9,
                        "peak_gbs": peak_bw}}
    clocks = clk.summary()

    # e2e through the public C ABI with HOST buffers: T streamed from pinned host memory each step
    e2e = None
    if not args.no_e2e:
        T_host = torch.empty(P.T.shape, dtype=torch.float64, pin_memory=True)
        T_host.copy_(P.T)
        w_host = torch.empty(n, dtype=torch.float64, pin_memory=True)
        w_host.copy_(w)
        gh = torch.empty(n + 1, dtype=torch.float64, pin_memory=True)
        xh = torch.empty(n, dtype=torch.float64, pin_memory=True)
        dl = tf.Dims(I, J, k1 - k0, R, K_total=K, k_begin=k0)
        gdev = torch.empty(n + 1, dtype=torch.float64, device=dev)
        wdev = torch.empty(n, dtype=torch.float64, device=dev)

        def step_e2e():
            ctx.tf_cpd_eval_host(dl, T_host, w_host, gh[n:], gh[:n])     # H2D of T (+w) inside, grad/f D2H
            gdev.copy_(gh, non_blocking=True)                               # H2D grad|f
            if world > 1:
                dist.all_reduce(gdev, op=dist.ReduceOp.SUM)
            wdev.copy_(w_host, non_blocking=True)                           # H2D w
            ctx.tf_grams(dglob, wdev, grams)
            torch.neg(gdev[:n], out=rhs)
            if cfg.cg_iters:
                ctx.tf_cg_solve(dglob, grams, wdev, rhs, cfg.lam, cfg.cg_iters, 0.0, False, x)
            xh.copy_(x, non_blocking=True)                                  # D2H step result
            torch.cuda.current_stream(dev).synchronize()

        step_e2e()
        barrier()
        e2e_steps = max(1, min(args.steps, args.e2e_steps))
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            step_e2e()
        barrier()
        sec = time.perf_counter() - t0
        sec = max_over_ranks(sec, dev, world)
        h2d = int(T_host.numel() * 8 + 2 * n * 8 + (n + 1) * 8)
        d2h = int((n + 1) * 8 + n * 8)
        e2e = {"value": e2e_steps / sec, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "steps": e2e_steps,
               "path": "tf_cpd_eval_host (T streamed from pinned host memory in 512 MB slabs, copies overlapped "
                       "with the fused kernel) + grad H2D + tf_grams + tf_cg_solve + x D2H"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        wn = w.cpu().numpy()
        k_sl = pick_k_slices(cfg, P.T[:1].cpu().numpy().reshape(-1), wn, 12.0, threads)
        Ts = P.T[:k_sl].cpu().numpy().reshape(-1)
        v, secs, sample = oracle_shard_sample(cfg, Ts, wn, k_sl, threads)
        cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample, "seconds": secs,
               "host": host_cpu()}
        # the same oracle on ONE host thread (SURVEY.md §8d asks for both runs): a smaller K-shard, same CG
        ks1 = max(1, k_sl // max(1, 2 * threads))
        v1, secs1, sample1 = oracle_shard_sample(cfg, P.T[:ks1].cpu().numpy().reshape(-1), wn, ks1, 1)
        cpu["single_thread"] = {"value": v1, "unit": UNIT, "cores": 1, "sample": sample1, "seconds": secs1}

    # compression stage (NEXT #3), measured once beside the step on the resident T (not part of `value`)
    stages = None
    if rank == 0 and world == 1 and not args.no_stages:
        Om = synth.omega_blocks((I, J, K), R, dev)
        ctx.tf_compress(dglob, P.T, Om)
        ctx.tf_unfolding_grams(dglob, P.T)
        torch.cuda.synchronize(dev)
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        ctx.tf_unfolding_grams(dglob, P.T)
        s1.record(stream)
        torch.cuda.synchronize(dev)
        gram_ms = s0.elapsed_time(s1)
        reps = 3
        s0.record(stream)
        for _ in range(reps):
            comp = ctx.tf_compress(dglob, P.T, Om)
        s1.record(stream)
        torch.cuda.synchronize(dev)
        comp_ms = s0.elapsed_time(s1) / reps
        gram_flops = sum((nl + 1) for nl in (I, J, K)) * float(I) * J * K   # symmetric T_(l) T_(l)^T, algorithmic
        # one Gauss-Newton matvec (Thm Hv) and the CG of the step, timed alone
        vv = rhs.clone()
        yy = torch.empty_like(vv)
        ctx.tf_gn_matvec(dglob, grams, w, vv, cfg.lam, yy)
        torch.cuda.synchronize(dev)
        s0.record(stream)
        for _ in range(10):
            ctx.tf_gn_matvec(dglob, grams, w, vv, cfg.lam, yy)
        s1.record(stream)
        torch.cuda.synchronize(dev)
        mv_us = s0.elapsed_time(s1) * 100.0
        s0.record(stream)
        ctx.tf_cg_solve(dglob, grams, w, rhs, cfg.lam, cfg.cg_iters, 0.0, False, x)
        s1.record(stream)
        torch.cuda.synchronize(dev)
        cg_ms = s0.elapsed_time(s1)
        stages = {"gn_matvec": {"us": mv_us, "cg_ms": cg_ms, "cg_iters": cfg.cg_iters,
                                "flops": (6 + 5 * (I + J + K)) * R * R,
                                "what": "tf_gn_matvec (Thm Hv, PAPER.md:2352-2370, one persistent launch) and "
                                        "tf_cg_solve(cg_iters) alone; latency-bound (O(R^2 sum I) work)"},
                  "compress": {"ms": comp_ms, "ranks": list(comp["ranks"]), "eig_iters": comp["eig_iters"],
                               "unfolding_grams_ms": gram_ms,
                               "unfolding_grams_tflops": gram_flops / (gram_ms * 1e-3) / 1e12,
                               "unfolding_grams_frac": gram_flops / (gram_ms * 1e-3) / 1e12 / peak_tf,
                               "what": "tf_compress: 3 unfolding Grams (k_gemm_dmma, symmetric tiles) + top-P "
                                       "eigenpairs (subspace iteration) + multilinear core; mlsvd_tol 1e-6"}}
        # the whole Tensor Fox flow (compression by ST-MLSVD -> random N(0,1) start on the core, as the paper's
        # benchmarks start -> dGN on the core, paper defaults maxiter 200, tol 1e-6 ->
        # uncompression -> unit columns), fit measured on the original T
        cgi = synth.cg_budget(200, seed=0)
        Ps = [min(x, R) for x in (I, J, K)]
        w0c = torch.cat([synth.randn((R, pl), dev, "cpd-init", l).reshape(-1) for l, pl in enumerate(Ps)])
        ctx.tf_cpd(dglob, P.T, Om, cgi, w0_core=w0c, maxiter=200, tol=1e-6, sequential=True)   # warm-up (buffers)
        torch.cuda.synchronize(dev)
        s0.record(stream)
        Wf, lamf, flow, fh = ctx.tf_cpd(dglob, P.T, Om, cgi, w0_core=w0c, maxiter=200, tol=1e-6, sequential=True)
        s1.record(stream)
        torch.cuda.synchronize(dev)
        stages["tf_cpd"] = {"ms": s0.elapsed_time(s1), "ranks": list(flow["ranks"]), "dgn_iters": flow["dgn"]["iters"],
                            "dgn_stop": flow["dgn"]["reason"], "rel_err": flow["rel_err"],
                            "noise_rel": P.sigma * math.sqrt(I * J * K) / math.sqrt(float(torch.sum(P.T * P.T))),
                            "what": "tf_cpd: ST-MLSVD compression + random N(0,1) core start + dGN on the R~^3 core "
                                    "(PAPER.md:2514-2533, defaults 2626/3137) + uncompression; rel_err on the full T"}
        # the dGN loop itself on the uncompressed tensor (NEXT #2; the paper's uncompressed 2000^3 run,
        # PAPER.md:4048): per iteration one guarded evaluation, Grams, gamma, CG with the paper's random budget,
        # the x^T J^T J x matvec of the gain ratio, norm balancing and the stopping tests (one host sync)
        wd = w.clone()
        cgb = synth.cg_budget(4, seed=0)
        ctx.tf_cpd_dgn(dglob, P.T, wd, cgb, maxiter=1, tol=0.0)   # warm-up
        dms = {}
        for its in (1, 4):   # the difference removes the set-up pass (||T||^2, mean|T|, F and grad at w0)
            wd.copy_(w)
            torch.cuda.synchronize(dev)
            s0.record(stream)
            dout, _ = ctx.tf_cpd_dgn(dglob, P.T, wd, cgb, maxiter=its, tol=0.0)
            s1.record(stream)
            torch.cuda.synchronize(dev)
            dms[its] = (s0.elapsed_time(s1), dout["iters"])
        stages["dgn"] = {"ms_per_iteration": (dms[4][0] - dms[1][0]) / max(1, dms[4][1] - dms[1][1]),
                         "setup_plus_first_ms": dms[1][0], "cg_budget": [int(x) for x in cgb],
                         "what": "tf_cpd_dgn on the uncompressed T from the evaluation point: Tensor Fox's dGN "
                                 "iteration (PAPER.md:2611-2793) with the paper's random CG budget, tol=0; "
                                 "(t(4 iterations) - t(1)) / 3"}
        # CP-ALS (NEXT #4): the three single-mode MTTKRPs and one sweep from the same point
        wa = w.clone()
        mt = []
        for mode in (1, 2, 3):
            M = ctx.tf_mttkrp(dglob, P.T, wa, mode)
            s0.record(stream)
            ctx.tf_mttkrp(dglob, P.T, wa, mode, M)
            s1.record(stream)
            torch.cuda.synchronize(dev)
            mt.append(s0.elapsed_time(s1))
        ctx.tf_als(dglob, P.T, wa, 1)
        torch.cuda.synchronize(dev)
        s0.record(stream)
        ctx.tf_als(dglob, P.T, wa, 1)
        s1.record(stream)
        torch.cuda.synchronize(dev)
        sweep_ms = s0.elapsed_time(s1)
        mt_flops = 2.0 * I * J * K * R
        stages["als"] = {"sweep_ms": sweep_ms, "mttkrp_ms": mt,
                         "mttkrp_tflops": [mt_flops / (x * 1e-3) / 1e12 for x in mt],
                         "mttkrp_frac": [mt_flops / (x * 1e-3) / 1e12 / peak_tf for x in mt],
                         "what": "tf_als: per mode one MTTKRP (chunked Khatri-Rao + k_gemm_dmma) + Grams + Jacobi "
                                 "pseudo-inverse + W = M V^+; tf_mttkrp alone timed per mode"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE.json recipe; no dataset)",
            "config": {"workload": f"{cfg.name}: {cfg.desc}", "I": I, "J": J, "K": K, "R": R,
                       "cg_iters": cfg.cg_iters, "lambda": cfg.lam, "point": point,
                       "parallelism": (f"K-sharded x{world} + 1 {backend.upper()} all-reduce of [grad|f]"
                                       + ("" if backend == "nccl" else " (development switch: ranks share a GPU; "
                                          "not a scaling measurement)")) if world > 1 else "1 GPU",
                       "l2": (f"T = {cfg.t_bytes / 1e6:.1f} MB could stay in the 126 MB L2: a 256 MB write flushes "
                              "L2 before every timed step, outside that step's CUDA-event pair" if flush_l2 else
                              f"inputs larger than L2 (T = {cfg.t_bytes / 1e9:.2f} GB > 126 MB), no flush"),
                       "step": "tf_cpd_eval (F, grad, Grams) + tf_cg_solve(cg_iters)" if world == 1 else
                               "tf_cpd_eval (local, + Grams of the full factors) + all_reduce([grad|f]) + tf_cg_solve(cg_iters)"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
            "gpu_launches": int(launches), "stages": stages,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-stages", action="store_true", help="skip the compression-stage measurement")
    ap.add_argument("--mock", action="store_true",
                    help="TEST ONLY: the multi-rank control path on CPU (gloo) with a stand-in evaluator; no numbers")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    if args.mock:
        return run_mock(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
