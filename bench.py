#!/usr/bin/env python
"""ESCA training-iteration throughput on B200 (BASELINE.json metric).

A "step" is one ESCA iteration (sampler -> SSC C_dk rebuild -> C_wk column sums ->
phi + L4/L3/Q) over the whole synthetic corpus, exactly the span the reference
times in run_iteration (proj/src/trainer.cpp:419-449).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]

N > 1 runs one rank per GPU (under torchrun; launched without it, bench.py re-launches
itself through torch.distributed.run), document shards with the M-step reduce-scatter /
all-reduce / all-gather fused into the kernels over NVLink peer memory (strong scaling: the
corpus is fixed).  value = corpus tokens per iteration / (max over ranks of the device time
per iteration).  See DESIGN.md "Measurement".
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

# BASELINE.json configs (synthetic, family G: LDA-generative).
CONFIGS = {
    "c1": dict(name="C1 oracle-shaped", D=1_000, V=1_000, T=100_000, K=100),
    "c2": dict(name="C2 NYTimes-shaped", D=300_000, V=100_000, T=100_000_000, K=1_000),
    "c3": dict(name="C3 PubMed-shaped", D=8_200_000, V=141_000, T=738_000_000, K=10_000),
    "c4": dict(name="C4 ClueWeb-subset-shaped", D=19_400_000, V=100_000, T=7_100_000_000, K=10_000),
    # One rank's document shard of C4 at 8 GPUs (T/8 tokens, D/8 documents): the per-GPU work of
    # the 8-B200 run, measurable on one GPU (the M-step collectives are not in this number).
    "c4_shard": dict(name="C4 ClueWeb-subset-shaped, one of 8 document shards", D=2_425_000, V=100_000,
                     T=887_500_000, K=10_000),
    "c5_k100": dict(name="C5 NYTimes-shaped K=100", D=300_000, V=100_000, T=100_000_000, K=100),
    "c5_k10000": dict(name="C5 NYTimes-shaped K=10K", D=300_000, V=100_000, T=100_000_000, K=10_000),
    "c5_k50000": dict(name="C5 NYTimes-shaped K=50K", D=300_000, V=100_000, T=100_000_000, K=50_000),
}
CORPUS_SEED = 20161008
TRAIN_SEED = 42
METRIC = "sampled tokens/sec per iteration (K=1K,10K) at 1/2/4/8 B200; % of HBM roofline"
DATA = ("synthetic family G (LDA-generative: K_true=100 Zipf(1) topics over seeded vocabulary "
        "permutations, Dirichlet(0.1) docs, lognormal(0.6) lengths rescaled to T; corpus seed 20161008)")


def measured_peak():
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "200",
                 "-i", str(self.device)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.thread.join(timeout=2)

    def summary(self):
        rows = []
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                rows.append((float(parts[1]), float(parts[2]), parts[5:9]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, flags in rows for i, f in enumerate(flags) if f.lower() == "active"})
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows)}


def sampler_bytes(T: int, row_entries: int, K: int, units: int) -> int:
    """SURVEY.md §8(d) canonical algorithmic bytes of one sampler launch:
    T*(8 token record + 8 row header + 2 topic) + 4*sum_d len_d*nnz_d + 8*K*U_staged."""
    return T * 18 + 4 * row_entries + 8 * K * units


def iteration_bytes(T: int, row_entries: int, K: int, V: int, D: int, nnz: int, units: int) -> int:
    """Whole iteration: sampler + SSC + recount + the M-step.  The M-step moves
    C_wk in (4 V K) and phi + the L8 level out (4.5 V K): SURVEY's canonical phi + L4 write
    (12 V K) counted an L4 array this engine no longer stores.  The z transpose
    (zmove.cu: the sampler's execution-order topics to slots) adds 22 B per token."""
    ssc = T * 6 + 4 * nnz + 8 * D
    recount = 2 * T + 4 * V * K
    mstep = 4 * V * K + (9 * V * K) // 2
    zmove = 22 * T
    return sampler_bytes(T, row_entries, K, units) + ssc + recount + mstep + zmove


def ncu_traffic():
    """dram__bytes_read+write of one sampler launch from the committed ncu --set full summary,
    with the algorithmic bytes of THAT launch (its iteration's E_t), so the two pair up."""
    p = REPO / "profiles" / "ncu_sampler_summary.json"
    if p.exists():
        try:
            d = json.loads(p.read_text())
            return d.get("dram_bytes_per_launch"), d.get("config"), d.get("algorithmic_bytes_at_capture")
        except (ValueError, KeyError):
            pass
    return None, None, None


# --------------------------------------------------------------------- reference
def reference_run(cfg: dict, sample_tokens: int, steps: int, warmup: int, threads: int):
    """The reference's own CPU implementation (oracle/_ref: proj/src/*.cpp compiled in place,
    unmodified) timed on this host's cores, through its run_iteration (IterationStats.elapsed_s).

    The full corpus does not fit a bounded run (C3: ~2.5 min per iteration on 16 cores), and a
    sample's tokens/s is biased low because the M-step (preprocess + rebuild_trees over V x K,
    trainer.cpp:436-438) does not shrink with the sample.  So the run is split into the two
    parts the reference's iteration consists of, each timed by the reference itself:
      * t_fixed: run_iteration on a one-document corpus with the full V and K -- the V x K
        reset / preprocess / tree build, with a ~100-token E-step;
      * t_sample: run_iteration on the first documents of the same corpus (>= sample_tokens);
    per-token E-step + SSC cost e = (t_sample - t_fixed) / T_sample, and the full corpus
    iteration t = t_fixed + e * T (median of `steps` iterations after `warmup`, each part).
    The workload comes from oracle/libcorpusgen.so (the generator alone): nothing of the
    product is loaded."""
    sys.path.insert(0, str(REPO / "tests"))
    from oracle_lib import REF_SO, CorpusGen, OracleModel, RefModel

    gen = CorpusGen(0, cfg["D"], cfg["V"], cfg["T"], seed=CORPUS_SEED, threads=threads)
    lens = gen.doc_lengths()
    csum = np.cumsum(lens.astype(np.int64))
    ndocs = min(int(np.searchsorted(csum, sample_tokens) + 1), cfg["D"])
    kind = "reference" if REF_SO.exists() else "port"
    workers = threads if kind == "reference" else 1

    def make(nd):
        toks = gen.docs(0, nd, lens)
        doc, word = toks[:, 0].copy(), toks[:, 1].copy()
        if kind == "reference":
            return RefModel(nd, cfg["V"], doc, word, None, K=cfg["K"], seed=TRAIN_SEED,
                            num_chunks=min(4 * workers, nd), workers=workers), len(doc)
        return OracleModel(nd, cfg["V"], doc, word, None, K=cfg["K"], seed=TRAIN_SEED), len(doc)

    def timed(m, n_steps, n_warm):
        times = []
        for i in range(n_warm + n_steps):
            t = time.perf_counter()
            m.iterate()
            el = m.last_elapsed if kind == "reference" else time.perf_counter() - t
            if i >= n_warm:
                times.append(el)
        return statistics.median(times)

    m, t_tiny = make(1)
    fixed_steps = max(3, min(steps, 5))
    t_fixed = timed(m, fixed_steps, 1)
    del m
    t0 = time.perf_counter()
    m, T_s = make(ndocs)
    init_s = time.perf_counter() - t0
    t_sample = timed(m, steps, warmup)
    del m
    e_tok = max(t_sample - t_fixed, 0.0) / T_s
    t_full = t_fixed + e_tok * cfg["T"]
    return {
        "value": cfg["T"] / t_full, "unit": "tokens/s", "cores": workers, "kind": kind,
        "sample": (f"{cfg['name']} iteration time reconstructed from two runs of the reference's own "
                   f"run_iteration: V x K M-step part t_fixed = {t_fixed:.3f} s (one-document corpus, median of "
                   f"{fixed_steps}), and the first {ndocs} documents ({T_s} tokens) at {t_sample:.3f} s (median of "
                   f"{steps} after {warmup} warm-up) -> E-step {e_tok * 1e9:.2f} ns/token; full corpus "
                   f"t = t_fixed + T * e = {t_full:.2f} s per iteration; sample rate {T_s / t_sample:.4g} tok/s; "
                   f"init_state {init_s:.1f} s untimed; "
                   + (f"oracle/_ref = unmodified reference sources, {workers} workers, "
                      f"{min(4 * workers, ndocs)} chunks" if kind == "reference" else "C oracle port, 1 thread")),
        "ms_per_step": t_full * 1e3, "tokens": T_s, "t_fixed_s": t_fixed, "t_sample_s": t_sample,
        "e_step_ns_per_token": e_tok * 1e9,
    }


# --------------------------------------------------------------------- ours
def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-sample-tokens", type=int, default=16_000_000)
    ap.add_argument("--cpu-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--trace-iters", type=int, default=50,
                    help="N=1: a fresh engine run this many iterations; iterations 1, 10 and N reported "
                         "(K_d and E_t drift, SURVEY.md 8(d)); 0 disables")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # One process per GPU: re-launch under torch.distributed.run (the driver's own launch
        # sets WORLD_SIZE and lands below).
        import socket

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
        sys.exit(subprocess.run(cmd).returncode)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: one rank per GPU required")
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    threads = os.cpu_count() or 1
    base_line = {"metric": METRIC, "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps,
                 "warmup": args.warmup, "higher_is_better": True, "scaling": "strong",
                 "vs_baseline": None, "dtype": "f32", "data": DATA}

    if args.impl == "reference":
        if rank != 0:
            return
        r = reference_run(cfg, args.cpu_sample_tokens, args.steps, args.warmup, threads)
        line = dict(base_line)
        line.update({
            "impl": "reference", "value": r["value"], "ms_per_step": r["ms_per_step"],
            "config": {"workload": cfg["name"], **{k: cfg[k] for k in "DVTK"},
                       "alpha": 50.0 / cfg["K"], "beta": 0.01, "seed": TRAIN_SEED, "corpus_seed": CORPUS_SEED,
                       "measured_as": "full-corpus iteration = t_fixed (V x K M-step) + T x per-token E-step, "
                                      "both timed by the reference's run_iteration (cpu_baseline.sample)",
                       "sample_tokens": r["tokens"], "t_fixed_s": r["t_fixed_s"], "t_sample_s": r["t_sample_s"]},
            "cpu_baseline": {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": r["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0,
        })
        print(json.dumps(line), flush=True)
        return

    import torch

    # SLDA_BENCH_ONE_GPU=1 (validation only): every rank on cuda:0, gloo for the host-side
    # plumbing -- exercises the N > 1 path (sharding, peer-memory exchange) on a one-GPU box.
    one_gpu = os.environ.get("SLDA_BENCH_ONE_GPU") == "1"
    dev = 0 if one_gpu else local_rank
    torch.cuda.set_device(dev)
    coll_dev = "cpu" if one_gpu else "cuda"
    dist = None
    if world > 1:
        import torch.distributed as dist

        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    import paper_1610_02496_b200 as slda
    import paper_1610_02496_b200._core as core

    # Shard bounds (chunk_boundaries rule) and this rank's documents only.
    _, lens = core.generate_tokens(0, cfg["D"], cfg["V"], cfg["T"], seed=CORPUS_SEED, doc_begin=0, doc_end=0)
    bounds = core.shard_bounds_from_lengths(lens, world)
    b, e = bounds[rank], bounds[rank + 1]
    csum = np.concatenate([[0], np.cumsum(lens.astype(np.int64))])
    toks_np, _ = core.generate_tokens(0, cfg["D"], cfg["V"], cfg["T"], seed=CORPUS_SEED, doc_begin=b, doc_end=e,
                                      threads=max(1, threads // max(1, int(os.environ.get("LOCAL_WORLD_SIZE", world)))))
    T_shard = len(toks_np)
    # Host buffers in pinned memory (the e2e leg copies from here).
    pinned = torch.empty((T_shard, 3), dtype=torch.int32, pin_memory=True)
    pinned.numpy().view(np.uint32)[:] = toks_np
    del toks_np
    host_tokens = pinned.numpy().view(np.uint32)

    tc = slda.TrainConfig()
    tc.num_topics = cfg["K"]
    tc.seed = TRAIN_SEED
    tc.device = dev
    tc.tree_branch = 32 if cfg["K"] <= 32768 else 41

    # Context / module warm-up outside any timed region.
    w_tok, _ = core.generate_tokens(0, 64, 64, 2048, seed=1)
    warm = core.init_view(w_tok, 64, 64, 0, 64, 0, tc)
    warm.run_iteration(tc)
    del warm
    # Process warm-up of device memory: the engine's footprint (setup scratch included, ~110
    # B/token) is mapped and released once, so the e2e leg does not pay the driver's first-touch
    # of pages another process (pytest, smoke) just freed.  Capped by the free memory.
    free_b, _ = torch.cuda.mem_get_info()
    warm_b = min(int(T_shard * 112 + (8 << 30)), int(free_b * 0.9))
    if warm_b > 0:
        blob = torch.empty(warm_b, dtype=torch.uint8, device="cuda")
        del blob
        torch.cuda.empty_cache()

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if not dist:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    assign_out = torch.empty(T_shard, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)

    # ---- e2e: public API from pinned host buffers: H2D + device PDOW/init + K iterations
    # + D2H of the assignments (result).  The whole sequence runs E2E_REPS times (each a fresh
    # engine) and the median is reported: the first run after another heavy process pays the
    # driver's page commits at run-to-run varying cost, all three are listed.
    if world > 1 and not one_gpu:
        # The peer-memory exchange needs P2P access between every pair of GPUs (NVLink /
        # NVSwitch, one node).
        local_world = int(os.environ.get("LOCAL_WORLD_SIZE", world))
        if local_world != world or not all(torch.cuda.can_device_access_peer(dev, o)
                                           for o in range(local_world) if o != dev):
            sys.exit("bench.py: N > 1 needs one node with P2P access between every GPU pair")

    def create():
        """init_state over this rank's shard; for N > 1 the engines meet through peer memory
        (CUDA IPC handles exchanged over torch.distributed, then slda_peer_attach)."""
        m = core.init_view(host_tokens, cfg["D"], cfg["V"], b, e, int(csum[b]), tc, rank, world, 1 if world > 1 else 0)
        if world > 1:
            handles = [None] * world
            dist.all_gather_object(handles, m.peer_handles())
            m.peer_attach(handles)
        return m

    E2E_REPS = 3
    e2e_runs = []
    model = None
    for rep in range(E2E_REPS):
        model = None  # the previous run's engine is released before the next one is timed
        barrier()
        t0 = time.perf_counter()
        model = create()
        t_init = time.perf_counter()
        it_wall = []
        for _ in range(args.steps):
            t_it = time.perf_counter()
            model.run_iteration(tc)
            it_wall.append(time.perf_counter() - t_it)
        t_iters = time.perf_counter()
        model.assignments(assign_out)
        torch.cuda.synchronize()
        e2e_runs.append(max_over_ranks(time.perf_counter() - t0))
        if os.environ.get("SLDA_BENCH_E2E_TRACE"):
            print(f"e2e run {rep}: init {t_init - t0:.3f} s, {args.steps} iterations {t_iters - t_init:.3f} s, "
                  f"assignments {time.perf_counter() - t_iters:.3f} s; per iteration (ms): "
                  + " ".join(f"{1e3 * w:.1f}" for w in it_wall), file=sys.stderr)
    e2e_s = statistics.median(e2e_runs)

    # ---- device-timed: W warm-up iterations, then exactly K timed iterations.
    stream = torch.cuda.ExternalStream(model.stream_ptr())
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev) as clocks:
        for _ in range(args.warmup):
            model.iterate_async()
        model.synchronize()
        barrier()
        start.record(stream)
        for _ in range(args.steps):
            model.iterate_async()
        end.record(stream)
        model.synchronize()
    barrier()
    region_ms = max_over_ranks(start.elapsed_time(end))
    kt = model.kernel_times_avg(min(args.steps, 64))
    info = model.info()

    ms_per_step = region_ms / args.steps
    value = cfg["T"] / (ms_per_step / 1e3)
    # Roofline of the dominant kernel (sampler) on this rank.
    row_entries = int(kt["sampler_row_entries"])
    s_bytes = sampler_bytes(T_shard, row_entries, cfg["K"], info["num_units"])
    peak, peak_src = measured_peak()
    achieved = s_bytes / (kt["sampler_ms"] / 1e3) / 1e9
    traffic, traffic_cfg, traffic_alg = ncu_traffic()
    it_bytes = iteration_bytes(T_shard, row_entries, cfg["K"], cfg["V"], e - b, info["doc_topic_nnz"],
                               info["num_units"])
    it_achieved = it_bytes / (kt["total_ms"] / 1e3) / 1e9

    xbytes = max_over_ranks(float(kt["exchange_bytes"]))
    if rank != 0:
        return
    line = dict(base_line)
    line.update({
        "value": value, "ms_per_step": ms_per_step,
        "config": {"workload": cfg["name"], "D": cfg["D"], "V": cfg["V"], "T": cfg["T"], "K": cfg["K"],
                   "alpha": 50.0 / cfg["K"], "beta": 0.01, "seed": TRAIN_SEED, "corpus_seed": CORPUS_SEED,
                   "parallelism": (f"doc-shards x{world}, sparse C_wk reduce-scatter + all-gather inside the M-step "
                                   "kernels over NVLink peer memory") if world > 1 else "1 GPU",
                   "l2": "inputs larger than L2 (C_dk rows, phi, L4 are GBs; no flush needed)"},
        "roofline": {"bound": "hbm", "kernel": "sampler", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "traffic_config": traffic_cfg,
                     "traffic_algorithmic_bytes": traffic_alg,
                     "traffic_over_algorithmic": traffic / traffic_alg if traffic and traffic_alg else None,
                     "peak_source": peak_src, "algorithmic_bytes_per_launch": s_bytes,
                     "sampler_ms": kt["sampler_ms"], "iteration_achieved": it_achieved,
                     "iteration_frac": it_achieved / peak, "E_t": row_entries / max(1, T_shard)},
        "kernels_ms": {k: kt[k] for k in ("reset_ms", "sampler_ms", "zmove_ms", "ssc_ms", "exchange_ms", "colsum_ms", "phi_ms",
                                          "join_ms", "total_ms")},
        "sampler_shape": info["sampler_shape"],
        "mean_doc_topics": info["doc_topic_nnz"] / max(1, e - b),
        "e2e": {"value": cfg["T"] * args.steps / e2e_s, "unit": "tokens/s",
                "h2d_bytes_per_step": int(12 * T_shard / args.steps),
                "d2h_bytes_per_step": int((4 * T_shard) / args.steps + 8),
                "includes": "H2D corpus (pinned) + device PDOW/init + K run_iteration + D2H assignments",
                "seconds": e2e_s, "runs_seconds": e2e_runs,
                "method": f"median of {E2E_REPS} complete runs, each a fresh engine"},
        "gpu_launches": int(kt["launches"]) * args.steps,
        "clocks": clocks.summary(),
    })
    if world > 1:
        line["exchange"] = {"bytes_read_per_rank": xbytes, "dense_c_wk_bytes": 4 * cfg["V"] * cfg["K"],
                            "what": "bytes each rank read from the other ranks' memory per M-step (sparse "
                                    "C_wk lists: reduce-scatter + all-gather), max over ranks"}
        if one_gpu:
            line["exchange"]["note"] = "all ranks shared one GPU (SLDA_BENCH_ONE_GPU=1): validation, not NVLink timing"
    if world == 1 and args.trace_iters > 0:
        # Per-iteration drift (report iterations 1, 10 and 50): a fresh engine from
        # the same host tokens, device times of single iterations, outside the timed region.
        model = None
        m2 = create()
        marks = sorted({1, 10, args.trace_iters} & set(range(1, args.trace_iters + 1)))
        trace = {}
        for i in range(1, args.trace_iters + 1):
            m2.run_iteration(tc)
            if i in marks:
                kt2, inf2 = m2.kernel_times(), m2.info()
                trace[str(i)] = {"ms": kt2["total_ms"], "sampler_ms": kt2["sampler_ms"],
                                 "tokens_per_s": T_shard / (kt2["total_ms"] / 1e3),
                                 "E_t": kt2["sampler_row_entries"] / max(1, T_shard),
                                 "K_d": inf2["doc_topic_nnz"] / max(1, e - b)}
        del m2
        line["by_iteration"] = {"what": "one fresh engine, device time of single iterations (not the timed "
                                        "region); E_t = mean C_dk row entries read per token, K_d = "
                                        "mean_doc_topics after the iteration", "iterations": trace}
    if world == 1 and not args.no_cpu_baseline:
        model = None
        r = reference_run(cfg, args.cpu_sample_tokens, args.cpu_steps, 1, threads)
        line["cpu_baseline"] = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")}
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
