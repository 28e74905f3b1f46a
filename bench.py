#!/usr/bin/env python
"""ESCA training-iteration throughput on B200 (BASELINE.json metric).

A "step" is one ESCA iteration (sampler -> SSC C_dk rebuild -> C_wk column sums ->
phi + L4/L3/Q) over the whole synthetic corpus, exactly the span the reference
times in run_iteration (proj/src/trainer.cpp:419-449).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]

N > 1 runs under torchrun, one rank per GPU, document shards with NCCL
reduce-scatter / all-reduce / all-gather inside each iteration (strong scaling:
the corpus is fixed).  value = corpus tokens per iteration / (max over ranks of
the device time per iteration).  See DESIGN.md "Measurement".
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
    """Whole iteration: sampler + SSC + recount + phi/L4."""
    ssc = T * 6 + 4 * nnz + 8 * D
    recount = 2 * T + 4 * V * K
    phi = 12 * V * K
    return sampler_bytes(T, row_entries, K, units) + ssc + recount + phi


def ncu_traffic():
    """dram__bytes_read+write per sampler launch from the committed ncu --set full summary."""
    p = REPO / "profiles" / "ncu_sampler_summary.json"
    if p.exists():
        try:
            d = json.loads(p.read_text())
            return d.get("dram_bytes_per_launch"), d.get("config")
        except (ValueError, KeyError):
            pass
    return None, None


# --------------------------------------------------------------------- reference
def reference_run(cfg: dict, sample_tokens: int, steps: int, warmup: int, threads: int):
    """The reference's own CPU implementation (oracle/_ref: proj/src/*.cpp compiled in place)
    on a bounded sample: the first documents of the same corpus, full V and K."""
    sys.path.insert(0, str(REPO / "tests"))
    import paper_1610_02496_b200._core as core
    from oracle_lib import REF_SO, OracleModel, RefModel

    _, lens = core.generate_tokens(0, cfg["D"], cfg["V"], cfg["T"], seed=CORPUS_SEED, doc_begin=0, doc_end=0)
    csum = np.cumsum(lens.astype(np.int64))
    ndocs = int(np.searchsorted(csum, sample_tokens) + 1)
    ndocs = min(ndocs, cfg["D"])
    toks, _ = core.generate_tokens(0, cfg["D"], cfg["V"], cfg["T"], seed=CORPUS_SEED, doc_begin=0, doc_end=ndocs)
    doc, word = toks[:, 0].copy(), toks[:, 1].copy()
    kind = "reference" if REF_SO.exists() else "port"
    workers = threads if kind == "reference" else 1
    t0 = time.perf_counter()
    if kind == "reference":
        m = RefModel(ndocs, cfg["V"], doc, word, None, K=cfg["K"], seed=TRAIN_SEED,
                     num_chunks=min(4 * workers, ndocs), workers=workers)
    else:
        m = OracleModel(ndocs, cfg["V"], doc, word, None, K=cfg["K"], seed=TRAIN_SEED)
    init_s = time.perf_counter() - t0
    times = []
    for i in range(warmup + steps):
        t = time.perf_counter()
        m.iterate()
        el = (m.last_elapsed if kind == "reference" else time.perf_counter() - t)
        if i >= warmup:
            times.append(el)
    med = statistics.median(times)
    T = len(doc)
    return {
        "value": T / med, "unit": "tokens/s", "cores": workers, "kind": kind,
        "sample": (f"first {ndocs} docs of the {cfg['name']} corpus ({T} tokens), full V={cfg['V']} "
                   f"K={cfg['K']}; median of {steps} iterations after {warmup} warm-up "
                   f"(IterationStats.elapsed_s); init_state {init_s:.1f}s untimed; "
                   f"{'oracle/_ref = unmodified reference sources, ' + str(workers) + ' workers, ' + str(min(4 * workers, ndocs)) + ' chunks' if kind == 'reference' else 'C oracle port, 1 thread'}"),
        "ms_per_step": med * 1e3, "tokens": T,
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
    ap.add_argument("--cpu-steps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--exchange", default="peer", choices=["peer", "nccl"],
                    help="N > 1: M-step exchange fused into the kernels over peer memory (default) or NCCL")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]

    world = int(os.environ.get("WORLD_SIZE", "1"))
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
            "config": {"workload": cfg["name"] + " (bounded CPU sample)", **{k: cfg[k] for k in "DVTK"},
                       "sample_tokens": r["tokens"]},
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

    nccl_id = b""
    if world > 1:
        obj = [core.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]

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
    # + D2H of the assignments (result).
    barrier()
    t0 = time.perf_counter()
    exchange = args.exchange if world > 1 else "none"
    if exchange == "peer" and not one_gpu:
        # Peer-memory exchange needs P2P access between every pair of GPUs (NVLink / NVSwitch);
        # any rank without it sends every rank to NCCL.
        local_world = int(os.environ.get("LOCAL_WORLD_SIZE", world))
        ok = all(torch.cuda.can_device_access_peer(dev, o) for o in range(local_world) if o != dev)
        flag = torch.tensor([1 if ok and local_world == world else 0], dtype=torch.int32, device=coll_dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if int(flag.item()) == 0:
            exchange = "nccl"

    def create():
        """init_state over this rank's shard; for N > 1 the engines meet through peer memory
        (CUDA IPC handles exchanged over torch.distributed, then slda_peer_attach) or NCCL.
        Any rank failing to map its peers falls every rank back to NCCL."""
        nonlocal exchange
        if exchange == "peer":
            m = core.init_view(host_tokens, cfg["D"], cfg["V"], b, e, int(csum[b]), tc, rank, world, b"", 1)
            handles = [None] * world
            dist.all_gather_object(handles, m.peer_handles())
            ok = torch.tensor([1], dtype=torch.int32, device=coll_dev)
            try:
                m.peer_attach(handles)
            except Exception as exc:  # noqa: BLE001
                print(f"rank {rank}: peer attach failed ({exc}); falling back to NCCL", file=sys.stderr)
                ok.zero_()
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            if int(ok.item()) == 1:
                return m
            del m
            exchange = "nccl"
        return core.init_view(host_tokens, cfg["D"], cfg["V"], b, e, int(csum[b]), tc, rank, world, nccl_id,
                              1 if world > 1 else 0)

    model = create()
    t_init = time.perf_counter()
    for _ in range(args.steps):
        model.run_iteration(tc)
    t_iters = time.perf_counter()
    model.assignments(assign_out)
    torch.cuda.synchronize()
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    if os.environ.get("SLDA_BENCH_E2E_TRACE"):
        print(f"e2e: init {t_init - t0:.3f} s, {args.steps} iterations {t_iters - t_init:.3f} s, "
              f"assignments {time.perf_counter() - t_iters:.3f} s", file=sys.stderr)

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
    traffic, traffic_cfg = ncu_traffic()
    it_bytes = iteration_bytes(T_shard, row_entries, cfg["K"], cfg["V"], e - b, info["doc_topic_nnz"],
                               info["num_units"])
    it_achieved = it_bytes / (kt["total_ms"] / 1e3) / 1e9

    if rank != 0:
        return
    line = dict(base_line)
    line.update({
        "value": value, "ms_per_step": ms_per_step,
        "config": {"workload": cfg["name"], "D": cfg["D"], "V": cfg["V"], "T": cfg["T"], "K": cfg["K"],
                   "alpha": 50.0 / cfg["K"], "beta": 0.01, "seed": TRAIN_SEED, "corpus_seed": CORPUS_SEED,
                   "parallelism": (f"doc-shards x{world}, M-step exchange: "
                                   + ("fused into the kernels over NVLink peer memory" if exchange == "peer"
                                      else "NCCL reduce-scatter / all-reduce / all-gather")) if world > 1 else "1 GPU",
                   "l2": "inputs larger than L2 (C_dk rows, phi, L4 are GBs; no flush needed)"},
        "roofline": {"bound": "hbm", "kernel": "sampler", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "traffic_config": traffic_cfg,
                     "peak_source": peak_src, "algorithmic_bytes_per_launch": s_bytes,
                     "sampler_ms": kt["sampler_ms"], "iteration_achieved": it_achieved,
                     "iteration_frac": it_achieved / peak, "E_t": row_entries / max(1, T_shard)},
        "kernels_ms": {k: kt[k] for k in ("reset_ms", "sampler_ms", "ssc_ms", "colsum_ms", "phi_ms", "comm_ms",
                                          "total_ms")},
        "mean_doc_topics": info["doc_topic_nnz"] / max(1, e - b),
        "e2e": {"value": cfg["T"] * args.steps / e2e_s, "unit": "tokens/s",
                "h2d_bytes_per_step": int(12 * T_shard / args.steps),
                "d2h_bytes_per_step": int((4 * T_shard) / args.steps + 8),
                "includes": "H2D corpus (pinned) + device PDOW/init + K run_iteration + D2H assignments",
                "seconds": e2e_s},
        "gpu_launches": int(kt["launches"]) * args.steps,
        "clocks": clocks.summary(),
    })
    if world == 1 and not args.no_cpu_baseline:
        r = reference_run(cfg, args.cpu_sample_tokens, args.cpu_steps, 1, threads)
        line["cpu_baseline"] = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")}
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
