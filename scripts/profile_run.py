"""Minimal driver for ncu captures: build one engine on a BASELINE config and run
N iterations (no warm-up engine, no CPU baseline), so `-k regex:<kernel> -s 1 -c 1`
selects the second iteration's launch of that kernel.

    ncu --set full -k regex:sampler -s 1 -c 1 -o prof python scripts/profile_run.py --config c2
"""
import argparse
import sys
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))

import bench  # noqa: E402  (CONFIGS, seeds)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2", choices=sorted(bench.CONFIGS))
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--shape", default=None, help="D,V,T,K override (experiments)")
    ap.add_argument("--chunks", type=int, default=0, help="num_chunks (streaming with --device-budget)")
    ap.add_argument("--device-budget", type=int, default=0, help="bytes; 1 forces streaming")
    args = ap.parse_args()
    import paper_1610_02496_b200 as slda
    import paper_1610_02496_b200._core as core

    cfg = dict(bench.CONFIGS[args.config])
    if args.shape:
        cfg.update(zip("DVTK", (int(x) for x in args.shape.split(","))))
    toks, _ = core.generate_tokens(0, cfg["D"], cfg["V"], cfg["T"], seed=bench.CORPUS_SEED)
    tc = slda.TrainConfig()
    tc.num_topics = cfg["K"]
    tc.seed = bench.TRAIN_SEED
    tc.device = 0
    tc.tree_branch = 32 if cfg["K"] <= 32768 else 41
    tc.num_chunks = args.chunks
    tc.device_budget = args.device_budget
    m = core.init_view(toks, cfg["D"], cfg["V"], 0, cfg["D"], 0, tc)
    for _ in range(args.iters):
        t = time.perf_counter()
        st = m.run_iteration(tc)
        kt = m.kernel_times()
        print(f"iter {st.iteration}: {st.device_ms:.2f} ms  " +
              " ".join(f"{k}={v:.3f}" for k, v in kt.items() if k.endswith("_ms")) +
              f" entries/T={kt['sampler_row_entries'] / cfg['T']:.1f} wall={time.perf_counter() - t:.3f}s",
              flush=True)
    print(m.info())


if __name__ == "__main__":
    main()
