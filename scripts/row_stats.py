"""C_dk row statistics of a real model (for row-format decisions): after `--iters` iterations,
the share of the sampler's row bytes (each row is read once per token of its document) in rows
whose largest count fits 2 / 3 / 4 / 8 bits, and the entries' count distribution.

    python scripts/row_stats.py --config c3 --iters 10
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--iters", type=int, default=10)
    args = ap.parse_args()
    import paper_1610_02496_b200 as slda
    import paper_1610_02496_b200._core as core

    cfg = bench.CONFIGS[args.config]
    toks, _ = core.generate_tokens(0, cfg["D"], cfg["V"], cfg["T"], seed=bench.CORPUS_SEED)
    tc = slda.TrainConfig()
    tc.num_topics = cfg["K"]
    tc.seed = bench.TRAIN_SEED
    tc.device = 0
    m = core.init_view(toks, cfg["D"], cfg["V"], 0, cfg["D"], 0, tc)
    for _ in range(args.iters):
        m.run_iteration(tc)
    offs, tops, cnts = m.doc_topic()
    del m
    offs = offs.astype(np.int64)
    nnz = np.diff(offs)
    lens = np.add.reduceat(cnts.astype(np.int64), offs[:-1]) if len(cnts) else np.zeros(0)
    lens[nnz == 0] = 0
    mx = np.maximum.reduceat(cnts, offs[:-1]).astype(np.int64)
    mx[nnz == 0] = 0
    weight = lens * (nnz + 1)  # entries read per iteration (header included)
    out = {"config": cfg["name"], "iteration": args.iters, "docs": int(len(nnz)), "entries": int(len(cnts)),
           "count_hist": {str(c): int((cnts == c).sum()) for c in range(1, 9)},
           "count_gt8": int((cnts > 8).sum())}
    for bits in (2, 3, 4, 8):
        ok = mx < (1 << bits)
        out[f"row_bytes_share_max_count_lt_2^{bits}"] = float(weight[ok].sum() / weight.sum())
        out[f"docs_share_max_count_lt_2^{bits}"] = float(ok.mean())
    print(json.dumps(out))


if __name__ == "__main__":
    main()
