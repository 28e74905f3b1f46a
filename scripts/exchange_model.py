"""Exact per-rank bytes of the sparse C_wk exchange at N ranks, from a real
one-GPU C3 run: the model's assignments at iteration `--iters` give every shard's partial C_wk
and the reduced one; the bytes a rank reads are those of the entry lists it gathers (4 B per
entry, a count above 65535 taking several) plus 8 B of row index per source row.

    python scripts/exchange_model.py --config c3 --iters 10 --ranks 2 4 8
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))

import bench  # noqa: E402


def pieces(counts: torch.Tensor) -> int:
    return int(((counts + 65534) // 65535).sum())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--ranks", type=int, nargs="+", default=[2, 4, 8])
    args = ap.parse_args()
    import paper_1610_02496_b200 as slda
    import paper_1610_02496_b200._core as core

    cfg = bench.CONFIGS[args.config]
    toks, lens = core.generate_tokens(0, cfg["D"], cfg["V"], cfg["T"], seed=bench.CORPUS_SEED)
    tc = slda.TrainConfig()
    tc.num_topics = cfg["K"]
    tc.seed = bench.TRAIN_SEED
    tc.device = 0
    m = core.init_view(toks, cfg["D"], cfg["V"], 0, cfg["D"], 0, tc)
    for _ in range(args.iters):
        m.run_iteration(tc)
    z = torch.from_numpy(m.assignments().astype(np.int64))
    del m
    torch.cuda.empty_cache()
    V, K = cfg["V"], cfg["K"]
    word = torch.from_numpy(toks[:, 1].astype(np.int64))
    key = (word * K + z).cuda()
    del z
    doc_lens = np.bincount(toks[:, 0], minlength=cfg["D"]).astype(np.uint32) if lens is None else lens
    csum = np.concatenate([[0], np.cumsum(np.asarray(doc_lens, np.int64))])
    full_keys, full_counts = torch.unique(key, return_counts=True)
    out = {"config": cfg["name"], "iteration": args.iters, "nnz_c_wk": int(full_keys.numel()),
           "entries_c_wk": pieces(full_counts), "dense_c_wk_bytes": 4 * V * K, "ranks": {}}
    for N in args.ranks:
        bounds = core.shard_bounds_from_lengths(np.asarray(doc_lens, np.uint32), N)
        rows = -(-V // N)  # slda_word_slice: ceil(V / N) rows per slice
        part = []
        for r in range(N):
            k, c = torch.unique(key[int(csum[bounds[r]]):int(csum[bounds[r + 1]])], return_counts=True)
            part.append(((k // K) // rows, (c + 65534) // 65535))  # (slice of each cell, its pieces)
        full_slice = (full_keys // K) // rows
        full_pieces = (full_counts + 65534) // 65535
        slice_entries = [int(full_pieces[full_slice == s].sum()) for s in range(N)]
        per_rank = []
        for r in range(N):
            rs = sum(int(part[p][1][part[p][0] == r].sum()) for p in range(N) if p != r)
            ag = sum(slice_entries[p] for p in range(N) if p != r)
            own_rows = max(0, min(V, (r + 1) * rows) - min(V, r * rows))
            index = 8 * ((N - 1) * own_rows + (V - own_rows))
            per_rank.append(4 * (rs + ag) + index)
        out["ranks"][N] = {"bytes_read_per_rank_max": max(per_rank), "bytes_read_per_rank_mean": sum(per_rank) / N,
                           "partial_entries_rank0": int(part[0][1].sum()),
                           "nvlink_ms_at_900GBps": max(per_rank) / 900e9 * 1e3}
        print(N, out["ranks"][N], flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
