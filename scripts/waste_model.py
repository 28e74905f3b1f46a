"""Lock-step waste of the quad-lane sampler's rounds (not product code).

Runs a C3-shaped corpus subset for a few iterations, then replays the sampler's round structure
on the host: units (word segments split at 8192 tokens, execution order = (word, doc length
desc, doc)), 32-token batches, rounds of 8 tokens x 4 sectors per group.  Reports the fraction
of loaded/issued 4-sector groups that belong to tokens whose row already ended (the round runs
to its longest row), and what sorting each batch by row length would leave.
"""
import sys
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
import bench  # noqa: E402
import paper_1610_02496_b200 as slda  # noqa: E402
import paper_1610_02496_b200._core as core  # noqa: E402

cfg = dict(bench.CONFIGS["c3"])
ND = 1_000_000
toks, lens = core.generate_tokens(0, cfg["D"], cfg["V"], cfg["T"], seed=bench.CORPUS_SEED, doc_begin=0, doc_end=ND)
tc = slda.TrainConfig()
tc.num_topics = cfg["K"]
tc.seed = bench.TRAIN_SEED
m = core.init_view(toks, ND, cfg["V"], 0, ND, 0, tc)
for _ in range(12):
    m.run_iteration(tc)
offs, _, _ = m.doc_topic()
nnz = np.diff(offs.astype(np.int64))
lay = m.chunk_layout()
doc_len = np.bincount(lay["sorted_doc"], minlength=ND)
# execution order inside each word segment: doc length desc, doc asc (stable)
seg_off, seg_len = lay["seg_offset"].astype(np.int64), lay["seg_length"].astype(np.int64)
sd = lay["sorted_doc"].astype(np.int64)
nsect = (nnz + 8) // 8
groups = (nsect + 3) // 4
tot_g = tot_lock = tot_sorted = 0
for o, n in zip(seg_off, seg_len):
    docs = sd[o:o + n]
    docs = docs[np.lexsort((docs, -doc_len[docs]))]
    for u0 in range(0, n, 8192):
        ud = docs[u0:u0 + 8192]
        g = groups[ud]
        for b in range(0, len(g), 32):
            bg = g[b:b + 32]
            tot_g += bg.sum()
            for sel in (bg, np.sort(bg)):
                lock = sum(sel[r:r + 8].max() * len(sel[r:r + 8]) for r in range(0, len(sel), 8))
                if sel is bg:
                    tot_lock += lock
                else:
                    tot_sorted += lock
print(f"tokens {len(sd)}, mean nnz {nnz.mean():.1f}, groups/token {tot_g / len(sd):.2f}")
print(f"round lock-step: {tot_lock / tot_g:.3f}x the useful groups; batch sorted by length: {tot_sorted / tot_g:.3f}x")
