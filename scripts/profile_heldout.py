"""Held-out LL on a C2-shaped model (for ncu -k regex:heldout): 3 training iterations, then
heldout_ll over a 20K-document held-out corpus of the same family (burn-in 20)."""
import sys
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))

import bench  # noqa: E402


def main():
    import paper_1610_02496_b200 as slda
    import paper_1610_02496_b200._core as core

    cfg = bench.CONFIGS["c2"]
    toks, _ = core.generate_tokens(0, cfg["D"], cfg["V"], cfg["T"], seed=bench.CORPUS_SEED)
    tc = slda.TrainConfig()
    tc.num_topics = cfg["K"]
    tc.seed = bench.TRAIN_SEED
    tc.device = 0
    m = core.init_view(toks, cfg["D"], cfg["V"], 0, cfg["D"], 0, tc)
    for _ in range(3):
        m.run_iteration(tc)
    hd = 20_000
    held_toks, _ = core.generate_tokens(0, hd, cfg["V"], hd * 333, seed=99)
    held = slda.Corpus.from_arrays(hd, cfg["V"], held_toks[:, 0].copy(), held_toks[:, 1].copy())
    t = time.perf_counter()
    ll = slda.heldout_ll(m, held, burn_in=20, workers=1, seed=5)
    print(f"heldout_ll {ll} in {time.perf_counter() - t:.3f} s")


if __name__ == "__main__":
    main()
