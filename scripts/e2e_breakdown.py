"""Where the end-to-end time of bench.py's e2e leg goes (not product code).

    SLDA_TRACE=1 python scripts/e2e_breakdown.py [--config c3] [--iters 3]

Times (host wall clock, device synchronised) the public-API calls of one e2e run:
init_view (H2D + device setup; SLDA_TRACE prints its phases), each run_iteration, and
the assignments read-back into a pinned and into a pageable buffer.
"""
import argparse
import sys
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1610_02496_b200 as slda  # noqa: E402
import paper_1610_02496_b200._core as core  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--iters", type=int, default=3)
args = ap.parse_args()
cfg = bench.CONFIGS[args.config]
t = time.perf_counter()
toks, lens = core.generate_tokens(0, cfg["D"], cfg["V"], cfg["T"], seed=bench.CORPUS_SEED, threads=0)
print(f"generate {time.perf_counter() - t:.2f} s", flush=True)
pinned = torch.empty((len(toks), 3), dtype=torch.int32, pin_memory=True)
pinned.numpy().view(np.uint32)[:] = toks
del toks
host = pinned.numpy().view(np.uint32)
tc = slda.TrainConfig()
tc.num_topics = cfg["K"]
tc.seed = bench.TRAIN_SEED
tc.device = 0
w_tok, _ = core.generate_tokens(0, 64, 64, 2048, seed=1)
core.init_view(w_tok, 64, 64, 0, 64, 0, tc).run_iteration(tc)
torch.cuda.synchronize()

t = time.perf_counter()
model = core.init_view(host, cfg["D"], cfg["V"], 0, cfg["D"], 0, tc)
print(f"init_view {time.perf_counter() - t:.3f} s", flush=True)
for i in range(args.iters):
    t = time.perf_counter()
    st = model.run_iteration(tc)
    print(f"run_iteration {i}: {time.perf_counter() - t:.3f} s (device {st.device_ms:.1f} ms)", flush=True)
out = torch.empty(cfg["T"], dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
for i in range(2):
    t = time.perf_counter()
    model.assignments(out)
    print(f"assignments -> pinned: {time.perf_counter() - t:.3f} s", flush=True)
t = time.perf_counter()
a = model.assignments()
print(f"assignments -> new array: {time.perf_counter() - t:.3f} s", flush=True)
assert np.array_equal(a, out)
