"""Generate tests/golden/*.json from the REFERENCE ITSELF (oracle/_ref).

oracle/_ref/libsparselda_ref.so is the unmodified reference (`proj/src/*.cpp`)
compiled in place by oracle/Makefile behind oracle/ref_shim.cpp.  This script
runs it on deterministic corpora and records bit-exact sha256 digests of every
per-iteration array (assignments, C_wk, phi, L4, Q, C_dk) plus scalar results.
The committed JSON pins both the C oracle (tests/test_oracle.py, CPU) and the
B200 engine (tests/test_gpu_parity.py, GPU) without /root/reference at run
time.

Corpora come from the product's host-only synthetic generator
(slda_generate_corpus, deterministic in its parameters); each fixture also
stores the corpus digest so generator drift is caught.

    make oracle && python tests/golden/make_golden.py
    python tests/golden/make_golden.py --big [NAME...]   # the throughput-config cases
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, str(HERE.parent.parent))

from oracle_lib import RefModel, digest, ref_lib  # noqa: E402
from corpora import corpus_arrays, BIG_CASES, CASES  # noqa: E402


def run_case(name: str, spec: dict) -> dict:
    doc, word, D, V = corpus_arrays(spec["corpus"])
    topic = None
    if spec.get("given_topics_seed") is not None:
        rng = np.random.default_rng(spec["given_topics_seed"])
        topic = rng.integers(0, spec["K"], size=len(doc), dtype=np.uint32)
    m = RefModel(D, V, doc, word, topic, K=spec["K"], alpha=spec.get("alpha", 0.0),
                 beta=spec.get("beta", 0.01), seed=spec["seed"],
                 num_chunks=spec.get("chunks", 1), workers=spec.get("workers", 1),
                 sampler=spec.get("sampler", "sparse"))
    out = {"spec": spec, "corpus_digest": digest(np.stack([doc, word])), "T": int(len(doc)),
           "alpha": m.alpha, "iterations": []}
    out["iterations"].append(m.digests())
    kd = []
    # Held-out LL curve (the reference's only LL, eval.cpp:49-133) every `ll_every` iterations.
    curve = {}
    held = corpus_arrays(spec["heldout"]) if spec.get("heldout") else None
    for it in range(1, spec["iterations"] + 1):
        m.iterate()
        out["iterations"].append(m.digests())
        kd.append(m.last_mean_doc_topics)
        if held is not None and spec.get("ll_every") and it % spec["ll_every"] == 0:
            hd, hw, hD, _ = held
            curve[str(it)] = m.heldout_ll(hD, V, hd, hw, burn_in=spec.get("burn_in", 20), seed=spec["seed"])[0]
    out["mean_doc_topics"] = kd
    if curve:
        out["ll_curve"] = curve
    if spec.get("heldout"):
        hd, hw, hD, _ = corpus_arrays(spec["heldout"])
        ll, n = m.heldout_ll(hD, V, hd, hw, burn_in=spec.get("burn_in", 20), seed=spec["seed"])
        out["heldout"] = {"per_token_ll": ll, "tokens": n}
    if spec.get("pdow"):
        ch = m.chunk(0)
        out["pdow"] = {k: digest(np.asarray(v)) for k, v in ch.items() if k != "doc_range"}
    return out


def kats() -> dict:
    lib = ref_lib()
    vecs = {
        "zeros": ([0, 0, 0, 0], [0, 0]),
        "ones": ([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2),
        "pi": ([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0]),
    }
    out = {}
    for k, (ctr, key) in vecs.items():
        o = np.zeros(4, np.uint32)
        lib.ref_philox(np.array(ctr, np.uint32), np.array(key, np.uint32), o)
        out[k] = [int(x) for x in o]
    import ctypes as C
    u0, u1 = C.c_double(), C.c_double()
    lib.ref_uniform2(42, 0, 7, C.byref(u0), C.byref(u1))
    return {"philox": out, "rng_42_0_7": [u0.value, u1.value]}


def main() -> None:
    """`make_golden.py` regenerates every case; `make_golden.py NAME...` (re)generates only
    those cases and keeps the others from the committed file."""
    only = sys.argv[1:]
    cases, path = CASES, HERE / "reference_digests.json"
    if only and only[0] == "--big":
        only = only[1:]
        cases, path = BIG_CASES, HERE / "reference_digests_big.json"
    if (only or cases is BIG_CASES) and path.exists():
        fixtures = json.loads(path.read_text())
    else:
        fixtures = {"kats": kats(), "cases": {}}
    for name, spec in cases.items():
        if only and name not in only:
            continue
        print("case", name, flush=True)
        fixtures["cases"][name] = run_case(name, spec)
        path.write_text(json.dumps(fixtures, indent=1, sort_keys=True))
    print("wrote", path)


if __name__ == "__main__":
    main()
