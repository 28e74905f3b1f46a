"""Deterministic test corpora shared by the golden generator and the tests.

Corpora are produced by the product's host-only generator
(``Corpus.generate`` -> slda_generate_corpus; no GPU needed) and optionally
transformed to exercise edge cases the reference tests: non doc-sorted token
order, empty documents, long documents, K = 1, K above the 48 KB shared
memory line, given (non-sentinel) topics.
"""
from __future__ import annotations

import numpy as np


def corpus_arrays(spec: dict):
    """Returns (doc, word, D, V) as uint32 arrays in corpus order."""
    import paper_1610_02496_b200 as slda

    c = slda.Corpus.generate(spec["family"], spec["D"], spec["V"], spec["T"], seed=spec["seed"],
                             latent_topics=spec.get("latent", 100), threads=0)
    toks = c.tokens()
    doc = toks[:, 0].copy()
    word = toks[:, 1].copy()
    D, V = spec["D"], spec["V"]
    if spec.get("spread_docs"):
        # Every other document id is empty (docs with zero tokens in the shard).
        doc = doc * 2
        D = 2 * D
    if spec.get("shuffle_seed") is not None:
        perm = np.random.default_rng(spec["shuffle_seed"]).permutation(len(doc))
        doc, word = doc[perm], word[perm]
    return doc.astype(np.uint32), word.astype(np.uint32), D, V


G = 0
U = 1

CASES: dict[str, dict] = {
    # BASELINE.json configs[0]: D=1K, V=1K, T=100K, K=100, 50 iterations.
    "c1": {"corpus": {"family": G, "D": 1000, "V": 1000, "T": 100_000, "seed": 20161008},
           "K": 100, "seed": 42, "iterations": 50, "pdow": True, "ll_every": 5,
           "heldout": {"family": G, "D": 200, "V": 1000, "T": 20_000, "seed": 7}},
    "k1": {"corpus": {"family": U, "D": 30, "V": 12, "T": 180, "seed": 5},
           "K": 1, "seed": 11, "iterations": 3},
    "u_k7_chunks": {"corpus": {"family": U, "D": 300, "V": 200, "T": 12_000, "seed": 6},
                    "K": 7, "seed": 11, "iterations": 5, "chunks": 3, "workers": 4, "pdow": True},
    "u_k64": {"corpus": {"family": U, "D": 120, "V": 64, "T": 10_200, "seed": 21},
              "K": 64, "seed": 7, "iterations": 4},
    "long_docs": {"corpus": {"family": U, "D": 40, "V": 500, "T": 40_000, "seed": 8},
                  "K": 300, "seed": 3, "iterations": 3, "pdow": True},
    "shuffled": {"corpus": {"family": U, "D": 200, "V": 300, "T": 8_000, "seed": 9, "shuffle_seed": 1},
                 "K": 16, "seed": 99, "iterations": 3, "pdow": True},
    "empty_docs": {"corpus": {"family": U, "D": 100, "V": 80, "T": 3_000, "seed": 10, "spread_docs": True},
                   "K": 12, "seed": 5, "iterations": 3, "pdow": True},
    "given_topics": {"corpus": {"family": U, "D": 150, "V": 120, "T": 6_000, "seed": 12},
                     "K": 20, "seed": 4, "iterations": 3, "given_topics_seed": 77},
    # Lognormal lengths 127..5413 tokens: every SSC pass (warp <= 512, medium warp <= 2048, CTA
    # histogram beyond), the last with the histogram in shared memory, then (K = 60,000) in global.
    "ssc_lengths": {"corpus": {"family": G, "D": 300, "V": 2000, "T": 300_000, "seed": 31},
                    "K": 3000, "seed": 9, "iterations": 3},
    "ssc_lengths_k60k": {"corpus": {"family": G, "D": 40, "V": 300, "T": 50_000, "seed": 32},
                         "K": 60_000, "seed": 5, "iterations": 2},
    "k_large": {"corpus": {"family": U, "D": 50, "V": 50, "T": 5_000, "seed": 13},
                "K": 20_000, "seed": 2, "iterations": 2},
    # phi row too large for shared memory: the sampler gathers phi through L1/L2.
    "k_global_phi": {"corpus": {"family": U, "D": 40, "V": 30, "T": 3_000, "seed": 17},
                     "K": 40_000, "seed": 6, "iterations": 2},
    "alpha_beta": {"corpus": {"family": G, "D": 400, "V": 600, "T": 40_000, "seed": 14, "latent": 20},
                   "K": 25, "alpha": 0.3, "beta": 0.05, "seed": 8, "iterations": 4,
                   "heldout": {"family": G, "D": 60, "V": 600, "T": 6_000, "seed": 15, "latent": 20}},
    "nytimes_small": {"corpus": {"family": G, "D": 1000, "V": 5000, "T": 300_000, "seed": 16},
                      "K": 1000, "seed": 42, "iterations": 3, "chunks": 4, "workers": 8},
    # SamplerKind::kVanilla: the O(K) dense-row baseline mode (trainer.cpp:281-285).
    "vanilla_c1": {"corpus": {"family": G, "D": 1000, "V": 1000, "T": 100_000, "seed": 20161008},
                   "K": 100, "seed": 42, "iterations": 8, "sampler": "vanilla"},
    "vanilla_u_k300": {"corpus": {"family": U, "D": 200, "V": 150, "T": 9_000, "seed": 23},
                       "K": 300, "alpha": 0.2, "seed": 5, "iterations": 4, "chunks": 3, "workers": 4,
                       "sampler": "vanilla"},
}


# Throughput-config cases (BASELINE.json configs), pinned bit for bit against digests the
# reference itself produced (tests/golden/reference_digests_big.json, make_golden.py --big;
# the reference ran with 8 workers and 32 chunks -- its results do not depend on either,
# acceptance.cpp:389-445).  They run the engine's DEFAULT kernel selection (no SLDA_* knobs).
BIG_CASES: dict[str, dict] = {
    # BASELINE configs[1] exactly: NYTimes-shaped D=300K, V=100K, T=100M, K=1K (heavy words split
    # into 8192-token units, multi-batch claiming in the 256-thread quad kernel).
    "c2_full": {"corpus": {"family": G, "D": 300_000, "V": 100_000, "T": 100_000_000, "seed": 20161008},
                "K": 1000, "seed": 42, "iterations": 3, "chunks": 32, "workers": 8},
    # PubMed-shaped (configs[2]) at a third of a GPU-hour of reference CPU time: V=141K, K=10,000,
    # T/D = 90, 25M tokens; 199 words exceed the 8192-token unit cap (the longest has 30,426
    # tokens), so split units and the 512-thread prefetching quad kernel run as in the bench.
    "pubmed_k10k": {"corpus": {"family": G, "D": 280_000, "V": 141_000, "T": 25_000_000, "seed": 20161008},
                    "K": 10_000, "seed": 42, "iterations": 3, "chunks": 32, "workers": 8},
    # C5's K=50,000 point (configs[4]) at a reduced vocabulary: tree_branch 41, the phi row does
    # not fit shared memory (global-phi quad kernel).
    "c5_k50k_small": {"corpus": {"family": G, "D": 6_000, "V": 5_000, "T": 2_000_000, "seed": 20161008},
                      "K": 50_000, "seed": 42, "iterations": 3, "chunks": 32, "workers": 8},
}
