"""CPU: pin the C oracle (oracle/slda_oracle.c) before trusting it.

1. Known-answer vectors the reference's own tests hold for this path
   (proj/tests/test_counts.cpp, test_sampler.cpp, test_corpus.cpp) and the
   Random123 Philox KATs the survey verified against the reference.
2. Per-iteration digests produced by the reference itself (oracle/_ref ->
   tests/golden/reference_digests.json, tests/golden/make_golden.py).
"""
import ctypes as C

import numpy as np
import pytest

from corpora import CASES, corpus_arrays
from oracle_lib import OracleModel, digest, oracle_lib, tokens_aos

RANDOM123 = {
    "zeros": ([0, 0, 0, 0], [0, 0], [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]),
    "ones": ([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2, [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]),
    "pi": ([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0],
           [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]),
}


@pytest.mark.parametrize("name", sorted(RANDOM123))
def test_philox_random123_kat(name, golden):
    ctr, key, expect = RANDOM123[name]
    out = np.zeros(4, np.uint32)
    oracle_lib().orc_philox(np.array(ctr, np.uint32), np.array(key, np.uint32), out)
    assert [int(x) for x in out] == expect
    assert golden["kats"]["philox"][name] == expect  # the reference agrees


def test_rng_stream_values(golden):
    u0, u1 = C.c_double(), C.c_double()
    oracle_lib().orc_uniform2(42, 0, 7, C.byref(u0), C.byref(u1))
    assert (u0.value, u1.value) == tuple(golden["kats"]["rng_42_0_7"])
    assert u0.value == 0.40588156361406069 and u1.value == 0.63216945057503438


def test_segmented_count_frozen_examples():
    # proj/tests/test_counts.cpp:62-73
    lib = oracle_lib()
    t, c = np.zeros(8, np.uint32), np.zeros(8, np.uint32)
    n = lib.orc_segmented_count(np.array([3, 1, 3, 2, 3], np.uint32), 5, t, c)
    assert (t[:n].tolist(), c[:n].tolist()) == ([1, 2, 3], [1, 1, 3])
    n = lib.orc_segmented_count(np.array([5, 5, 5, 5], np.uint32), 4, t, c)
    assert (t[:n].tolist(), c[:n].tolist()) == ([5], [4])
    assert lib.orc_segmented_count(np.zeros(1, np.uint32), 0, t, c) == 0


def test_preprocess_examples():
    # proj/tests/test_counts.cpp:14-29
    lib = oracle_lib()
    out = np.zeros(2, np.float32)
    assert lib.orc_preprocess(2, 1, np.array([1, 3], np.uint32), 0.01, out) == 0
    assert out[0] == np.float32(1.01 / 4.02) and out[1] == np.float32(3.01 / 4.02)
    out = np.zeros(24, np.float32)
    assert lib.orc_preprocess(8, 3, np.zeros(24, np.uint32), 0.5, out) == 0
    assert np.all(out == np.float32(0.125))
    assert lib.orc_preprocess(2, 2, np.zeros(4, np.uint32), 0.0, np.zeros(4, np.float32)) == -1


def test_wary_tree_worked_example():
    # proj/tests/test_sampler.cpp:69-86: 3-ary tree
    lib = oracle_lib()
    w = np.array([2, 1, 1, 3, 1, 1, 2, 1, 0], np.float64)
    n3, n4, total = C.c_uint32(), C.c_uint32(), C.c_double()
    lib.orc_wary_tree_d(w, 9, 3, None, None, None, C.byref(n3), C.byref(n4), C.byref(total))
    l2, l3, l4 = np.zeros(3), np.zeros(n3.value), np.zeros(n4.value)
    assert lib.orc_wary_tree_d(w, 9, 3, l2.ctypes.data, l3.ctypes.data, l4.ctypes.data, C.byref(n3),
                               C.byref(n4), C.byref(total)) == 0
    assert total.value == 12
    assert l4.tolist() == [2, 3, 4, 7, 8, 9, 11, 12, 12]
    assert l3[:3].tolist() == [4, 9, 12]
    assert lib.orc_wary_sample_d(l2, l3, l4, 9, 3, 12.0, 7.5) == 4
    assert lib.orc_wary_sample_d(l2, l3, l4, 9, 3, 12.0, 0.0) == 0


def test_tree_equals_lower_bound_many_widths():
    # acceptance.cpp:140-200 / test_sampler.cpp:113-134 -- the device uses lower_bound on L4.
    lib = oracle_lib()
    rng = np.random.default_rng(23)
    for W in (2, 3, 8, 32):
        for _ in range(10):
            K = int(rng.integers(1, min(W ** 3, 3000) + 1))
            w = np.where(rng.random(K) < 0.15, 0.0, rng.random(K))
            n3, n4, total = C.c_uint32(), C.c_uint32(), C.c_double()
            lib.orc_wary_tree_d(w, K, W, None, None, None, C.byref(n3), C.byref(n4), C.byref(total))
            l2, l3, l4 = np.zeros(W), np.zeros(n3.value), np.zeros(n4.value)
            lib.orc_wary_tree_d(w, K, W, l2.ctypes.data, l3.ctypes.data, l4.ctypes.data, C.byref(n3),
                                C.byref(n4), C.byref(total))
            for x in list(rng.random(60) * total.value) + [0.0, total.value]:
                lb = min(int(np.searchsorted(l4[:K], x, side="left")), K - 1)
                assert lib.orc_wary_sample_d(l2, l3, l4, K, W, total.value, x) == lb


def test_prefix_search_examples():
    # proj/tests/test_sampler.cpp:30-36, :59-64
    lib = oracle_lib()
    p = np.array([0.25, 0.375, 0.75, 1.0])
    assert [lib.orc_prefix_search_d(p, 4, x) for x in (0.3, 0.0, 1.0)] == [1, 0, 3]
    pf = np.array([0.5, 1.0], np.float32)
    assert lib.orc_prefix_search_f(pf, 2, np.nextafter(np.float32(1), np.float32(2))) == 1
    assert lib.orc_prefix_search_f(pf, 2, 1.5) == -1


def test_decomposition_fixture_distribution():
    # proj/tests/test_sampler.cpp:205-221: A_d = {0:2, 2:1}, alpha=.5, bhat=[.2,.3,.5]
    lib = oracle_lib()
    bhat = np.array([0.2, 0.3, 0.5], np.float32)
    l4 = np.zeros(3, np.float32)
    total = lib.orc_row_prefix(bhat, 3, l4)
    q = np.float32(0.5) * np.float32(total)
    law = np.array([0.357142857143, 0.107142857143, 0.535714285714])
    hist = np.zeros(3)
    u0, u1 = C.c_double(), C.c_double()
    for i in range(50_000):
        lib.orc_uniform2(99, 0, i, C.byref(u0), C.byref(u1))
        hist[lib.orc_sample_token(2, np.array([0, 2], np.uint32), np.array([2, 1], np.uint32), bhat,
                                  float(q), l4, 3, u0.value, u1.value)] += 1
    assert 0.5 * np.abs(hist / hist.sum() - law).sum() < 0.01


def test_pdow_stable_sort_example():
    # proj/tests/test_corpus.cpp:117-142 (one chunk here: same (word, doc, id) order)
    doc = np.array([0, 0, 1, 2], np.uint32)
    word = np.array([1, 0, 0, 2], np.uint32)
    m = OracleModel(3, 3, doc, word, np.zeros(4, np.uint32), K=1)
    p = m.pdow()
    assert p["sorted_word"].tolist() == [0, 0, 1, 2]
    assert p["sorted_doc"].tolist() == [0, 1, 0, 2]
    assert p["token_ids"].tolist() == [1, 2, 0, 3]
    assert p["doc_offsets"].tolist() == [0, 2, 3, 4]


@pytest.mark.parametrize("name", sorted(CASES))
def test_oracle_matches_reference_digests(name, golden):
    spec = CASES[name]
    fx = golden["cases"][name]
    doc, word, D, V = corpus_arrays(spec["corpus"])
    assert digest(np.stack([doc, word])) == fx["corpus_digest"], "generator drift"
    topic = None
    if spec.get("given_topics_seed") is not None:
        topic = np.random.default_rng(spec["given_topics_seed"]).integers(0, spec["K"], size=len(doc),
                                                                          dtype=np.uint32)
    m = OracleModel(D, V, doc, word, topic, K=spec["K"], alpha=spec.get("alpha", 0.0),
                    beta=spec.get("beta", 0.01), seed=spec["seed"], sampler=spec.get("sampler", "sparse"))
    assert m.alpha == fx["alpha"]
    iters = fx["iterations"]
    # Cheap cases: every iteration.  c1: every iteration too (50 x 100K tokens, ~2 s).
    for it, expect in enumerate(iters):
        got = m.digests()
        assert got == expect, (name, it, {k: v for k, v in got.items() if v != expect[k]})
        if it + 1 < len(iters):
            m.iterate()
            assert abs(m.mean_doc_topics() - fx["mean_doc_topics"][it]) == 0
    if "ll_curve" in fx:  # the last point of the curve: same model state as the run's end
        hd, hw, hD, _ = corpus_arrays(spec["heldout"])
        last = str(spec["iterations"])
        assert m.heldout_ll(hD, V, hd, hw, burn_in=20, seed=spec["seed"])[0] == fx["ll_curve"][last]
    if "heldout" in fx:
        hd, hw, hD, _ = corpus_arrays(spec["heldout"])
        ll, n = m.heldout_ll(hD, V, hd, hw, burn_in=20, seed=spec["seed"])
        assert n == fx["heldout"]["tokens"]
        assert ll == fx["heldout"]["per_token_ll"]


def test_oracle_rejects_like_reference():
    doc = np.array([0, 1], np.uint32)
    word = np.array([0, 1], np.uint32)
    with pytest.raises(ValueError):
        OracleModel(2, 2, doc, word, None, K=0)
    with pytest.raises(ValueError):  # topic >= K before any invalid (trainer.cpp:369-378)
        OracleModel(2, 2, doc, word, np.array([5, 0], np.uint32), K=3)
    # the first invalid topic ends the check: all redrawn
    OracleModel(2, 2, doc, word, np.array([0xFFFFFFFF, 9], np.uint32), K=3)
