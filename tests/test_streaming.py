"""GPU: out-of-core streaming (the reference's file-backed ChunkStore, trainer.cpp:65-198 and
:406-415, with the GPU's memory as the budget).

With TrainConfig.num_chunks > 1 and a corpus state above TrainConfig.device_budget, the engine
keeps each chunk's state (PDOW, topics, C_dk rows) in pinned host memory and passes the chunks
through the GPU once per iteration, C_wk accumulating over them before one M-step.  A budget of
1 byte forces that on test-sized corpora.  The result must be the reference's, bit for bit, at
every iteration (the reference's own chunk-count invariance, acceptance.cpp:426-445) -- against
the same golden digests the resident engine meets.
"""
import numpy as np
import pytest

from corpora import CASES
from test_gpu_parity import make_model, model_digests

pytestmark = pytest.mark.gpu


def streamed(spec, chunks):
    m, cfg, corpus = make_model(spec)
    s = __import__("paper_1610_02496_b200")
    cfg2 = s.TrainConfig()
    for k in ("num_topics", "alpha", "beta", "seed", "iterations", "tree_branch", "sampler"):
        setattr(cfg2, k, getattr(cfg, k))
    cfg2.num_chunks = chunks
    cfg2.device_budget = 1  # any real state exceeds it: stream
    del m
    return s.init_state(corpus, cfg2), cfg2


@pytest.mark.parametrize("name,chunks", [("c1", 4), ("shuffled", 3), ("empty_docs", 5), ("long_docs", 2),
                                         ("given_topics", 3), ("vanilla_c1", 3), ("k_global_phi", 2),
                                         ("ssc_lengths", 3), ("ssc_lengths_k60k", 2)])
def test_streamed_chunks_match_reference_every_iteration(name, chunks, golden):
    spec = CASES[name]
    fx = golden["cases"][name]
    m, cfg = streamed(spec, chunks)
    info = m.info()
    assert info["streaming"] and info["num_chunks"] == chunks
    iters = min(len(fx["iterations"]) - 1, 8)
    for it in range(iters + 1):
        got = model_digests(m)
        assert got == fx["iterations"][it], (name, it, sorted(k for k in got if got[k] != fx["iterations"][it][k]))
        if it < iters:
            st = m.run_iteration(cfg)
            assert st.tokens == fx["T"]
            assert st.mean_doc_topics == fx["mean_doc_topics"][it]


def test_streaming_only_when_over_budget():
    """The same chunk count with room on the device keeps one resident shard."""
    s = __import__("paper_1610_02496_b200")
    m, cfg, corpus = make_model(CASES["u_k64"])
    cfg.num_chunks = 4
    cfg.device_budget = 0  # the free device memory
    m2 = s.init_state(corpus, cfg)
    assert not m2.info()["streaming"] and m2.info()["num_chunks"] == 1


def test_streamed_heldout_ll_matches_resident():
    spec = CASES["c1"]
    s = __import__("paper_1610_02496_b200")
    m, cfg, corpus = make_model(spec)
    ms, cfg2 = streamed(spec, 4)
    for _ in range(3):
        m.run_iteration(cfg)
        ms.run_iteration(cfg2)
    doc, word = np.arange(60, dtype=np.uint32).repeat(20), (np.arange(1200, dtype=np.uint32) * 7) % 1000
    held = s.Corpus.from_arrays(60, 1000, doc, word)
    assert s.heldout_ll(m, held, burn_in=5, workers=1, seed=3) == s.heldout_ll(ms, held, burn_in=5, workers=1, seed=3)


@pytest.mark.parametrize("name,chunks", [("c1", 4), ("shuffled", 3), ("empty_docs", 5)])
def test_streamed_layout_is_the_single_chunk_layout(name, chunks):
    """chunk_layout() of a streaming engine merges its chunks into build_chunks(corpus, 1)'s
    arrays -- the same the resident engine (itself checked against the reference) returns."""
    spec = CASES[name]
    m, _, _ = make_model(spec, iterations=0)
    ms, _ = streamed(spec, chunks)
    a, b = m.chunk_layout(), ms.chunk_layout()
    for key in ("sorted_doc", "sorted_word", "token_ids", "shuffle_ptrs", "doc_offsets", "seg_word", "seg_offset",
                "seg_length", "schedule"):
        assert np.array_equal(np.asarray(a[key]), np.asarray(b[key])), key
    assert ms.info()["num_segments"] == m.info()["num_segments"]
