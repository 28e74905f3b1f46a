"""GPU, BASELINE full size: size-independent invariants of the trained state.

The per-iteration digests pin the engine to the reference at sizes the reference finishes in
seconds (test_gpu_parity.py).  At C2 (NYTimes-shaped: D=300K, V=100K, T=100M, K=1K,
BASELINE.json configs[1]) the reference is too slow to run here, so after three iterations
every quantity that has an exact closed form is recomputed on the host from the engine's own
counts, with the reference's arithmetic:

* C_wk column sums == the histogram of the assignments; row sums == the word frequencies;
* C_dk rows: topics strictly ascending, counts >= 1, row sums == document lengths, and the
  rows equal per-document histograms of the assignments;
* phi == f32((C_wk + beta) / (C_k + V*beta)) in f64 (counts.cpp:37-63), bit for bit;
* L4 == the sequential f32 prefix of each phi row, Q == f32(alpha) * L4[K-1] (trainer.cpp:237-248).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_c2_invariants_after_three_iterations():
    import paper_1610_02496_b200 as slda
    import paper_1610_02496_b200._core as core

    D, V, T, K = 300_000, 100_000, 100_000_000, 1_000
    toks, _ = core.generate_tokens(0, D, V, T, seed=20161008)
    doc, word = toks[:, 0].astype(np.int64), toks[:, 1].astype(np.int64)
    cfg = slda.TrainConfig()
    cfg.num_topics = K
    cfg.seed = 42
    cfg.alpha = 0.0  # -> 50/K (trainer.cpp:18)
    cfg.beta = 0.01
    cfg.device = 0
    m = core.init_view(toks, D, V, 0, D, 0, cfg)
    for _ in range(3):
        m.run_iteration(cfg)

    z = m.assignments().astype(np.int64)
    assert z.shape == (T,) and z.min() >= 0 and z.max() < K
    B = m.word_topic().astype(np.int64)
    assert np.array_equal(B.sum(0), np.bincount(z, minlength=K))
    assert np.array_equal(B.sum(1), np.bincount(word, minlength=V))

    offs, tops, cnts = m.doc_topic()
    offs = offs.astype(np.int64)
    assert offs[0] == 0 and offs[-1] == len(tops) == m.info()["doc_topic_nnz"]
    assert cnts.min() >= 1
    lens = np.bincount(doc, minlength=D)
    row_sum = np.add.reduceat(cnts.astype(np.int64), offs[:-1]) if len(tops) else np.zeros(D, np.int64)
    row_sum[offs[:-1] == offs[1:]] = 0  # empty documents
    assert np.array_equal(row_sum, lens)
    first = np.zeros(len(tops), bool)
    first[offs[:-1][offs[:-1] < offs[1:]]] = True
    assert np.all(np.diff(tops.astype(np.int64))[~first[1:]] > 0)  # ascending within a row
    # Rows equal per-document histograms of the assignments (CSR of the (doc, topic) counts).
    key = np.unique(doc * K + z, return_counts=True)
    assert np.array_equal(key[0] % K, tops) and np.array_equal(key[1], cnts)

    beta = 0.01
    alpha = 50.0 / K
    colsum = B.sum(0).astype(np.float64)
    phi = ((B.astype(np.float64) + beta) / (colsum + V * beta)).astype(np.float32)
    assert np.array_equal(m.word_topic_prob(), phi)
    l4 = np.cumsum(phi, axis=1, dtype=np.float32)
    assert np.array_equal(m.tree_prefix(), l4)
    assert np.array_equal(m.tree_mass(), np.float32(alpha) * l4[:, -1])
