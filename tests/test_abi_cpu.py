"""CPU: the C-ABI library loads and exports every symbol include/saberlda.h
declares; host-only entry points (sharding, synthetic corpora) and the
pybind surface behave like the reference's, without touching a GPU."""
import ctypes as C

import numpy as np
import pytest

import abi
from oracle_lib import oracle_lib


def test_library_exports_every_declared_symbol():
    lib = abi.lib()
    syms = abi.header_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(lib, s)]
    assert missing == []
    assert lib.slda_abi_version() == 5


def test_shard_bounds_follow_chunk_boundaries():
    # corpus.cpp:103-121 via the C oracle restatement
    rng = np.random.default_rng(3)
    for _ in range(50):
        D = int(rng.integers(1, 300))
        lens = rng.integers(0, 50, size=D).astype(np.uint32)
        T = int(lens.sum())
        for n in sorted({1, 2, 3, 8, D}):
            if n > D:
                continue
            ours = np.zeros(n + 1, np.uint32)
            ref = np.zeros(n + 1, np.uint32)
            abi.check(abi.lib().slda_shard_bounds(D, T, lens.ctypes.data, n, ours.ctypes.data))
            assert oracle_lib().orc_chunk_boundaries(D, T, lens, n, ref) == 0
            assert ours.tolist() == ref.tolist()
    bad = np.zeros(3, np.uint32)
    assert abi.lib().slda_shard_bounds(1, 1, np.ones(1, np.uint32).ctypes.data, 2, bad.ctypes.data) == 1


@pytest.mark.parametrize("family", [0, 1])
def test_generator_is_deterministic_across_thread_counts(family):
    outs = []
    for threads in (1, 3, 8):
        p = abi.GenParams(family, 500, 700, 40_000, 0, 0.0, 0.0, 0.0, 123, threads)
        T = C.c_uint64()
        abi.check(abi.lib().slda_generate_corpus_size(C.byref(p), C.byref(T)))
        buf = np.empty((T.value, 3), np.uint32)
        abi.check(abi.lib().slda_generate_corpus(C.byref(p), buf.ctypes.data, T.value))
        outs.append(buf)
    assert all((o == outs[0]).all() for o in outs)
    toks = outs[0]
    if family == 0:
        assert len(toks) == 40_000  # exact T
    assert np.all(np.diff(toks[:, 0].astype(np.int64)) >= 0)  # doc-major
    assert toks[:, 1].max() < 700 and np.all(toks[:, 2] == 0xFFFFFFFF)
    assert np.all(np.bincount(toks[:, 0], minlength=500) >= 1)


def test_family_g_is_zipf_skewed():
    import paper_1610_02496_b200 as slda

    c = slda.Corpus.generate(0, 2000, 5000, 200_000, seed=20161008)
    freq = np.sort(np.bincount(c.tokens()[:, 1], minlength=5000))[::-1]
    # A mixture of 100 Zipf(1) topics over independent permutations: skewed, not flat.
    assert freq[0] > 8 * np.median(freq)


# ---- the reference's python smoke surface that needs no GPU (test_smoke.py) ----

def make_corpus(num_docs=30, vocab=20, seed=7):
    import random

    import paper_1610_02496_b200 as slda

    rng = random.Random(seed)
    cells = {}
    for d in range(1, num_docs + 1):
        for _ in range(rng.randint(4, 12)):
            w = rng.randint(1, vocab)
            cells[(d, w)] = cells.get((d, w), 0) + 1
    lines = [str(num_docs), str(vocab), str(len(cells))]
    lines += [f"{d} {w} {c}" for (d, w), c in sorted(cells.items())]
    return slda.Corpus.from_text("\n".join(lines) + "\n", "\n".join(f"word{i}" for i in range(vocab)) + "\n")


def test_api_names_match_reference():
    import paper_1610_02496_b200 as slda

    reference_all = ["Corpus", "IterationStats", "IoError", "Model", "SamplerKind", "TrainConfig",
                     "ValidationError", "WaryTree", "__version__", "heldout_ll", "prefix_search",
                     "segmented_count", "top_words", "train"]
    for name in reference_all:
        assert hasattr(slda, name), name
    cfg = slda.TrainConfig()
    assert (cfg.beta, cfg.iterations, cfg.num_chunks, cfg.memory_budget) == (0.01, 100, 0, 1 << 30)


def test_corpus_counts():
    c = make_corpus()
    assert (c.num_docs, c.vocab_size, len(c.vocab)) == (30, 20, 20)
    assert c.num_tokens > 0


def test_uci_parse_errors_are_value_errors():
    import paper_1610_02496_b200 as slda

    with pytest.raises(ValueError):
        slda.Corpus.from_text("1\n1\n1\nbogus\n", "a\n")
    with pytest.raises(ValueError, match="line 4"):
        slda.Corpus.from_text("2\n4\n1\n3 1 1\n", "a\nb\nc\nd\n")
    with pytest.raises(ValueError, match="wordID"):
        slda.Corpus.from_text("2\n4\n1\n1 5 1\n", "a\nb\nc\nd\n")
    with pytest.raises(ValueError, match="count"):
        slda.Corpus.from_text("2\n4\n1\n1 4 0\n", "a\nb\nc\nd\n")
    with pytest.raises(ValueError, match="line 5"):
        slda.Corpus.from_text("2\n4\n2\n1 1 1\n", "a\nb\nc\nd\n")
    with pytest.raises(ValueError):
        slda.Corpus.from_text("2\n4\n1\n1 1 1\n", "a\nb\n")
    with pytest.raises(IOError):
        slda.Corpus.from_files("/nonexistent/docword", "/nonexistent/vocab")
    c = slda.Corpus.from_text("3\n5\n6\n1 1 1\n1 5 1\n2 2 1\n2 5 1\n2 1 1\n3 3 3\n",
                              "apple\norange\niphone\nandroid\nscreen\n")
    assert (c.num_docs, c.vocab_size, c.num_tokens) == (3, 5, 8)
    assert c.doc_lengths().tolist() == [2, 3, 3]
    assert c.vocab[2] == "iphone"


def test_init_assignments_matches_oracle():
    import paper_1610_02496_b200 as slda

    c = make_corpus()
    c.init_assignments(12, 31337)
    toks = c.tokens()
    expect = [oracle_lib().orc_uniform_topic(31337, 0xFFFFFFFF, t, 12) for t in range(len(toks))]
    assert toks[:, 2].tolist() == expect
    with pytest.raises(ValueError):
        c.init_assignments(0, 1)


def test_wary_tree_matches_bisect():
    import bisect
    import math
    import random

    import paper_1610_02496_b200 as slda

    rng = random.Random(3)
    weights = [rng.random() for _ in range(500)]
    tree = slda.WaryTree(weights, branch=32)
    prefix, total = [], 0.0
    for w in weights:
        total += w
        prefix.append(total)
    assert math.isclose(tree.total, total, rel_tol=1e-12)
    for _ in range(2000):
        x = rng.random() * total
        assert tree.sample(x) == bisect.bisect_left(prefix, x)
    t3 = slda.WaryTree([2, 1, 1, 3, 1, 1, 2, 1, 0], 3)
    assert t3.level4() == [2, 3, 4, 7, 8, 9, 11, 12, 12] and t3.sample(7.5) == 4
    with pytest.raises(ValueError):
        slda.WaryTree([1.0] * 65, 4)


def test_segmented_count_and_prefix_search():
    import collections
    import random

    import paper_1610_02496_b200 as slda

    rng = random.Random(11)
    seg = [rng.randint(0, 30) for _ in range(400)]
    assert slda.segmented_count(seg) == sorted(collections.Counter(seg).items())
    assert [slda.prefix_search([0.25, 0.375, 0.75, 1.0], x) for x in (0.3, 0.0, 1.0)] == [1, 0, 3]
    with pytest.raises(ValueError):
        slda.prefix_search([0.5, 1.0], 1.5)


def test_config_validation_without_gpu():
    import paper_1610_02496_b200 as slda

    c = make_corpus()
    cfg = slda.TrainConfig()
    cfg.num_topics = 0
    with pytest.raises(ValueError):
        slda.train(c, cfg)
    cfg.num_topics = 40000  # beyond 32^3 (test_trainer.cpp:250-252)
    with pytest.raises(ValueError):
        slda.train(c, cfg)


def test_standalone_generator_equals_the_products():
    """oracle/libcorpusgen.so (bench.py's reference-arm workload) is the product's generator
    source compiled on its own: same lengths and tokens, whole corpus and a document range."""
    import paper_1610_02496_b200._core as core
    from oracle_lib import CorpusGen

    for family, D, V, T in ((0, 700, 900, 60_000), (1, 300, 250, 9_000)):
        gen = CorpusGen(family, D, V, T, seed=77)
        toks, lens = core.generate_tokens(family, D, V, T, seed=77)
        assert np.array_equal(gen.doc_lengths(), lens)
        assert np.array_equal(gen.docs(0, D), toks)
        part, _ = core.generate_tokens(family, D, V, T, seed=77, doc_begin=100, doc_end=250)
        assert np.array_equal(gen.docs(100, 250), part)
