"""GPU parity: the B200 engine against the reference, bit for bit.

Every case in tests/corpora.py is run through the product path (pybind ->
C++ shim -> C-ABI -> sm_100a kernels) and compared, at EVERY iteration, with
sha256 digests the reference itself produced (tests/golden/, made by
oracle/_ref): assignments, C_wk, phi, the tree's L4 prefix, Q and C_dk.
PDOW layouts are compared array-for-array with the C oracle.  Held-out LL is
compared with a stated tolerance (device log vs glibc log: |rel| <= 1e-12).
"""
import numpy as np
import pytest

from corpora import BIG_CASES, CASES, G, U, corpus_arrays
from oracle_lib import OracleModel, digest

pytestmark = pytest.mark.gpu

HELDOUT_REL_TOL = 1e-12  # only the f64 log() may differ from glibc by an ulp


def slda():
    import paper_1610_02496_b200 as m

    return m


def make_model(spec, iterations=None):
    """init_state through the public API (pybind -> C++ shim -> C-ABI)."""
    s = slda()
    doc, word, D, V = corpus_arrays(spec["corpus"])
    topic = None
    if spec.get("given_topics_seed") is not None:
        topic = np.random.default_rng(spec["given_topics_seed"]).integers(0, spec["K"], size=len(doc),
                                                                          dtype=np.uint32)
    corpus = s.Corpus.from_arrays(D, V, doc, word, topic)
    cfg = s.TrainConfig()
    cfg.num_topics = spec["K"]
    cfg.alpha = spec.get("alpha", 0.0)
    cfg.beta = spec.get("beta", 0.01)
    cfg.seed = spec["seed"]
    cfg.iterations = spec["iterations"] if iterations is None else iterations
    cfg.tree_branch = 32 if spec["K"] <= 32768 else 41  # as the reference run (oracle/ref_shim.cpp)
    if spec.get("sampler") == "vanilla":
        cfg.sampler = s.SamplerKind.VANILLA
    return s.init_state(corpus, cfg), cfg, corpus


def model_digests(m):
    offs, tops, cnts = m.doc_topic()
    return {
        "assignments": digest(m.assignments()),
        "word_topic": digest(m.word_topic()),
        "word_topic_prob": digest(m.word_topic_prob()),
        "l4": digest(m.tree_prefix()),
        "tree_mass": digest(m.tree_mass()),
        "doc_topic": digest(np.concatenate([offs.view(np.uint32), tops, cnts])),
    }


@pytest.mark.parametrize("name", sorted(CASES))
def test_engine_matches_reference_every_iteration(name, golden):
    spec = CASES[name]
    fx = golden["cases"][name]
    m, cfg, _ = make_model(spec)
    assert m.alpha == fx["alpha"]
    for it, expect in enumerate(fx["iterations"]):
        got = model_digests(m)
        assert got == expect, (name, it, sorted(k for k in got if got[k] != expect[k]))
        if it + 1 < len(fx["iterations"]):
            st = m.run_iteration(cfg)
            assert st.iteration == it + 1
            assert st.tokens == fx["T"]
            assert st.mean_doc_topics == fx["mean_doc_topics"][it]


@pytest.mark.parametrize("name", sorted(n for n, s in CASES.items() if s.get("pdow")))
def test_pdow_layout_matches_reference(name, golden):
    spec = CASES[name]
    m, _, _ = make_model(spec, iterations=0)
    lay = m.chunk_layout()
    doc, word, D, V = corpus_arrays(spec["corpus"])
    o = OracleModel(D, V, doc, word, None, K=spec["K"], seed=spec["seed"])
    p = o.pdow()
    for key in ("sorted_doc", "sorted_word", "shuffle_ptrs", "doc_offsets", "seg_word", "seg_offset",
                "seg_length"):
        assert np.array_equal(np.asarray(lay[key]), p[key].astype(np.asarray(lay[key]).dtype)), key
    assert np.array_equal(lay["token_ids"], p["token_ids"].astype(np.uint64))
    # build_schedule (corpus.cpp:200-210): stable by (length desc, word asc).
    order = sorted(range(len(p["seg_word"])), key=lambda s: (-int(p["seg_length"][s]), int(p["seg_word"][s])))
    assert lay["schedule"].tolist() == order
    # ... and the reference's own chunk arrays (digests from oracle/_ref) when it ran one chunk.
    if spec.get("chunks", 1) != 1:
        return
    ref = golden["cases"][name]["pdow"]
    assert digest(lay["sorted_doc"]) == ref["sorted_doc"]
    assert digest(lay["sorted_word"]) == ref["sorted_word"]
    assert digest(lay["token_ids"].astype(np.uint32)) == ref["token_ids"]
    assert digest(lay["shuffle_ptrs"]) == ref["shuffle_ptrs"]
    assert digest(lay["doc_offsets"]) == ref["doc_offsets"]


@pytest.mark.parametrize("name", sorted(n for n, s in CASES.items() if s.get("heldout")))
def test_heldout_ll_matches_reference(name, golden):
    spec = CASES[name]
    fx = golden["cases"][name]
    m, cfg, _ = make_model(spec)
    for _ in range(spec["iterations"]):
        m.run_iteration(cfg)
    hd, hw, hD, V = corpus_arrays(spec["heldout"])
    held = slda().Corpus.from_arrays(hD, V, hd, hw)
    ll, n = slda().heldout_ll(m, held, burn_in=20, workers=1, seed=spec["seed"])
    assert n == fx["heldout"]["tokens"]
    ref = fx["heldout"]["per_token_ll"]
    assert abs(ll - ref) <= HELDOUT_REL_TOL * abs(ref), (ll, ref)


def test_heldout_ll_curve_tracks_reference(golden):
    """North star: the per-iteration log-likelihood tracks the reference over the full run
    (C1, 50 iterations, held-out LL every 5 iterations, |rel| <= 1e-12)."""
    spec = CASES["c1"]
    curve = golden["cases"]["c1"]["ll_curve"]
    m, cfg, _ = make_model(spec)
    hd, hw, hD, V = corpus_arrays(spec["heldout"])
    held = slda().Corpus.from_arrays(hD, V, hd, hw)
    for it in range(1, spec["iterations"] + 1):
        m.run_iteration(cfg)
        if str(it) in curve:
            ll, _ = slda().heldout_ll(m, held, burn_in=20, workers=1, seed=spec["seed"])
            assert abs(ll - curve[str(it)]) <= HELDOUT_REL_TOL * abs(curve[str(it)]), (it, ll, curve[str(it)])


def test_device_draws_pass_chi_square():
    """Acceptance criterion 1 (acceptance.cpp:48-135) on device draws: one document of one
    word, so every token of an iteration draws from the same law
    p(k) ~ (A_dk + alpha) * bhat_k; the histogram of the new topics must pass chi-square
    (z = 3.09, cells < 5 pooled) against the enumerated law."""
    s = slda()
    K, T = 24, 200_000
    doc = np.zeros(T, np.uint32)
    word = np.zeros(T, np.uint32)
    corpus = s.Corpus.from_arrays(1, 2, doc, word)
    cfg = s.TrainConfig()
    cfg.num_topics = K
    cfg.seed = 99
    m = s.init_state(corpus, cfg)
    offs, tops, cnts = m.doc_topic()
    bhat = m.word_topic_prob()[0].astype(np.float64)
    a = np.zeros(K)
    a[tops] = cnts
    law = (a + m.alpha) * bhat
    law /= law.sum()
    m.run_iteration(cfg)
    hist = np.bincount(m.assignments(), minlength=K).astype(np.float64)
    expected = law * T
    small = expected < 5
    stat = (((hist[~small] - expected[~small]) ** 2) / expected[~small]).sum()
    cells = int((~small).sum())
    if small.any():
        stat += (hist[small].sum() - expected[small].sum()) ** 2 / expected[small].sum()
        cells += 1
    df = max(cells - 1, 1)
    h = 2.0 / (9.0 * df)
    critical = df * (1 - h + 3.09 * np.sqrt(h)) ** 3  # Wilson-Hilferty, oracles.cpp:46-84
    assert stat <= critical, (stat, critical)


def test_async_iterations_equal_sync():
    spec = CASES["u_k64"]
    a, cfg, _ = make_model(spec)
    b, _, _ = make_model(spec)
    for _ in range(3):
        a.run_iteration(cfg)
        b.iterate_async()
    b.synchronize()
    assert model_digests(a) == model_digests(b)


def test_raw_c_abi_round_trip(golden):
    import abi

    spec = CASES["u_k7_chunks"]
    doc, word, D, V = corpus_arrays(spec["corpus"])
    e = abi.Engine(D, V, doc, word, spec["K"], seed=spec["seed"])
    for it in range(spec["iterations"]):
        st = e.iterate()
        assert st.iteration == it + 1 and st.device_ms > 0
    exp = golden["cases"]["u_k7_chunks"]["iterations"][-1]
    assert digest(e.assignments()) == exp["assignments"]
    assert digest(e.word_topic()) == exp["word_topic"]
    assert digest(e.word_topic_prob()) == exp["word_topic_prob"]
    t = e.kernel_times()
    assert t.sampler_ms > 0 and t.launches >= 5
    assert t.sampler_row_entries > 0


def test_sampler_kind_is_fixed_at_init():
    """The O(K) vanilla mode (SamplerKind.VANILLA) is chosen at init_state; an iteration asked
    for with the other kind is refused instead of running on the wrong doc-topic state."""
    s = slda()
    m, cfg, _ = make_model(CASES["vanilla_u_k300"], iterations=1)
    cfg.sampler = s.SamplerKind.SPARSE
    with pytest.raises(ValueError, match="sampler kind"):
        m.run_iteration(cfg)
    cfg.sampler = s.SamplerKind.VANILLA
    assert m.run_iteration(cfg).iteration == 1


def test_validation_errors_map_to_value_error():
    s = slda()
    doc, word, D, V = corpus_arrays(CASES["k1"]["corpus"])
    corpus = s.Corpus.from_arrays(D, V, doc, word)
    cfg = s.TrainConfig()
    cfg.num_topics = 70000
    cfg.tree_branch = 64
    with pytest.raises(ValueError, match="65536"):
        s.init_state(corpus, cfg)
    cfg = s.TrainConfig()
    cfg.num_topics = 3
    bad = s.Corpus.from_arrays(D, V, doc, word, np.full(len(doc), 7, np.uint32))
    with pytest.raises(ValueError, match="exceeds configured K"):
        s.init_state(bad, cfg)
    cfg.beta = 0.0
    with pytest.raises(ValueError):
        s.init_state(corpus, cfg)


def test_training_is_deterministic_and_normalized():
    s = slda()
    spec = CASES["alpha_beta"]
    a, cfg, _ = make_model(spec)
    b, _, _ = make_model(spec)
    for _ in range(3):
        a.run_iteration(cfg)
        b.run_iteration(cfg)
    assert (a.assignments() == b.assignments()).all()
    bhat = a.word_topic_prob().astype(np.float64)
    assert np.all(np.abs(bhat.sum(axis=0) - 1.0) < 1e-5)  # acceptance.cpp:281-303
    wt = a.word_topic()
    assert int(wt.sum()) == a.num_tokens
    ranked = s.top_words(a, 3)
    assert len(ranked) == a.num_topics and all(len(w) == 3 for w in ranked)


def test_checkpoint_roundtrip_and_resume(tmp_path):
    s = slda()
    spec = CASES["given_topics"]
    full, cfg, corpus = make_model(spec)
    for _ in range(4):
        full.run_iteration(cfg)
    half, _, _ = make_model(spec)
    for _ in range(2):
        half.run_iteration(cfg)
    path = str(tmp_path / "half.ckpt")
    half.save(path)
    loaded = s.Model.load(path)
    assert (loaded.word_topic() == half.word_topic()).all()
    assert (loaded.word_topic_prob() == half.word_topic_prob()).all()
    assert loaded.iteration == 2
    resumed = s.resume(corpus, path, cfg)
    for _ in range(2):
        resumed.run_iteration(cfg)
    assert (resumed.assignments() == full.assignments()).all()
    assert (resumed.word_topic() == full.word_topic()).all()
    text = open(path).read().splitlines()
    assert text[0].startswith("sparselda-checkpoint 1 ")
    assert len(text) == 1 + half.num_tokens + 1 + int((half.word_topic() != 0).sum())


@pytest.mark.parametrize("name,iters", [("given_topics", 2), ("c1", 5), ("k_large", 2), ("ssc_lengths", 3),
                                        ("ssc_lengths_k60k", 2)])
def test_checkpoint_bytes_equal_reference(name, iters, tmp_path):
    """Acceptance criterion 7's byte-identical checkpoints (acceptance.cpp:389-421) across the
    two engines: the device model's save() after N iterations is the same file, byte for byte, as
    the reference's own save_checkpoint (trainer.cpp:469-478, counts.cpp:140-150) after N
    iterations of the same corpus and seed (oracle/_ref)."""
    from oracle_lib import RefModel

    spec = CASES[name]
    m, cfg, _ = make_model(spec)
    doc, word, D, V = corpus_arrays(spec["corpus"])
    topic = None
    if spec.get("given_topics_seed") is not None:
        topic = np.random.default_rng(spec["given_topics_seed"]).integers(0, spec["K"], size=len(doc),
                                                                          dtype=np.uint32)
    ref = RefModel(D, V, doc, word, topic, K=spec["K"], alpha=spec.get("alpha", 0.0),
                   beta=spec.get("beta", 0.01), seed=spec["seed"], num_chunks=3, workers=2)
    for _ in range(iters):
        m.run_iteration(cfg)
        ref.iterate()
    ours, theirs = tmp_path / "device.ckpt", tmp_path / "reference.ckpt"
    m.save(str(ours))
    ref.save_checkpoint(str(theirs))
    assert ours.read_bytes() == theirs.read_bytes()


VARIANT_CASES = ["c1", "long_docs", "empty_docs", "k_large", "nytimes_small", "k1"]


@pytest.mark.parametrize("variant", ["SLDA_SAMPLER=round", "SLDA_SAMPLER=quad512", "SLDA_SAMPLER=quad256",
                                     "SLDA_SAMPLER=global", "SLDA_PHI_SHAPE=16x8", "SLDA_PHI_SHAPE=32x3",
                                     "SLDA_PHI_SHAPE=64x2", "SLDA_PHI_SHAPE=tma", "SLDA_ZMOVE=0",
                                     "SLDA_SAMPLER=quad512,SLDA_ASYNC_NEXT=0"])
@pytest.mark.parametrize("name", VARIANT_CASES)
def test_kernel_variants_match_reference(name, variant, golden, monkeypatch):
    """Every sampler launch shape (quad-lane 256/512-thread CTAs, the round-based kernel, the
    global-phi quad kernel) and every phi tile shape gives the reference's digests, whichever
    shape the default selection would pick for the case; SLDA_ZMOVE=0 stores the topics straight
    to z[slot] instead of through the z transpose; SLDA_ASYNC_NEXT=0 prefetches each round's first
    row line into registers instead of by cp.async.  The sampler shape and the z path are read when
    the engine is built (engine.cu), the phi shape at each launch."""
    for setting in variant.split(","):
        key, value = setting.split("=")
        monkeypatch.setenv(key, value)
    spec = CASES[name]
    fx = golden["cases"][name]
    m, cfg, _ = make_model(spec)
    iters = min(spec["iterations"], 6)
    for it in range(iters + 1):
        assert model_digests(m) == fx["iterations"][it], (name, variant, it)
        if it < iters:
            m.run_iteration(cfg)


# Default kernel selection per throughput case (sampler.cu launch_sampler): the shape the bench
# configs run.
BIG_SHAPES = {"c2_full": "quad256", "pubmed_k10k": "quad512", "c5_k50k_small": "global"}


@pytest.mark.parametrize("name", sorted(BIG_CASES))
def test_throughput_configs_match_reference_every_iteration(name, golden_big, monkeypatch):
    """BASELINE's throughput configs (C2 exactly; PubMed-shaped K=10,000 at 25M tokens; C5's
    K=50,000) against digests the reference itself produced, at every iteration, through the
    DEFAULT kernel selection: heavy words split into 8192-token units with in-CTA batch claiming,
    the 512-thread prefetching quad-lane kernel at K=10K, the global-phi kernel at K=50K."""
    for k in ("SLDA_SAMPLER", "SLDA_PHI_SHAPE", "SLDA_SERIAL", "SLDA_ZMOVE", "SLDA_ASYNC_NEXT"):
        monkeypatch.delenv(k, raising=False)
    spec = BIG_CASES[name]
    fx = golden_big["cases"][name]
    m, cfg, _ = make_model(spec)
    info = m.info()
    assert info["sampler_shape"] == BIG_SHAPES[name]
    if name != "c5_k50k_small":  # T = 2M: no word reaches the 8192-token unit cap
        assert info["num_units"] > info["num_segments"]  # some words were split (> 8192 tokens)
    for it, expect in enumerate(fx["iterations"]):
        got = model_digests(m)
        assert got == expect, (name, it, sorted(k for k in got if got[k] != expect[k]))
        if it + 1 < len(fx["iterations"]):
            st = m.run_iteration(cfg)
            assert st.mean_doc_topics == fx["mean_doc_topics"][it]


def test_acceptance_sublinear_scaling_in_k():
    """acceptance.cpp:306-342 (criterion 5) on the device: one sparse-sampler iteration grows
    by at most 4x from K=100 to K=3200, while the O(K) vanilla mode grows by more than 10x
    (device time of the iteration, median of 5 after 2 warm-ups; same corpus shape: 50K docs,
    V=20K, 64 tokens per document)."""
    s = slda()
    doc, word, D, V = corpus_arrays({"family": U, "D": 50_000, "V": 20_000, "T": 3_200_000, "seed": 5150})
    corpus = s.Corpus.from_arrays(D, V, doc, word)

    def iteration_ms(K, kind):
        cfg = s.TrainConfig()
        cfg.num_topics = K
        cfg.seed = 31
        cfg.sampler = kind
        m = s.init_state(corpus, cfg)
        for _ in range(2):
            m.run_iteration(cfg)
        return float(np.median([m.run_iteration(cfg).device_ms for _ in range(5)]))

    sparse = iteration_ms(3200, s.SamplerKind.SPARSE) / iteration_ms(100, s.SamplerKind.SPARSE)
    vanilla = iteration_ms(3200, s.SamplerKind.VANILLA) / iteration_ms(100, s.SamplerKind.VANILLA)
    print(f"K 100 -> 3200: sparse x{sparse:.2f}, vanilla x{vanilla:.1f}")
    assert sparse <= 4.0
    assert vanilla > 10.0


def _windowed_corpus(D, seed, V=8000, latent=20, window=400, dirichlet=0.08, mean_len=150.0):
    """The reference's topic-structured test fixture (tests/support/fixtures.cpp:69-104),
    restated with numpy's generator (same distribution, not the same draws): per document
    theta ~ Dirichlet(0.08) over 20 latent topics, length max(2, Poisson(150)), each token a
    latent topic ~ theta and a word uniform in that topic's disjoint 400-word window."""
    rng = np.random.default_rng(seed)
    stride = V // latent
    lens = np.maximum(2, rng.poisson(mean_len, D))
    theta = rng.gamma(dirichlet, 1.0, (D, latent))
    theta /= theta.sum(1, keepdims=True)
    doc = np.repeat(np.arange(D, dtype=np.uint32), lens)
    cdf = np.cumsum(theta, 1)[doc]
    topic = np.minimum((cdf < rng.random(len(doc))[:, None]).sum(1), latent - 1)
    word = ((topic * stride + rng.integers(0, window, len(doc))) % V).astype(np.uint32)
    return doc, word, D, V


def test_acceptance_convergence_sparse_vs_vanilla():
    """acceptance.cpp:344-385 (criterion 6) on the device: on the topic-structured fixture
    (20 latent topics with disjoint 400-word windows, 5000 documents of ~150 tokens, V=8000)
    the sparse sampler gains >= 1 nat of held-out per-token LL from iteration 1 to 50 at K=50,
    and the O(K) vanilla mode ends within 0.05 nats of it."""
    s = slda()
    doc, word, D, V = _windowed_corpus(5000, 101)
    hd, hw, hD, _ = _windowed_corpus(500, 202)
    corpus = s.Corpus.from_arrays(D, V, doc, word)
    held = s.Corpus.from_arrays(hD, V, hd, hw)

    def run(kind):
        cfg = s.TrainConfig()
        cfg.num_topics = 50
        cfg.seed = 4096
        cfg.sampler = kind
        m = s.init_state(corpus, cfg)
        first = None
        for i in range(1, 51):
            m.run_iteration(cfg)
            if i == 1:
                first = s.heldout_ll(m, held, burn_in=20, workers=2, seed=cfg.seed)[0]
        return first, s.heldout_ll(m, held, burn_in=20, workers=2, seed=cfg.seed)[0]

    sparse_first, sparse_last = run(s.SamplerKind.SPARSE)
    _, vanilla_last = run(s.SamplerKind.VANILLA)
    print(f"sparse LL {sparse_first:.4f} -> {sparse_last:.4f}; vanilla final {vanilla_last:.4f}")
    assert sparse_last - sparse_first >= 1.0
    assert abs(sparse_last - vanilla_last) <= 0.05


def test_acceptance_streaming_chunk_counts():
    """acceptance.cpp:424-445 (criterion 8): 1, 4 and 16 chunks give identical assignments.
    The device engine keeps one resident shard per GPU (num_chunks only sets the reference's
    streaming granularity), so the result must not depend on it -- and it equals the
    reference's own multi-chunk runs (u_k7_chunks, nytimes_small cases)."""
    s = slda()
    doc, word, D, V = corpus_arrays({"family": U, "D": 64, "V": 30, "T": 960, "seed": 808})
    corpus = s.Corpus.from_arrays(D, V, doc, word)
    out = []
    for chunks in (1, 4, 16):
        cfg = s.TrainConfig()
        cfg.num_topics = 8
        cfg.iterations = 3
        cfg.num_chunks = chunks
        cfg.num_workers = 2
        cfg.seed = 99
        out.append(s.train(corpus, cfg).assignments())
    assert np.array_equal(out[0], out[1]) and np.array_equal(out[0], out[2])


def test_failed_setups_release_device_memory():
    """A setup that fails validation after its scratch arena was reserved gives the memory back
    (the arena is normally released by a helper thread after a successful setup)."""
    import torch

    s = slda()
    doc, word, D, V = corpus_arrays(CASES["nytimes_small"]["corpus"])
    cfg = s.TrainConfig()
    cfg.num_topics = 3
    bad = s.Corpus.from_arrays(D, V, doc, word, np.full(len(doc), 7, np.uint32))
    free0 = torch.cuda.mem_get_info()[0]
    for _ in range(5):
        with pytest.raises(ValueError, match="exceeds configured K"):
            s.init_state(bad, cfg)
    torch.cuda.synchronize()
    assert torch.cuda.mem_get_info()[0] >= free0 - (64 << 20)
