"""ctypes bindings for the CHECKERS (test infrastructure only).

* ``OracleModel`` -- oracle/liboracle.so, the plain-C restatement of the
  reference path (oracle/slda_oracle.c).
* ``RefModel``    -- oracle/_ref/libsparselda_ref.so, the unmodified reference
  sources compiled in place (oracle/Makefile) behind oracle/ref_shim.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/reference
legs may import this module.  The product never does.
"""
from __future__ import annotations

import ctypes as C
import hashlib
import os
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
ORACLE_SO = REPO / "oracle" / "liboracle.so"
REF_SO = REPO / "oracle" / "_ref" / "libsparselda_ref.so"
GEN_SO = REPO / "oracle" / "libcorpusgen.so"

_u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")


def digest(arr: np.ndarray) -> str:
    """sha256 of the raw little-endian bytes (bit-exact fingerprint)."""
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()[:32]


def tokens_aos(doc: np.ndarray, word: np.ndarray, topic: np.ndarray | None = None) -> np.ndarray:
    """(doc, word, topic) triples laid out exactly like sparselda::Token."""
    t = np.empty((len(doc), 3), dtype=np.uint32)
    t[:, 0] = doc
    t[:, 1] = word
    t[:, 2] = 0xFFFFFFFF if topic is None else topic
    return np.ascontiguousarray(t)


_oracle = None
_ref = None


def oracle_lib():
    global _oracle
    if _oracle is None:
        lib = C.CDLL(str(ORACLE_SO))
        lib.orc_philox.argtypes = [_u32p, _u32p, _u32p]
        lib.orc_uniform2.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.POINTER(C.c_double),
                                     C.POINTER(C.c_double)]
        lib.orc_uniform_topic.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint32]
        lib.orc_uniform_topic.restype = C.c_uint32
        lib.orc_chunk_boundaries.argtypes = [C.c_uint32, C.c_uint64, _u32p, C.c_uint32, _u32p]
        lib.orc_segmented_count.argtypes = [_u32p, C.c_uint32, _u32p, _u32p]
        lib.orc_segmented_count.restype = C.c_uint32
        lib.orc_preprocess.argtypes = [C.c_uint32, C.c_uint32, _u32p, C.c_double, _f32p]
        lib.orc_prefix_search_f.argtypes = [_f32p, C.c_uint64, C.c_float]
        lib.orc_prefix_search_f.restype = C.c_int64
        lib.orc_prefix_search_d.argtypes = [_f64p, C.c_uint64, C.c_double]
        lib.orc_prefix_search_d.restype = C.c_int64
        vp = C.c_void_p
        lib.orc_wary_tree_d.argtypes = [_f64p, C.c_uint32, C.c_uint32, vp, vp, vp,
                                        C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                        C.POINTER(C.c_double)]
        lib.orc_wary_sample_d.argtypes = [_f64p, _f64p, _f64p, C.c_uint32, C.c_uint32,
                                          C.c_double, C.c_double]
        lib.orc_wary_sample_d.restype = C.c_uint32
        lib.orc_row_prefix.argtypes = [_f32p, C.c_uint32, _f32p]
        lib.orc_row_prefix.restype = C.c_float
        lib.orc_sample_token.argtypes = [C.c_uint32, _u32p, _u32p, _f32p, C.c_float, _f32p,
                                         C.c_uint32, C.c_double, C.c_double]
        lib.orc_sample_token.restype = C.c_uint32
        lib.orc_init.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, _u32p, C.c_uint32,
                                 C.c_double, C.c_double, C.c_uint64, C.c_char_p, C.c_size_t]
        lib.orc_init.restype = C.c_void_p
        lib.orc_set_sampler.argtypes = [C.c_void_p, C.c_uint32]
        lib.orc_vanilla_token.argtypes = [C.c_uint32, _u32p, _u32p, _f32p, C.c_uint32, C.c_float,
                                          C.c_double]
        lib.orc_vanilla_token.restype = C.c_uint32
        lib.orc_free.argtypes = [C.c_void_p]
        lib.orc_iterate.argtypes = [C.c_void_p]
        lib.orc_iteration.argtypes = [C.c_void_p]
        lib.orc_iteration.restype = C.c_uint32
        lib.orc_alpha.argtypes = [C.c_void_p]
        lib.orc_alpha.restype = C.c_double
        lib.orc_get_word_topic.argtypes = [C.c_void_p, _u32p]
        lib.orc_get_word_topic_prob.argtypes = [C.c_void_p, _f32p]
        lib.orc_get_l4.argtypes = [C.c_void_p, _f32p]
        lib.orc_get_tree_mass.argtypes = [C.c_void_p, _f32p]
        lib.orc_get_assignments.argtypes = [C.c_void_p, _u32p]
        lib.orc_doc_topic_nnz.argtypes = [C.c_void_p]
        lib.orc_doc_topic_nnz.restype = C.c_uint64
        lib.orc_get_doc_topic.argtypes = [C.c_void_p, _u64p, _u32p, _u32p]
        lib.orc_mean_doc_topics.argtypes = [C.c_void_p]
        lib.orc_mean_doc_topics.restype = C.c_double
        lib.orc_num_segments.argtypes = [C.c_void_p]
        lib.orc_num_segments.restype = C.c_uint32
        lib.orc_get_pdow.argtypes = [C.c_void_p] + [_u32p] * 8
        lib.orc_heldout_ll.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint64, _u32p,
                                       C.c_uint32, C.c_uint64, C.POINTER(C.c_double),
                                       C.POINTER(C.c_uint64)]
        _oracle = lib
    return _oracle


def ref_available() -> bool:
    return REF_SO.exists()


def ref_lib():
    global _ref
    if _ref is None:
        lib = C.CDLL(str(REF_SO))
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_philox.argtypes = [_u32p, _u32p, _u32p]
        lib.ref_uniform2.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.POINTER(C.c_double),
                                     C.POINTER(C.c_double)]
        lib.ref_init.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, _u32p, C.c_uint32,
                                 C.c_double, C.c_double, C.c_uint64, C.c_uint32, C.c_uint32]
        lib.ref_init.restype = C.c_void_p
        lib.ref_init_sampler.argtypes = lib.ref_init.argtypes + [C.c_uint32]
        lib.ref_init_sampler.restype = C.c_void_p
        lib.ref_free.argtypes = [C.c_void_p]
        lib.ref_iterate.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        for name in ("ref_num_workers", "ref_num_chunks"):
            getattr(lib, name).argtypes = [C.c_void_p]
            getattr(lib, name).restype = C.c_uint32
        lib.ref_alpha.argtypes = [C.c_void_p]
        lib.ref_alpha.restype = C.c_double
        lib.ref_get_word_topic.argtypes = [C.c_void_p, _u32p]
        lib.ref_get_word_topic_prob.argtypes = [C.c_void_p, _f32p]
        lib.ref_get_l4.argtypes = [C.c_void_p, _f32p]
        lib.ref_get_tree_mass.argtypes = [C.c_void_p, _f32p]
        lib.ref_get_assignments.argtypes = [C.c_void_p, _u32p]
        lib.ref_doc_topic_nnz.argtypes = [C.c_void_p]
        lib.ref_doc_topic_nnz.restype = C.c_uint64
        lib.ref_get_doc_topic.argtypes = [C.c_void_p, _u64p, _u32p, _u32p]
        lib.ref_chunk_size.argtypes = [C.c_void_p, C.c_uint32]
        lib.ref_chunk_size.restype = C.c_uint32
        lib.ref_chunk_segments.argtypes = [C.c_void_p, C.c_uint32]
        lib.ref_chunk_segments.restype = C.c_uint32
        lib.ref_get_chunk.argtypes = [C.c_void_p, C.c_uint32] + [_u32p] * 9
        lib.ref_save_checkpoint.argtypes = [C.c_void_p, C.c_char_p]
        lib.ref_heldout_ll.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint64, _u32p,
                                       C.c_uint32, C.c_uint32, C.c_uint64,
                                       C.POINTER(C.c_double), C.POINTER(C.c_uint64)]
        lib.ref_segmented_count.argtypes = [_u32p, C.c_uint32, _u32p, _u32p]
        lib.ref_segmented_count.restype = C.c_uint32
        lib.ref_preprocess.argtypes = [C.c_uint32, C.c_uint32, _u32p, C.c_double, _f32p]
        lib.ref_sample_token.argtypes = [C.c_uint32, _u32p, _u32p, _f32p, C.c_uint32, C.c_float,
                                         C.c_uint64, C.c_uint32, C.c_uint64]
        lib.ref_sample_token.restype = C.c_uint32
        _ref = lib
    return _ref


class _ModelBase:
    """Common getters; subclasses bind the prefix ('orc' or 'ref')."""

    def __init__(self, D, V, doc, word, topic, K, alpha, beta, seed):
        self.D, self.V, self.K = int(D), int(V), int(K)
        self.T = int(len(doc))
        self.tokens = tokens_aos(doc, word, topic)

    def word_topic(self):
        out = np.empty((self.V, self.K), np.uint32)
        self._call("get_word_topic", out)
        return out

    def word_topic_prob(self):
        out = np.empty((self.V, self.K), np.float32)
        self._call("get_word_topic_prob", out)
        return out

    def l4(self):
        out = np.empty((self.V, self.K), np.float32)
        self._call("get_l4", out)
        return out

    def tree_mass(self):
        out = np.empty(self.V, np.float32)
        self._call("get_tree_mass", out)
        return out

    def assignments(self):
        out = np.empty(self.T, np.uint32)
        self._call("get_assignments", out)
        return out

    def doc_topic(self):
        nnz = self._call("doc_topic_nnz")
        offs = np.empty(self.D + 1, np.uint64)
        tops = np.empty(max(nnz, 1), np.uint32)
        cnts = np.empty(max(nnz, 1), np.uint32)
        self._call("get_doc_topic", offs, tops, cnts)
        return offs, tops[:nnz], cnts[:nnz]

    def digests(self) -> dict:
        offs, tops, cnts = self.doc_topic()
        return {
            "assignments": digest(self.assignments()),
            "word_topic": digest(self.word_topic()),
            "word_topic_prob": digest(self.word_topic_prob()),
            "l4": digest(self.l4()),
            "tree_mass": digest(self.tree_mass()),
            "doc_topic": digest(np.concatenate([offs.view(np.uint32), tops, cnts])),
        }


class OracleModel(_ModelBase):
    def __init__(self, D, V, doc, word, topic=None, K=8, alpha=0.0, beta=0.01, seed=0,
                 sampler="sparse"):
        super().__init__(D, V, doc, word, topic, K, alpha, beta, seed)
        lib = oracle_lib()
        err = C.create_string_buffer(256)
        h = lib.orc_init(self.D, self.V, self.T, self.tokens.reshape(-1), self.K, alpha, beta,
                         seed, err, 256)
        if not h:
            raise ValueError(err.value.decode())
        self.h = h
        lib.orc_set_sampler(h, 1 if sampler == "vanilla" else 0)
        self.alpha = lib.orc_alpha(h)

    def _call(self, name, *args):
        return getattr(oracle_lib(), "orc_" + name)(self.h, *args)

    def iterate(self):
        if oracle_lib().orc_iterate(self.h) != 0:
            raise ValueError("oracle iteration failed")

    @property
    def iteration(self):
        return oracle_lib().orc_iteration(self.h)

    def mean_doc_topics(self):
        return oracle_lib().orc_mean_doc_topics(self.h)

    def pdow(self):
        lib = oracle_lib()
        ns = lib.orc_num_segments(self.h)
        T = max(self.T, 1)
        arrs = [np.empty(T, np.uint32) for _ in range(4)]
        doc_off = np.empty(self.D + 1, np.uint32)
        segs = [np.empty(max(ns, 1), np.uint32) for _ in range(3)]
        lib.orc_get_pdow(self.h, *arrs, doc_off, *segs)
        names = ["sorted_doc", "sorted_word", "token_ids", "shuffle_ptrs"]
        out = {n: a[: self.T] for n, a in zip(names, arrs)}
        out["doc_offsets"] = doc_off
        out["seg_word"], out["seg_offset"], out["seg_length"] = (s[:ns] for s in segs)
        return out

    def heldout_ll(self, D, V, doc, word, burn_in=20, seed=0):
        toks = tokens_aos(doc, word)
        ll = C.c_double()
        n = C.c_uint64()
        if oracle_lib().orc_heldout_ll(self.h, D, V, len(doc), toks.reshape(-1), burn_in, seed,
                                       C.byref(ll), C.byref(n)) != 0:
            raise ValueError("oracle heldout_ll failed")
        return ll.value, n.value

    def __del__(self):
        if getattr(self, "h", None):
            oracle_lib().orc_free(self.h)
            self.h = None


class RefModel(_ModelBase):
    """The reference itself (oracle/_ref)."""

    def __init__(self, D, V, doc, word, topic=None, K=8, alpha=0.0, beta=0.01, seed=0,
                 num_chunks=1, workers=1, sampler="sparse"):
        super().__init__(D, V, doc, word, topic, K, alpha, beta, seed)
        lib = ref_lib()
        h = lib.ref_init_sampler(self.D, self.V, self.T, self.tokens.reshape(-1), self.K, alpha, beta,
                                 seed, num_chunks, workers, 1 if sampler == "vanilla" else 0)
        if not h:
            raise ValueError(lib.ref_last_error().decode())
        self.h = h
        self.alpha = lib.ref_alpha(h)
        self.last_elapsed = None
        self.last_mean_doc_topics = None

    def _call(self, name, *args):
        return getattr(ref_lib(), "ref_" + name)(self.h, *args)

    def iterate(self):
        el = C.c_double()
        kd = C.c_double()
        if ref_lib().ref_iterate(self.h, C.byref(el), C.byref(kd)) != 0:
            raise ValueError(ref_lib().ref_last_error().decode())
        self.last_elapsed = el.value
        self.last_mean_doc_topics = kd.value

    @property
    def workers(self):
        return ref_lib().ref_num_workers(self.h)

    @property
    def chunks(self):
        return ref_lib().ref_num_chunks(self.h)

    def chunk(self, c: int):
        lib = ref_lib()
        n = lib.ref_chunk_size(self.h, c)
        ns = lib.ref_chunk_segments(self.h, c)
        rng = np.empty(2, np.uint32)
        arrs = [np.empty(max(n, 1), np.uint32) for _ in range(4)]
        tmp_off = np.empty(self.D + 1, np.uint32)  # chunk doc count <= D
        segs = [np.empty(max(ns, 1), np.uint32) for _ in range(3)]
        lib.ref_get_chunk(self.h, c, rng, *arrs, tmp_off, *segs)
        docs = int(rng[1] - rng[0])
        names = ["sorted_doc", "sorted_word", "token_ids", "shuffle_ptrs"]
        out = {k: a[:n] for k, a in zip(names, arrs)}
        out["doc_range"] = (int(rng[0]), int(rng[1]))
        out["doc_offsets"] = tmp_off[: docs + 1]
        out["seg_word"], out["seg_offset"], out["seg_length"] = (s[:ns] for s in segs)
        return out

    def save_checkpoint(self, path: str) -> None:
        if ref_lib().ref_save_checkpoint(self.h, str(path).encode()) != 0:
            raise ValueError(ref_lib().ref_last_error().decode())

    def heldout_ll(self, D, V, doc, word, burn_in=20, seed=0, workers=1):
        toks = tokens_aos(doc, word)
        ll = C.c_double()
        n = C.c_uint64()
        if ref_lib().ref_heldout_ll(self.h, D, V, len(doc), toks.reshape(-1), burn_in, workers,
                                    seed, C.byref(ll), C.byref(n)) != 0:
            raise ValueError(ref_lib().ref_last_error().decode())
        return ll.value, n.value

    def __del__(self):
        if getattr(self, "h", None):
            ref_lib().ref_free(self.h)
            self.h = None


class _GenParams(C.Structure):  # slda_gen_params (include/saberlda.h)
    _fields_ = [("family", C.c_uint32), ("num_docs", C.c_uint32), ("vocab_size", C.c_uint32),
                ("num_tokens", C.c_uint64), ("latent_topics", C.c_uint32), ("zipf_s", C.c_double),
                ("doc_dirichlet", C.c_double), ("length_sigma", C.c_double), ("seed", C.c_uint64),
                ("threads", C.c_uint32)]


class CorpusGen:
    """The synthetic-corpus generator built on its own (oracle/libcorpusgen.so, from
    paper_1610_02496_b200/csrc/corpus_gen.cpp): the workload of bench.py's reference arm,
    generated without loading the product's libraries."""

    def __init__(self, family, D, V, T, seed=20161008, latent_topics=100, threads=0):
        self.lib = C.CDLL(str(GEN_SO))
        self.lib.slda_gen_last_error.restype = C.c_char_p
        self.p = _GenParams(family=family, num_docs=D, vocab_size=V, num_tokens=T, latent_topics=latent_topics,
                            seed=seed, threads=threads)
        self.D = D

    def _check(self, rc):
        if rc != 0:
            raise ValueError(self.lib.slda_gen_last_error().decode())

    def doc_lengths(self) -> np.ndarray:
        out = np.empty(self.D, np.uint32)
        self._check(self.lib.slda_generate_doc_lengths(C.byref(self.p), out.ctypes.data_as(C.c_void_p)))
        return out

    def docs(self, doc_begin: int, doc_end: int, lengths: np.ndarray | None = None) -> np.ndarray:
        """(T, 3) tokens (doc, word, kInvalidTopic) of documents [doc_begin, doc_end)."""
        lens = self.doc_lengths() if lengths is None else lengths
        n = int(lens[doc_begin:doc_end].astype(np.int64).sum())
        out = np.empty((n, 3), np.uint32)
        self._check(self.lib.slda_generate_docs(C.byref(self.p), doc_begin, doc_end,
                                                out.ctypes.data_as(C.c_void_p), C.c_uint64(n)))
        return out


def random_corpus(num_docs: int, vocab: int, mean_len: float, seed: int):
    """Family-U style corpus (uniform words, Poisson lengths >= 1), doc-major.

    Same shape family as the reference fixture random_corpus
    (proj/tests/support/fixtures.cpp:50-67); numpy's generator, not mt19937.
    """
    rng = np.random.default_rng(seed)
    lens = np.maximum(1, rng.poisson(mean_len, size=num_docs)).astype(np.int64)
    doc = np.repeat(np.arange(num_docs, dtype=np.uint32), lens)
    word = rng.integers(0, vocab, size=len(doc), dtype=np.uint32)
    return doc, word
