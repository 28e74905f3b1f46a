"""ctypes binding of the raw C-ABI (include/saberlda.h) -> libsaberlda.so.

This is the binding a reference-side maintainer would add for an FFI caller
(see INTEGRATION.md); tests use it to exercise the boundary without the
C++/pybind layers.
"""
from __future__ import annotations

import ctypes as C
import re
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
HEADER = REPO / "include" / "saberlda.h"
LIB = REPO / "paper_1610_02496_b200" / "libsaberlda.so"


class CorpusView(C.Structure):
    _fields_ = [("num_docs", C.c_uint32), ("vocab_size", C.c_uint32), ("num_tokens", C.c_uint64),
                ("tokens", C.c_void_p), ("doc_begin", C.c_uint32), ("doc_end", C.c_uint32),
                ("token_id_base", C.c_uint64), ("token_ids", C.c_void_p)]


class Config(C.Structure):
    _fields_ = [("num_topics", C.c_uint32), ("alpha", C.c_double), ("beta", C.c_double),
                ("seed", C.c_uint64), ("tree_branch", C.c_uint32), ("init_mode", C.c_uint32),
                ("device", C.c_int32), ("rank", C.c_uint32), ("world_size", C.c_uint32),
                ("sampler", C.c_uint32), ("num_chunks", C.c_uint32), ("device_budget", C.c_uint64)]


class IterationStats(C.Structure):
    _fields_ = [("iteration", C.c_uint32), ("tokens", C.c_uint64), ("elapsed_s", C.c_double),
                ("mtokens_per_s", C.c_double), ("mean_doc_topics", C.c_double), ("device_ms", C.c_double)]


class Info(C.Structure):
    _fields_ = [("num_docs", C.c_uint32), ("vocab_size", C.c_uint32), ("num_topics", C.c_uint32),
                ("iteration", C.c_uint32), ("num_tokens", C.c_uint64), ("doc_begin", C.c_uint32),
                ("doc_end", C.c_uint32), ("rank", C.c_uint32), ("world_size", C.c_uint32),
                ("alpha", C.c_double), ("beta", C.c_double), ("seed", C.c_uint64),
                ("num_segments", C.c_uint32), ("num_units", C.c_uint32), ("doc_topic_nnz", C.c_uint64),
                ("device_bytes", C.c_uint64), ("doc_major", C.c_uint32), ("padded_topics", C.c_uint32),
                ("sampler_shape", C.c_uint32), ("num_chunks", C.c_uint32), ("streaming", C.c_uint32)]


class KernelTimes(C.Structure):
    _fields_ = [("reset_ms", C.c_double), ("sampler_ms", C.c_double), ("ssc_ms", C.c_double),
                ("colsum_ms", C.c_double), ("phi_ms", C.c_double), ("join_ms", C.c_double),
                ("total_ms", C.c_double), ("sampler_row_entries", C.c_uint64), ("launches", C.c_uint32),
                ("exchange_ms", C.c_double), ("exchange_bytes", C.c_uint64),
                ("zmove_ms", C.c_double)]


class GenParams(C.Structure):
    _fields_ = [("family", C.c_uint32), ("num_docs", C.c_uint32), ("vocab_size", C.c_uint32),
                ("num_tokens", C.c_uint64), ("latent_topics", C.c_uint32), ("zipf_s", C.c_double),
                ("doc_dirichlet", C.c_double), ("length_sigma", C.c_double), ("seed", C.c_uint64),
                ("threads", C.c_uint32)]


def header_symbols() -> list[str]:
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(slda_[a-z0-9_]+)\s*\(", text)))


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(str(LIB))
        L.slda_last_error.restype = C.c_char_p
        L.slda_abi_version.restype = C.c_uint32
        L.slda_create.argtypes = [C.POINTER(CorpusView), C.POINTER(Config), C.POINTER(C.c_void_p)]
        L.slda_destroy.argtypes = [C.c_void_p]
        L.slda_iterate.argtypes = [C.c_void_p, C.POINTER(IterationStats)]
        L.slda_iterate_async.argtypes = [C.c_void_p]
        L.slda_synchronize.argtypes = [C.c_void_p]
        L.slda_get_info.argtypes = [C.c_void_p, C.POINTER(Info)]
        L.slda_get_kernel_times.argtypes = [C.c_void_p, C.POINTER(KernelTimes)]
        L.slda_stream.argtypes = [C.c_void_p]
        L.slda_stream.restype = C.c_void_p
        for n in ("slda_get_word_topic", "slda_get_word_topic_prob", "slda_get_tree_mass",
                  "slda_get_tree_prefix", "slda_get_assignments"):
            getattr(L, n).argtypes = [C.c_void_p, C.c_void_p]
        L.slda_shard_bounds.argtypes = [C.c_uint32, C.c_uint64, C.c_void_p, C.c_uint32, C.c_void_p]
        L.slda_word_slice.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32] + [C.POINTER(C.c_uint32)] * 3
        L.slda_generate_corpus_size.argtypes = [C.POINTER(GenParams), C.POINTER(C.c_uint64)]
        L.slda_generate_corpus.argtypes = [C.POINTER(GenParams), C.c_void_p, C.c_uint64]
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != 0:
        raise RuntimeError(f"slda error {rc}: {lib().slda_last_error().decode()}")


class Engine:
    """Minimal RAII wrapper over slda_create / slda_iterate / getters."""

    def __init__(self, D, V, doc, word, K, seed=0, alpha=0.0, beta=0.01, topic=None, device=0):
        self.tokens = np.empty((len(doc), 3), np.uint32)
        self.tokens[:, 0], self.tokens[:, 1] = doc, word
        self.tokens[:, 2] = 0xFFFFFFFF if topic is None else topic
        self.V, self.K, self.T = V, K, len(doc)
        view = CorpusView(D, V, len(doc), self.tokens.ctypes.data, 0, D, 0, None)
        cfg = Config(K, alpha, beta, seed, 0, 0, device, 0, 1, 0)
        h = C.c_void_p()
        check(lib().slda_create(C.byref(view), C.byref(cfg), C.byref(h)))
        self.h = h

    def iterate(self) -> IterationStats:
        st = IterationStats()
        check(lib().slda_iterate(self.h, C.byref(st)))
        return st

    def _get(self, name, dtype, shape):
        out = np.empty(shape, dtype)
        check(getattr(lib(), name)(self.h, out.ctypes.data))
        return out

    def word_topic(self):
        return self._get("slda_get_word_topic", np.uint32, (self.V, self.K))

    def word_topic_prob(self):
        return self._get("slda_get_word_topic_prob", np.float32, (self.V, self.K))

    def assignments(self):
        return self._get("slda_get_assignments", np.uint32, (self.T,))

    def kernel_times(self) -> KernelTimes:
        t = KernelTimes()
        check(lib().slda_get_kernel_times(self.h, C.byref(t)))
        return t

    def __del__(self):
        if getattr(self, "h", None):
            lib().slda_destroy(self.h)
            self.h = None
