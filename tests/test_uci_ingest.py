"""CPU: the multi-threaded UCI docword parser (sparselda_b200.cpp load_docword_buffer) against
the reference's own parser (corpus.cpp:30-68, run from oracle/_ref through ref_load_docword).

Every input -- well-formed files large enough to be split across all host threads, files cut
short, files with extra lines, CRLF line ends, signs, tabs, overflow, and one bad line planted
at many positions of a large file -- must give the same tokens in the same order, or the same
error message with the same line number (the first failing line in file order).
"""
import ctypes as C

import numpy as np
import pytest

from oracle_lib import ref_available, ref_lib

pytestmark = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built (make oracle)")


def _ref(text: str):
    lib = ref_lib()
    lib.ref_load_docword.argtypes = [C.c_char_p, C.c_uint64, C.c_void_p, C.c_uint64]
    lib.ref_load_docword.restype = C.c_int64
    raw = text.encode()
    n = lib.ref_load_docword(raw, len(raw), None, 0)
    if n < 0:
        return ("error", lib.ref_last_error().decode())
    out = np.zeros((max(n, 1), 3), np.uint32)
    lib.ref_load_docword(raw, len(raw), out.ctypes.data, n)
    return ("ok", out[:n, :2].copy())


def _ours(text: str, V: int):
    import paper_1610_02496_b200 as slda

    try:  # the vocab file must hold exactly V lines, V as the header says
        V = int(text.split("\n")[1])
    except (IndexError, ValueError):
        pass
    vocab = "".join(f"w{i}\n" for i in range(V))
    try:
        c = slda.Corpus.from_text(text, vocab)
    except ValueError as e:
        return ("error", str(e))
    t = c.tokens().reshape(-1, 3) if c.num_tokens else np.zeros((0, 3), np.uint32)
    return ("ok", t[:, :2].copy())


def _same(text: str, V: int):
    a, b = _ref(text), _ours(text, V)
    assert a[0] == b[0], (a[0], b[0], a[1] if a[0] == "error" else "", b[1] if b[0] == "error" else "")
    if a[0] == "error":
        assert a[1] == b[1]
    else:
        assert np.array_equal(a[1], b[1])


def _big(rng, D=3000, V=500, nnz=250_000):
    d = np.sort(rng.integers(1, D + 1, nnz))
    w = rng.integers(1, V + 1, nnz)
    n = rng.integers(1, 4, nnz)
    lines = [f"{a} {b} {c}" for a, b, c in zip(d, w, n)]
    return D, V, lines


@pytest.mark.parametrize("text", [
    "2\n3\n2\n1 1 2\n2 3 1\n",
    "2\n3\n2\n1 1 2\n2 3 1",            # no final newline
    "2\n3\n2\n1 1 2\r\n2 3 1\r\n",      # CRLF
    "2\n3\n2\n\t1\t1   2 \n 2 3 +1\n",  # tabs, padding, a sign
    "2\n3\n3\n1 1 2\n2 3 1\n",          # cut short
    "2\n3\n1\n1 1 2\n2 3 x\n",          # junk after the NNZ lines is never read
    "2\n3\n2\n1 1 2\n\n",               # empty entry line
    "2\n3\n2\n1 1 2\n2 3 1 4\n",        # trailing data
    "2\n3\n2\n1 1 2.5\n2 3 1\n",
    "2\n3\n2\n1 1 -2\n2 3 1\n",
    "2\n3\n2\n0 1 2\n2 3 1\n",
    "2\n3\n2\n1 4 2\n2 3 1\n",
    "2\n3\n2\n1 1 99999999999999999999\n2 3 1\n",  # overflow
    "2\n3\n0\n",
    "2\n3\n",
    "x\n3\n1\n1 1 1\n",
    "2\n3\n1 2\n1 1 1\n",
])
def test_small_inputs_match_reference(text):
    _same(text, 4)


def test_large_file_matches_reference_tokens():
    rng = np.random.default_rng(3)
    D, V, lines = _big(rng)
    _same(f"{D}\n{V}\n{len(lines)}\n" + "\n".join(lines) + "\n", V)
    # More lines than NNZ: the rest is never read.
    _same(f"{D}\n{V}\n{len(lines) - 1234}\n" + "\n".join(lines) + "\nnot an entry\n", V)
    # Fewer lines than NNZ: unexpected end of file at the first missing line.
    _same(f"{D}\n{V}\n{len(lines) + 5}\n" + "\n".join(lines) + "\n", V)


def test_first_bad_line_in_file_order_wins():
    rng = np.random.default_rng(4)
    D, V, lines = _big(rng, nnz=200_000)
    for pos in (0, 1, 777, 50_000, 99_999, 100_000, 150_001, 199_999):
        bad = list(lines)
        bad[pos] = "1 2"
        if pos + 60_000 < len(bad):
            bad[pos + 60_000] = f"{D + 1} 1 1"  # a later, different error
        _same(f"{D}\n{V}\n{len(bad)}\n" + "\n".join(bad) + "\n", V)
