"""The `sparselda` CLI (csrc/cli.cpp), mirroring the reference's CLI suite
(proj/tests/test_cli.cpp) and its tool (proj/tools/main.cpp): subcommands, outputs, manifest
replay, exit codes.  Usage and validation / io failures run on CPU (no engine is built before
they are raised); training, evaluation and topics run on the GPU, and the trained checkpoint is
compared byte for byte with the reference's own train() + save_checkpoint on the same files.
"""
import json
import subprocess
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parent.parent
CLI = REPO / "paper_1610_02496_b200" / "sparselda"


def run_cli(*args, env=None):
    import os

    e = dict(os.environ)
    for k in [k for k in e if k.startswith("SPARSELDA_")]:
        del e[k]
    e.update(env or {})
    p = subprocess.run([str(CLI), *map(str, args)], capture_output=True, text=True, env=e, timeout=600)
    return p.returncode, p.stdout, p.stderr


def write_uci(path_docword, path_vocab, D, V, mean_len, seed):
    """random_corpus-style (fixtures.cpp): uniform words, Poisson lengths; UCI triples in doc order."""
    rng = np.random.default_rng(seed)
    lines = []
    for d in range(D):
        n = max(1, int(rng.poisson(mean_len)))
        words, counts = np.unique(rng.integers(0, V, n), return_counts=True)
        lines += [f"{d + 1} {w + 1} {c}" for w, c in zip(words, counts)]
    Path(path_docword).write_text(f"{D}\n{V}\n{len(lines)}\n" + "\n".join(lines) + "\n")
    Path(path_vocab).write_text("".join(f"term{v}\n" for v in range(V)))


def read_uci_tokens(path_docword):
    """load_docword's token order (corpus.cpp:30-68): each triple expanded `count` times."""
    rows = Path(path_docword).read_text().split("\n")
    D, V = int(rows[0]), int(rows[1])
    doc, word = [], []
    for line in rows[3:]:
        if not line.strip():
            continue
        d, w, c = map(int, line.split())
        doc += [d - 1] * c
        word += [w - 1] * c
    return D, V, np.array(doc, np.uint32), np.array(word, np.uint32)


@pytest.fixture
def fx(tmp_path):
    write_uci(tmp_path / "docword.txt", tmp_path / "vocab.txt", 40, 25, 12.0, 1001)
    write_uci(tmp_path / "heldout.txt", tmp_path / "heldout_vocab.txt", 8, 25, 10.0, 1002)
    return tmp_path


def train_args(fx, out, *extra):
    return ["train", "--docword", fx / "docword.txt", "--vocab", fx / "vocab.txt", "--topics", 5, "--iters", 4,
            "--seed", 77, "--workers", 2, "--out", fx / out, *extra]


# ---------------------------------------------------------------- CPU ----
def test_cli_usage_and_parse_errors():
    rc, out, _ = run_cli("--help")
    assert rc == 0 and "train" in out and "topics" in out
    rc, out, _ = run_cli("train", "--help")
    assert rc == 0 and "--docword" in out and "SPARSELDA_DOCWORD" in out
    assert run_cli()[0] == 1                        # a subcommand is required
    assert run_cli("fit")[0] == 1                   # unknown subcommand
    assert run_cli("train", "--bogus", "1")[0] == 1  # unknown flag
    assert run_cli("train", "--topics")[0] == 1      # missing value
    assert run_cli("train", "--topics", "x")[0] == 1  # not a number
    assert run_cli("eval", "--model", "m.ckpt")[0] == 1  # --heldout is required


def test_cli_exit_codes_distinguish_validation_from_io(fx):
    """test_cli.cpp 'exit codes distinguish validation from io failures'."""
    rc, _, err = run_cli("train", "--docword", fx / "docword.txt", "--vocab", fx / "vocab.txt", "--topics", 0,
                         "--iters", 1, "--out", fx / "bad")
    assert rc == 1 and err.startswith("error: ")
    rc, _, err = run_cli("train", "--docword", "/nonexistent/docword.txt", "--vocab", fx / "vocab.txt",
                         "--topics", 3, "--out", fx / "bad2")
    assert rc == 2 and err.startswith("io error: ")
    rc, _, _ = run_cli("eval", "--model", "/nonexistent/model.ckpt", "--heldout", fx / "heldout.txt")
    assert rc == 2
    rc, _, _ = run_cli("topics", "--model", "/nonexistent/model.ckpt")
    assert rc == 2
    rc, _, err = run_cli("train", "--vocab", fx / "vocab.txt", "--topics", 3)
    assert rc == 1 and "requires --docword and --vocab" in err
    rc, _, _ = run_cli("train", "--docword", fx / "docword.txt", "--vocab", fx / "vocab.txt", "--topics", 3,
                       "--sampler", "gibbs", "--out", fx / "bad3")
    assert rc == 1
    rc, _, _ = run_cli("train", "--from-manifest", fx / "missing.json")
    assert rc == 2


def test_cli_env_fallbacks_feed_the_flags(fx):
    # SPARSELDA_DOCWORD / SPARSELDA_VOCAB stand in for the flags; the failure is then the
    # validation of --topics 0 (exit 1), not the missing-input check.
    rc, _, err = run_cli("train", "--topics", 0, env={"SPARSELDA_DOCWORD": str(fx / "docword.txt"),
                                                      "SPARSELDA_VOCAB": str(fx / "vocab.txt"),
                                                      "SPARSELDA_OUT": str(fx / "envrun")})
    assert rc == 1 and "requires --docword" not in err


# ---------------------------------------------------------------- GPU ----
@pytest.mark.gpu
def test_cli_train_writes_metrics_manifest_and_checkpoint(fx):
    rc, out, err = run_cli(*train_args(fx, "run1"))
    assert rc == 0, err
    assert out.startswith("trained ") and "K=5, 4 iterations" in out
    metrics = [l for l in (fx / "run1/metrics.log").read_text().splitlines() if l]
    assert len(metrics) == 4
    for line in metrics:
        it, elapsed, thr = line.split()[:3]
        int(it), float(elapsed), float(thr)
    m = json.loads((fx / "run1/manifest.json").read_text())
    assert m["command"] == "train" and m["config"]["topics"] == 5 and m["config"]["seed"] == 77
    assert m["inputs"]["heldout"] is None
    assert m["inputs"]["docword"]["digest"].startswith("0x") and len(m["inputs"]["docword"]["digest"]) == 18
    assert (fx / "run1/model.ckpt").exists()


@pytest.mark.gpu
def test_cli_default_alpha_recorded_as_50_over_k(fx):
    rc, _, err = run_cli("train", "--docword", fx / "docword.txt", "--vocab", fx / "vocab.txt", "--topics", 1000,
                         "--iters", 0, "--chunks", 1, "--seed", 5, "--out", fx / "alpha_run")
    assert rc == 0, err
    text = (fx / "alpha_run/manifest.json").read_text()
    assert '"alpha": 0.05' in text and '"seed": 5' in text


@pytest.mark.gpu
def test_cli_reruns_and_manifest_replay_are_byte_identical(fx):
    assert run_cli(*train_args(fx, "run_a"))[0] == 0
    assert run_cli(*train_args(fx, "run_b"))[0] == 0
    a = (fx / "run_a/model.ckpt").read_bytes()
    assert a == (fx / "run_b/model.ckpt").read_bytes()
    rc, _, err = run_cli("train", "--from-manifest", fx / "run_a/manifest.json", "--out", fx / "run_c")
    assert rc == 0, err
    assert a == (fx / "run_c/model.ckpt").read_bytes()


@pytest.mark.gpu
def test_cli_checkpoint_equals_reference_train(fx):
    """The CLI's model.ckpt is the reference's own train() + save_checkpoint on the same UCI files
    and seed (oracle/_ref), byte for byte."""
    from oracle_lib import RefModel, ref_available

    if not ref_available():
        pytest.skip("oracle/_ref not built")
    assert run_cli(*train_args(fx, "run_ref"))[0] == 0
    D, V, doc, word = read_uci_tokens(fx / "docword.txt")
    ref = RefModel(D, V, doc, word, None, K=5, seed=77, num_chunks=2, workers=2)
    for _ in range(4):
        ref.iterate()
    ref.save_checkpoint(str(fx / "ref.ckpt"))
    assert (fx / "run_ref/model.ckpt").read_bytes() == (fx / "ref.ckpt").read_bytes()


@pytest.mark.gpu
def test_cli_train_with_heldout_logs_ll(fx):
    rc, _, err = run_cli(*train_args(fx, "run_ho", "--heldout", fx / "heldout.txt", "--eval-every", 2))
    assert rc == 0, err
    lines = [l.split() for l in (fx / "run_ho/metrics.log").read_text().splitlines() if l]
    assert [len(f) for f in lines] == [3, 4, 3, 4]  # LL column every 2nd iteration
    assert all(float(f[3]) < 0 for f in lines if len(f) == 4)
    m = json.loads((fx / "run_ho/manifest.json").read_text())
    assert m["inputs"]["heldout"]["path"].endswith("heldout.txt")


@pytest.mark.gpu
def test_cli_eval_is_reproducible(fx):
    assert run_cli(*train_args(fx, "run_eval"))[0] == 0
    model = fx / "run_eval/model.ckpt"
    rc1, out1, _ = run_cli("eval", "--model", model, "--heldout", fx / "heldout.txt")
    rc2, out2, _ = run_cli("eval", "--model", model, "--heldout", fx / "heldout.txt")
    assert rc1 == rc2 == 0 and out1 == out2
    it, ll, toks = out1.split()
    assert int(it) == 4 and float(ll) < 0 and int(toks) > 0


@pytest.mark.gpu
def test_cli_topics_output(fx):
    assert run_cli(*train_args(fx, "run_topics"))[0] == 0
    model = fx / "run_topics/model.ckpt"
    rc, out, _ = run_cli("topics", "--model", model, "--top-n", 4, "--vocab", fx / "vocab.txt")
    assert rc == 0
    lines = [l for l in out.splitlines() if l]
    assert len(lines) == 5
    for line in lines:
        assert line.startswith("topic ") and line.count(":") == 5 and "term" in line
    rc, out, _ = run_cli("topics", "--model", model, "--top-n", 0)
    assert rc == 0 and len([l for l in out.splitlines() if l]) == 5
    assert run_cli("topics", "--model", model, "--top-n", 26)[0] == 1
    assert run_cli("topics", "--model", model, "--vocab", fx / "heldout_vocab.txt")[0] == 0  # 25 terms: ok
