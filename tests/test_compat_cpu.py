"""CPU: the source-compatible `sparselda` headers (paper_1610_02496_b200/compat/sparselda/).

A caller written against the reference's API compiles against them, and their host building
blocks (Philox RngStream, WaryTree<Real>, prefix_search, sample_token) reproduce the reference's
known answers -- no GPU needed (nothing here creates an engine).
"""
import subprocess
import textwrap
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parent.parent
PKG = REPO / "paper_1610_02496_b200"
INC = [f"-I{PKG / 'compat'}", f"-I{PKG / 'csrc'}", f"-I{REPO / 'include'}"]

CALLER = textwrap.dedent(r"""
    // A reference-API caller (the shapes acceptance.cpp / module.cpp use).
    #include <cstdio>
    #include <sstream>
    #include "sparselda/corpus.hpp"
    #include "sparselda/counts.hpp"
    #include "sparselda/eval.hpp"
    #include "sparselda/parallel.hpp"
    #include "sparselda/rng.hpp"
    #include "sparselda/sampler.hpp"
    #include "sparselda/trainer.hpp"
    using namespace sparselda;
    int train_something(const Corpus& corpus) {
        TrainConfig cfg;
        cfg.num_topics = 8;
        cfg.num_chunks = 2;
        ModelState state = init_state(corpus, cfg);
        run_iteration(state, cfg);
        std::uint64_t t = state.word_topic.total() + state.word_topic.row_total(0);
        ChunkSlot& slot = state.chunks.acquire(0);
        t += slot.doc_topic.row(0).counts.size() + slot.chunk.doc_begin;
        state.chunks.release(0);
        const HeldoutSet h = HeldoutSet::from_corpus(corpus);
        t += static_cast<std::uint64_t>(heldout_ll(state, h, 5, 1, 3).per_token_ll);
        t += state.trees[0].size() + static_cast<std::uint64_t>(state.tree_mass[0]);
        t += top_words(state.word_topic_prob, 1).size();
        save_checkpoint("/tmp/x.ckpt", state);
        const Checkpoint c = load_checkpoint("/tmp/x.ckpt");
        ModelState m2 = model_from_checkpoint(c, 1);
        t += m2.word_topic == c.word_topic;
        t += state.gather_assignments().size();
        return static_cast<int>(t);
    }
    int main() {
        // Random123 Philox4x32-10 known answers and the reference's RngStream(42, 0, 7).
        const auto o = philox::block({0, 0, 0, 0}, {0, 0});
        RngStream r(42, 0, 7);
        const double u0 = r.next_double(), u1 = r.next_double();
        std::printf("%08x %08x %08x %08x %.17g %.17g\n", o[0], o[1], o[2], o[3], u0, u1);
        // WaryTree == first->= search; prefix_search clamp.
        std::vector<float> w = {1, 0, 2, 0.5f, 0, 0, 3};
        WaryTree<float> tree(w, 2);
        const auto pre = tree.prefix();
        int bad = 0;
        for (float x = 0.0f; x <= tree.total(); x += 0.01f)
            bad += tree.sample(x) != prefix_search<float>(pre, x);
        // sample_token over a tiny row.
        SparseTopicRow row{{1, 3}, {2, 1}};
        std::vector<float> bhat = {0.1f, 0.2f, 0.3f, 0.4f};
        const auto built = build_tree<float>(bhat, 0.5f);
        std::vector<float> scratch;
        RngStream s(7, 1, 99);
        const TopicId k = sample_token<float>({row.topics, row.counts}, bhat, built.q, built.tree, s, scratch);
        std::printf("%d %u %zu\n", bad, k, segmented_count(std::vector<TopicId>{3, 1, 3, 2, 3}).size());
        return 0;
    }
""")


@pytest.fixture(scope="module")
def caller(tmp_path_factory):
    if not (PKG / "libsparselda_compat.so").exists():
        pytest.skip("libsparselda_compat.so not built")
    d = tmp_path_factory.mktemp("compat")
    src = d / "caller.cpp"
    src.write_text(CALLER)
    exe = d / "caller"
    subprocess.run(["g++", "-std=gnu++20", "-O1", *INC, str(src), "-o", str(exe), f"-L{PKG}",
                    "-lsparselda_compat", "-lsaberlda", f"-Wl,-rpath,{PKG}"], check=True)
    return exe


def test_reference_api_caller_compiles_and_host_blocks_match(caller):
    out = subprocess.run([str(caller)], capture_output=True, text=True, check=True).stdout.split("\n")
    # Random123 KAT (ctr 0, key 0) and RngStream(42, 0, 7).
    assert out[0] == "6627e8d5 e169c58d bc57ac4c 9b00dbd8 0.40588156361406069 0.63216945057503438"
    bad, topic, nrow = out[1].split()
    assert bad == "0" and topic in {"0", "1", "2", "3"} and nrow == "3"
