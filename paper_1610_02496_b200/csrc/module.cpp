// module.cpp -- pybind11 `_core`: the reference's Python surface
// (proj/bindings/module.cpp:59-172, proj/python/sparselda/__init__.py) over the
// B200 engine, plus device-introspection extras used by tests and bench.py.
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <cstring>
#include <fstream>
#include <sstream>

#include "sparselda_b200.hpp"

namespace py = pybind11;
using namespace sparselda_b200;

namespace {

template <class T>
py::array_t<T> matrix(const std::vector<T>& v, std::size_t rows, std::size_t cols) {
    py::array_t<T> out({rows, cols});
    std::memcpy(out.mutable_data(), v.data(), v.size() * sizeof(T));
    return out;
}

template <class T>
py::array_t<T> vec(const std::vector<T>& v) {
    py::array_t<T> out(v.size());
    if (!v.empty()) std::memcpy(out.mutable_data(), v.data(), v.size() * sizeof(T));
    return out;
}

Corpus corpus_from_arrays(std::uint32_t num_docs, std::uint32_t vocab_size,
                          py::array_t<std::uint32_t, py::array::c_style | py::array::forcecast> doc,
                          py::array_t<std::uint32_t, py::array::c_style | py::array::forcecast> word,
                          py::object topic) {
    if (doc.size() != word.size()) throw ValidationError("doc and word arrays differ in length");
    Corpus c;
    c.num_docs = num_docs;
    c.vocab_size = vocab_size;
    const auto n = static_cast<std::size_t>(doc.size());
    c.tokens.resize(n);
    const std::uint32_t* d = doc.data();
    const std::uint32_t* w = word.data();
    for (std::size_t i = 0; i < n; ++i) {
        if (d[i] >= num_docs) throw ValidationError("doc id out of range");
        if (w[i] >= vocab_size) throw ValidationError("word id out of range");
        c.tokens[i] = Token{d[i], w[i], kInvalidTopic};
    }
    if (!topic.is_none()) {
        auto t = py::array_t<std::uint32_t, py::array::c_style | py::array::forcecast>::ensure(topic);
        if (!t || static_cast<std::size_t>(t.size()) != n) throw ValidationError("topic array length mismatch");
        for (std::size_t i = 0; i < n; ++i) c.tokens[i].topic = t.data()[i];
    }
    c.finalize();
    return c;
}

py::dict kernel_times_dict(const slda_kernel_times& t) {
    py::dict d;
    d["reset_ms"] = t.reset_ms;
    d["sampler_ms"] = t.sampler_ms;
    d["ssc_ms"] = t.ssc_ms;
    d["colsum_ms"] = t.colsum_ms;
    d["phi_ms"] = t.phi_ms;
    d["join_ms"] = t.join_ms;
    d["total_ms"] = t.total_ms;
    d["sampler_row_entries"] = t.sampler_row_entries;
    d["launches"] = t.launches;
    d["exchange_ms"] = t.exchange_ms;
    d["exchange_bytes"] = t.exchange_bytes;
    d["zmove_ms"] = t.zmove_ms;
    return d;
}

py::dict info_dict(const slda_info& i) {
    py::dict d;
    d["num_docs"] = i.num_docs;
    d["vocab_size"] = i.vocab_size;
    d["num_topics"] = i.num_topics;
    d["iteration"] = i.iteration;
    d["num_tokens"] = i.num_tokens;
    d["doc_begin"] = i.doc_begin;
    d["doc_end"] = i.doc_end;
    d["rank"] = i.rank;
    d["world_size"] = i.world_size;
    d["alpha"] = i.alpha;
    d["beta"] = i.beta;
    d["seed"] = i.seed;
    d["num_segments"] = i.num_segments;
    d["num_units"] = i.num_units;
    d["doc_topic_nnz"] = i.doc_topic_nnz;
    d["device_bytes"] = i.device_bytes;
    d["doc_major"] = i.doc_major;
    d["padded_topics"] = i.padded_topics;
    static const char* kShapes[] = {"round", "quad512", "quad256", "global", "vanilla"};
    d["sampler_shape"] = i.sampler_shape < 5 ? kShapes[i.sampler_shape] : "unknown";
    d["num_chunks"] = i.num_chunks;
    d["streaming"] = i.streaming != 0;
    return d;
}

}  // namespace

PYBIND11_MODULE(_core, m) {
    m.doc() = "B200-native sparsity-aware LDA trainer (SaberLDA ESCA)";
    m.attr("__version__") = kVersion;

    py::register_exception<ValidationError>(m, "ValidationError", PyExc_ValueError);
    py::register_exception<IoError>(m, "IoError", PyExc_IOError);
    py::register_exception<DeviceError>(m, "DeviceError", PyExc_RuntimeError);

    py::class_<Corpus>(m, "Corpus")
        .def_static("from_text",
                    [](const std::string& docword, const std::string& vocab) {
                        std::istringstream d(docword), v(vocab);
                        return load_uci(d, v);
                    },
                    py::arg("docword"), py::arg("vocab"))
        .def_static("from_files",
                    [](const std::string& docword_path, const std::string& vocab_path) {
                        return load_uci_files(docword_path, vocab_path);
                    },
                    py::arg("docword_path"), py::arg("vocab_path"))
        .def_static("from_arrays", &corpus_from_arrays, py::arg("num_docs"), py::arg("vocab_size"),
                    py::arg("doc"), py::arg("word"), py::arg("topic") = py::none())
        .def_static("generate",
                    [](std::uint32_t family, std::uint32_t num_docs, std::uint32_t vocab_size,
                       std::uint64_t num_tokens, std::uint64_t seed, std::uint32_t latent_topics,
                       std::uint32_t threads) {
                        slda_gen_params p{};
                        p.family = family;
                        p.num_docs = num_docs;
                        p.vocab_size = vocab_size;
                        p.num_tokens = num_tokens;
                        p.seed = seed;
                        p.latent_topics = latent_topics;
                        p.threads = threads;
                        py::gil_scoped_release release;
                        return generate_corpus(p);
                    },
                    py::arg("family"), py::arg("num_docs"), py::arg("vocab_size"), py::arg("num_tokens"),
                    py::arg("seed") = 20161008, py::arg("latent_topics") = 100, py::arg("threads") = 0)
        .def_readonly("num_docs", &Corpus::num_docs)
        .def_readonly("vocab_size", &Corpus::vocab_size)
        .def_readonly("num_tokens", &Corpus::num_tokens)
        .def_readonly("vocab", &Corpus::vocab)
        .def("init_assignments", &init_assignments, py::arg("num_topics"), py::arg("seed"))
        .def("tokens",
             [](const Corpus& c) {
                 py::array_t<std::uint32_t> out({c.tokens.size(), static_cast<std::size_t>(3)});
                 if (!c.tokens.empty()) std::memcpy(out.mutable_data(), c.tokens.data(), c.tokens.size() * 12);
                 return out;
             })
        .def("doc_lengths", [](const Corpus& c) { return vec(c.doc_lengths); })
        .def("__repr__", [](const Corpus& c) {
            return "Corpus(D=" + std::to_string(c.num_docs) + ", V=" + std::to_string(c.vocab_size) +
                   ", T=" + std::to_string(c.num_tokens) + ")";
        });

    py::enum_<SamplerKind>(m, "SamplerKind")
        .value("SPARSE", SamplerKind::kSparse)
        .value("VANILLA", SamplerKind::kVanilla);

    py::class_<TrainConfig>(m, "TrainConfig")
        .def(py::init<>())
        .def_readwrite("num_topics", &TrainConfig::num_topics)
        .def_readwrite("alpha", &TrainConfig::alpha)
        .def_readwrite("beta", &TrainConfig::beta)
        .def_readwrite("iterations", &TrainConfig::iterations)
        .def_readwrite("num_chunks", &TrainConfig::num_chunks)
        .def_readwrite("num_workers", &TrainConfig::num_workers)
        .def_readwrite("seed", &TrainConfig::seed)
        .def_readwrite("memory_budget", &TrainConfig::memory_budget)
        .def_readwrite("device_budget", &TrainConfig::device_budget)
        .def_readwrite("eval_every", &TrainConfig::eval_every)
        .def_readwrite("sampler", &TrainConfig::sampler)
        .def_readwrite("tree_branch", &TrainConfig::tree_branch)
        .def_readwrite("device", &TrainConfig::device);

    py::class_<IterationStats>(m, "IterationStats")
        .def_readonly("iteration", &IterationStats::iteration)
        .def_readonly("tokens", &IterationStats::tokens)
        .def_readonly("elapsed_s", &IterationStats::elapsed_s)
        .def_readonly("mtokens_per_s", &IterationStats::mtokens_per_s)
        .def_readonly("mean_doc_topics", &IterationStats::mean_doc_topics)
        .def_readonly("device_ms", &IterationStats::device_ms);

    py::class_<ModelState>(m, "Model")
        .def_readonly("num_docs", &ModelState::num_docs)
        .def_readonly("vocab_size", &ModelState::vocab_size)
        .def_readonly("num_tokens", &ModelState::num_tokens)
        .def_readonly("num_topics", &ModelState::num_topics)
        .def_readonly("alpha", &ModelState::alpha)
        .def_readonly("beta", &ModelState::beta)
        .def_readonly("iteration", &ModelState::iteration)
        .def("word_topic",
             [](const ModelState& s) { return matrix(s.word_topic(), s.vocab_size, s.num_topics); })
        .def("word_topic_prob",
             [](const ModelState& s) { return matrix(s.word_topic_prob(), s.vocab_size, s.num_topics); })
        .def("assignments",
             [](const ModelState& s, py::object out) -> py::object {
                 // gather_assignments (trainer.cpp:203-213), written straight into a numpy
                 // buffer (optionally a caller-provided, e.g. pinned, one).
                 if (!s.has_chunks()) throw ValidationError("model carries no chunks (loaded from a checkpoint)");
                 py::array_t<std::uint32_t, py::array::c_style> a;
                 if (out.is_none()) {
                     a = py::array_t<std::uint32_t>(static_cast<py::ssize_t>(s.num_tokens));
                 } else {
                     if (!py::array_t<std::uint32_t, py::array::c_style>::check_(out))
                         throw ValidationError("out must be a C-contiguous uint32 array");
                     a = py::reinterpret_borrow<py::array_t<std::uint32_t, py::array::c_style>>(out);
                     if (a.size() != static_cast<py::ssize_t>(s.num_tokens) || !a.writeable())
                         throw ValidationError("out must be a writeable uint32 array of num_tokens elements");
                 }
                 std::uint32_t* ptr = a.mutable_data();
                 {
                     py::gil_scoped_release release;
                     check(slda_get_assignments(s.engine(), ptr));
                 }
                 return a;
             },
             py::arg("out") = py::none())
        .def("run_iteration", &run_iteration, py::arg("config"), py::call_guard<py::gil_scoped_release>())
        .def("save", [](const ModelState& s, const std::string& path) { save_checkpoint(path, s); })
        .def_static("load",
                    [](const std::string& path, unsigned workers) {
                        return model_from_checkpoint(load_checkpoint(path), workers);
                    },
                    py::arg("path"), py::arg("workers") = 0)
        // Device-introspection extras.
        .def("tree_mass", [](const ModelState& s) { return vec(s.tree_mass()); })
        .def("tree_prefix",
             [](const ModelState& s) { return matrix(s.tree_prefix(), s.vocab_size, s.num_topics); })
        .def("doc_topic",
             [](const ModelState& s) {
                 const DocTopicMatrix a = s.doc_topic();
                 return py::make_tuple(vec(a.row_offsets), vec(a.topics), vec(a.counts));
             })
        .def("chunk_layout",
             [](const ModelState& s) {
                 const ChunkLayout c = s.chunk_layout();
                 py::dict d;
                 d["doc_range"] = py::make_tuple(c.doc_begin, c.doc_end);
                 d["sorted_doc"] = vec(c.sorted_doc);
                 d["sorted_word"] = vec(c.sorted_word);
                 d["token_ids"] = vec(c.token_ids);
                 d["shuffle_ptrs"] = vec(c.shuffle_ptrs);
                 d["doc_offsets"] = vec(c.doc_offsets);
                 d["seg_word"] = vec(c.seg_word);
                 d["seg_offset"] = vec(c.seg_offset);
                 d["seg_length"] = vec(c.seg_length);
                 d["schedule"] = vec(c.schedule);
                 return d;
             })
        .def("kernel_times", [](const ModelState& s) { return kernel_times_dict(s.kernel_times()); })
        .def("kernel_times_avg",
             [](const ModelState& s, std::uint32_t last_n) {
                 slda_kernel_times t{};
                 check(slda_get_kernel_times_avg(s.engine(), last_n, &t));
                 return kernel_times_dict(t);
             },
             py::arg("last_n"))
        .def("info", [](const ModelState& s) { return info_dict(s.info()); })
        .def("iterate_async",
             [](ModelState& s) { check(slda_iterate_async(s.engine())); },
             py::call_guard<py::gil_scoped_release>())
        .def("synchronize", [](ModelState& s) { check(slda_synchronize(s.engine())); },
             py::call_guard<py::gil_scoped_release>())
        .def("peer_handles",
             [](const ModelState& s) {
                 slda_peer_handles h{};
                 check(slda_peer_export(s.engine(), &h));
                 return py::bytes(reinterpret_cast<const char*>(&h), sizeof(h));
             })
        .def("peer_attach",
             [](ModelState& s, const std::vector<std::string>& all) {
                 std::vector<slda_peer_handles> hs(all.size());
                 for (std::size_t r = 0; r < all.size(); ++r) {
                     if (all[r].size() != sizeof(slda_peer_handles))
                         throw ValidationError("peer handles must be " + std::to_string(sizeof(slda_peer_handles)) +
                                               " bytes per rank");
                     std::memcpy(&hs[r], all[r].data(), sizeof(slda_peer_handles));
                 }
                 py::gil_scoped_release release;
                 check(slda_peer_attach(s.engine(), hs.data()));
             },
             py::arg("all_ranks"))
        .def("stream_ptr",
             [](const ModelState& s) { return reinterpret_cast<std::uintptr_t>(slda_stream(s.engine())); });

    m.def("init_state", &init_state, py::arg("corpus"), py::arg("config"),
          py::call_guard<py::gil_scoped_release>());
    m.def(
        "init_shard",
        [](const Corpus& corpus, const TrainConfig& cfg, std::uint32_t rank, std::uint32_t world) {
            py::gil_scoped_release release;
            return init_shard(corpus, cfg, rank, world);
        },
        py::arg("corpus"), py::arg("config"), py::arg("rank"), py::arg("world"));
    m.def("shard_bounds", [](const Corpus& c, std::uint32_t world) { return shard_bounds(c, world); },
          py::arg("corpus"), py::arg("world"));
    m.def(
        "shard_bounds_from_lengths",
        [](py::array_t<std::uint32_t, py::array::c_style | py::array::forcecast> lengths, std::uint32_t world) {
            std::uint64_t T = 0;
            for (py::ssize_t i = 0; i < lengths.size(); ++i) T += lengths.data()[i];
            std::vector<std::uint32_t> b(static_cast<std::size_t>(world) + 1);
            check(slda_shard_bounds(static_cast<std::uint32_t>(lengths.size()), T, lengths.data(), world, b.data()));
            return b;
        },
        py::arg("doc_lengths"), py::arg("world"));
    // Engine over a (T, 3) uint32 token array (sparselda::Token layout) of one document shard.
    m.def(
        "init_view",
        [](py::array_t<std::uint32_t, py::array::c_style> tokens, std::uint32_t num_docs, std::uint32_t vocab_size,
           std::uint32_t doc_begin, std::uint32_t doc_end, std::uint64_t token_id_base, const TrainConfig& cfg,
           std::uint32_t rank, std::uint32_t world, std::uint32_t init_mode) {
            if (tokens.ndim() != 2 || tokens.shape(1) != 3) throw ValidationError("tokens must be (T, 3) uint32");
            slda_corpus_view v{};
            v.num_docs = num_docs;
            v.vocab_size = vocab_size;
            v.num_tokens = static_cast<std::uint64_t>(tokens.shape(0));
            v.tokens = tokens.data();
            v.doc_begin = doc_begin;
            v.doc_end = doc_end;
            v.token_id_base = token_id_base;
            py::gil_scoped_release release;
            return init_view(v, cfg, rank, world, init_mode);
        },
        py::arg("tokens"), py::arg("num_docs"), py::arg("vocab_size"), py::arg("doc_begin"), py::arg("doc_end"),
        py::arg("token_id_base"), py::arg("config"), py::arg("rank") = 0, py::arg("world") = 1,
        py::arg("init_mode") = 0);
    // Synthetic corpora as raw (T, 3) arrays (bench.py): whole corpus or a document range.
    m.def(
        "generate_tokens",
        [](std::uint32_t family, std::uint32_t num_docs, std::uint32_t vocab_size, std::uint64_t num_tokens,
           std::uint64_t seed, std::uint32_t doc_begin, std::int64_t doc_end, std::uint32_t threads) {
            slda_gen_params p{};
            p.family = family;
            p.num_docs = num_docs;
            p.vocab_size = vocab_size;
            p.num_tokens = num_tokens;
            p.seed = seed;
            p.threads = threads;
            const std::uint32_t e = doc_end < 0 ? num_docs : static_cast<std::uint32_t>(doc_end);
            std::vector<std::uint32_t> len(num_docs);
            check(slda_generate_doc_lengths(&p, len.data()));
            std::uint64_t n = 0;
            for (std::uint32_t d = doc_begin; d < e && d < num_docs; ++d) n += len[d];
            py::array_t<std::uint32_t> out({static_cast<std::size_t>(n), static_cast<std::size_t>(3)});
            std::uint32_t* ptr = out.mutable_data();
            {
                py::gil_scoped_release release;
                check(slda_generate_docs(&p, doc_begin, e, ptr, n));
            }
            py::array_t<std::uint32_t> lens(len.size());
            std::memcpy(lens.mutable_data(), len.data(), len.size() * 4);
            return py::make_tuple(out, lens);
        },
        py::arg("family"), py::arg("num_docs"), py::arg("vocab_size"), py::arg("num_tokens"),
        py::arg("seed") = 20161008, py::arg("doc_begin") = 0, py::arg("doc_end") = -1, py::arg("threads") = 0);
    m.def(
        "train", [](const Corpus& corpus, const TrainConfig& cfg) { return train(corpus, cfg); },
        py::arg("corpus"), py::arg("config"), py::call_guard<py::gil_scoped_release>());
    m.def(
        "resume",
        [](const Corpus& corpus, const std::string& path, const TrainConfig& cfg) {
            return resume_from_checkpoint(corpus, load_checkpoint(path), cfg);
        },
        py::arg("corpus"), py::arg("checkpoint"), py::arg("config"));
    m.def(
        "heldout_ll",
        [](ModelState& model, const Corpus& heldout, std::uint32_t burn_in, unsigned workers,
           std::uint64_t seed) {
            EvalReport r;
            {
                py::gil_scoped_release release;
                r = heldout_ll(model, heldout, burn_in, workers, seed);
            }
            return py::make_tuple(r.per_token_ll, r.tokens_evaluated);
        },
        py::arg("model"), py::arg("heldout"), py::arg("burn_in") = 20, py::arg("workers") = 1,
        py::arg("seed") = 0);
    m.def("top_words", &top_words, py::arg("model"), py::arg("n"));
    m.def("segmented_count", [](const std::vector<TopicId>& segment) {
        const SparseTopicRow r = segmented_count(segment);
        std::vector<std::pair<TopicId, std::uint32_t>> pairs;
        for (std::size_t i = 0; i < r.size(); ++i) pairs.emplace_back(r.topics[i], r.counts[i]);
        return pairs;
    });
    m.def(
        "prefix_search", [](const std::vector<double>& prefix, double x) { return prefix_search(prefix, x); },
        py::arg("prefix"), py::arg("x"));
    py::class_<WaryTree>(m, "WaryTree")
        .def(py::init([](const std::vector<double>& weights, std::uint32_t branch) {
                 return WaryTree(weights, branch);
             }),
             py::arg("weights"), py::arg("branch") = 32)
        .def_property_readonly("total", &WaryTree::total)
        .def_property_readonly("size", &WaryTree::size)
        .def("sample", &WaryTree::sample, py::arg("x"))
        .def("level2", &WaryTree::level2)
        .def("level3", &WaryTree::level3)
        .def("level4", &WaryTree::level4);
    m.def("format_metrics_line", [](const IterationStats& s, py::object ll) {
        MetricsEntry e;
        e.stats = s;
        if (!ll.is_none()) e.heldout_ll = ll.cast<double>();
        return format_metrics_line(e);
    }, py::arg("stats"), py::arg("heldout_ll") = py::none());
    m.def("abi_version", &slda_abi_version);
}
