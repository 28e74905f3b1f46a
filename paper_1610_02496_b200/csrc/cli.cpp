// cli.cpp -- the `sparselda` command-line tool over the B200 engine.
//
// Replaces the reference CLI (proj/tools/main.cpp) with the same subcommands, flags,
// environment variables, outputs and exit codes:
//   train  --docword --vocab --topics --alpha --beta --iters --chunks --workers --seed --heldout
//          --eval-every --burn-in --out --mem-budget --sampler --from-manifest   (main.cpp:257-291)
//          -> <out>/manifest.json (FNV-1a 64 input digests, main.cpp:22-38,157-183),
//             <out>/metrics.log (format_metrics_line per iteration), <out>/model.ckpt
//   eval   --model --heldout --burn-in --workers --seed                         (main.cpp:293-302)
//   topics --model --top-n --vocab                                              (main.cpp:304-308)
// Exit codes (main.cpp:310-325): 0 ok; 1 usage / ValidationError ("error: ..."); 2 IoError
// ("io error: ...").  The reference parses with CLI11 and writes the manifest with nlohmann::json;
// neither is in this image, so both are hand-written here: a flag parser with the same
// `--flag value` / `--flag=value` forms and env fallbacks, and a small JSON value with sorted keys
// and 2-space indentation (nlohmann's dump(2) layout, shortest round-trip doubles).
#include <cerrno>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <map>
#include <memory>
#include <optional>
#include <random>
#include <sstream>
#include <string>
#include <variant>
#include <vector>

#include "sparselda_b200.hpp"

namespace sl = sparselda_b200;

namespace {

struct UsageError : std::runtime_error {
    explicit UsageError(const std::string& m) : std::runtime_error(m) {}
};

// ------------------------------------------------------------------ JSON --
struct Json {
    using Object = std::map<std::string, Json>;  // sorted keys, as nlohmann::json's default map
    using Array = std::vector<Json>;
    std::variant<std::nullptr_t, bool, std::uint64_t, std::int64_t, double, std::string, Array, Object> v;

    Json() : v(nullptr) {}
    Json(std::nullptr_t) : v(nullptr) {}
    Json(bool b) : v(b) {}
    Json(double d) : v(d) {}
    Json(std::uint64_t u) : v(u) {}
    Json(std::uint32_t u) : v(static_cast<std::uint64_t>(u)) {}
    Json(std::int64_t i) : v(i) {}
    Json(const std::string& s) : v(s) {}
    Json(const char* s) : v(std::string(s)) {}
    Json(Object o) : v(std::move(o)) {}

    bool is_null() const { return std::holds_alternative<std::nullptr_t>(v); }
    bool contains(const std::string& k) const {
        const auto* o = std::get_if<Object>(&v);
        return o && o->count(k);
    }
    const Json& at(const std::string& k) const {
        const auto* o = std::get_if<Object>(&v);
        if (!o || !o->count(k)) throw sl::ValidationError("manifest: missing key \"" + k + "\"");
        return o->at(k);
    }
    Json& operator[](const std::string& k) {
        if (!std::holds_alternative<Object>(v)) v = Object{};
        return std::get<Object>(v)[k];
    }
    std::string str() const {
        if (const auto* s = std::get_if<std::string>(&v)) return *s;
        throw sl::ValidationError("manifest: expected a string");
    }
    double num() const {
        if (const auto* d = std::get_if<double>(&v)) return *d;
        if (const auto* u = std::get_if<std::uint64_t>(&v)) return static_cast<double>(*u);
        if (const auto* i = std::get_if<std::int64_t>(&v)) return static_cast<double>(*i);
        throw sl::ValidationError("manifest: expected a number");
    }
    std::uint64_t uint() const {
        if (const auto* u = std::get_if<std::uint64_t>(&v)) return *u;
        if (const auto* i = std::get_if<std::int64_t>(&v); i && *i >= 0) return static_cast<std::uint64_t>(*i);
        if (const auto* d = std::get_if<double>(&v); d && *d >= 0 && *d == static_cast<double>(static_cast<std::uint64_t>(*d)))
            return static_cast<std::uint64_t>(*d);
        throw sl::ValidationError("manifest: expected an unsigned integer");
    }
};

// Shortest decimal that reads back to the same double; integral values keep a ".0".
std::string format_double(double d) {
    char buf[40];
    for (int prec = 1; prec <= 17; ++prec) {
        std::snprintf(buf, sizeof(buf), "%.*g", prec, d);
        if (std::strtod(buf, nullptr) == d) break;
    }
    std::string s = buf;
    if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
    return s;
}

std::string quote(const std::string& s) {
    std::string out = "\"";
    for (const unsigned char c : s) {
        switch (c) {
            case '"': out += "\\\""; break;
            case '\\': out += "\\\\"; break;
            case '\n': out += "\\n"; break;
            case '\r': out += "\\r"; break;
            case '\t': out += "\\t"; break;
            case '\b': out += "\\b"; break;
            case '\f': out += "\\f"; break;
            default:
                if (c < 0x20) {
                    char u[8];
                    std::snprintf(u, sizeof(u), "\\u%04x", c);
                    out += u;
                } else {
                    out += static_cast<char>(c);
                }
        }
    }
    return out + "\"";
}

void dump(const Json& j, std::string& out, int indent) {
    const std::string pad(static_cast<std::size_t>(indent) + 2, ' ');
    std::visit(
        [&](const auto& x) {
            using T = std::decay_t<decltype(x)>;
            if constexpr (std::is_same_v<T, std::nullptr_t>) out += "null";
            else if constexpr (std::is_same_v<T, bool>) out += x ? "true" : "false";
            else if constexpr (std::is_same_v<T, std::uint64_t> || std::is_same_v<T, std::int64_t>) out += std::to_string(x);
            else if constexpr (std::is_same_v<T, double>) out += format_double(x);
            else if constexpr (std::is_same_v<T, std::string>) out += quote(x);
            else if constexpr (std::is_same_v<T, Json::Array>) {
                if (x.empty()) { out += "[]"; return; }
                out += "[\n";
                for (std::size_t i = 0; i < x.size(); ++i) {
                    out += pad;
                    dump(x[i], out, indent + 2);
                    out += i + 1 < x.size() ? ",\n" : "\n";
                }
                out += std::string(static_cast<std::size_t>(indent), ' ') + "]";
            } else {
                if (x.empty()) { out += "{}"; return; }
                out += "{\n";
                std::size_t i = 0;
                for (const auto& [k, val] : x) {
                    out += pad + quote(k) + ": ";
                    dump(val, out, indent + 2);
                    out += ++i < x.size() ? ",\n" : "\n";
                }
                out += std::string(static_cast<std::size_t>(indent), ' ') + "}";
            }
        },
        j.v);
}

struct JsonParser {
    const std::string& s;
    std::size_t p = 0;

    [[noreturn]] void fail(const char* what) const {
        throw sl::ValidationError(std::string("manifest: ") + what + " at offset " + std::to_string(p));
    }
    void ws() {
        while (p < s.size() && (s[p] == ' ' || s[p] == '\n' || s[p] == '\r' || s[p] == '\t')) ++p;
    }
    bool lit(const char* w) {
        const std::size_t n = std::strlen(w);
        if (s.compare(p, n, w) == 0) { p += n; return true; }
        return false;
    }
    std::string string() {
        if (s[p] != '"') fail("expected a string");
        ++p;
        std::string out;
        while (p < s.size() && s[p] != '"') {
            char c = s[p++];
            if (c == '\\') {
                if (p >= s.size()) fail("bad escape");
                c = s[p++];
                switch (c) {
                    case 'n': out += '\n'; break;
                    case 'r': out += '\r'; break;
                    case 't': out += '\t'; break;
                    case 'b': out += '\b'; break;
                    case 'f': out += '\f'; break;
                    case 'u': {
                        if (p + 4 > s.size()) fail("bad \\u escape");
                        const unsigned cp = static_cast<unsigned>(std::stoul(s.substr(p, 4), nullptr, 16));
                        p += 4;
                        if (cp < 0x80) out += static_cast<char>(cp);
                        else if (cp < 0x800) { out += static_cast<char>(0xC0 | (cp >> 6)); out += static_cast<char>(0x80 | (cp & 0x3F)); }
                        else { out += static_cast<char>(0xE0 | (cp >> 12)); out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F)); out += static_cast<char>(0x80 | (cp & 0x3F)); }
                        break;
                    }
                    default: out += c;
                }
            } else {
                out += c;
            }
        }
        if (p >= s.size()) fail("unterminated string");
        ++p;
        return out;
    }
    Json value() {
        ws();
        if (p >= s.size()) fail("unexpected end");
        const char c = s[p];
        if (c == '{') {
            ++p;
            Json::Object o;
            ws();
            if (s[p] == '}') { ++p; return Json(std::move(o)); }
            for (;;) {
                ws();
                std::string k = string();
                ws();
                if (s[p++] != ':') fail("expected ':'");
                o[k] = value();
                ws();
                if (s[p] == ',') { ++p; continue; }
                if (s[p] == '}') { ++p; break; }
                fail("expected ',' or '}'");
            }
            return Json(std::move(o));
        }
        if (c == '[') {
            ++p;
            Json j;
            j.v = Json::Array{};
            auto& a = std::get<Json::Array>(j.v);
            ws();
            if (s[p] == ']') { ++p; return j; }
            for (;;) {
                a.push_back(value());
                ws();
                if (s[p] == ',') { ++p; continue; }
                if (s[p] == ']') { ++p; break; }
                fail("expected ',' or ']'");
            }
            return j;
        }
        if (c == '"') return Json(string());
        if (lit("null")) return Json(nullptr);
        if (lit("true")) return Json(true);
        if (lit("false")) return Json(false);
        const std::size_t b = p;
        bool real = false;
        while (p < s.size() && std::strchr("+-0123456789.eE", s[p])) real |= std::strchr(".eE", s[p++]) != nullptr;
        if (b == p) fail("unexpected character");
        const std::string t = s.substr(b, p - b);
        if (real) return Json(std::strtod(t.c_str(), nullptr));
        if (t[0] == '-') return Json(static_cast<std::int64_t>(std::strtoll(t.c_str(), nullptr, 10)));
        return Json(static_cast<std::uint64_t>(std::strtoull(t.c_str(), nullptr, 10)));
    }
};

// ------------------------------------------------------------- arguments --
// One option: its value slot parses the string; envname fills it when the flag is absent.
struct Option {
    std::string flag, help, envname;
    bool required = false;
    bool is_flag_set = false;  // seen on the command line or in the environment
    std::function<void(const std::string&)> set;
};

struct Command {
    std::string name, help;
    std::vector<Option> opts;

    template <class T>
    Option& add(const std::string& flag, T& slot, const std::string& help) {
        Option o;
        o.flag = flag;
        o.help = help;
        o.set = [&slot, flag](const std::string& text) { parse_into(slot, flag, text); };
        opts.push_back(std::move(o));
        return opts.back();
    }
    std::size_t count(const std::string& flag) const {
        for (const auto& o : opts)
            if (o.flag == flag) return o.is_flag_set ? 1 : 0;
        return 0;
    }
    Option* find(const std::string& flag) {
        for (auto& o : opts)
            if (o.flag == flag) return &o;
        return nullptr;
    }

    static void parse_into(std::string& slot, const std::string&, const std::string& text) { slot = text; }
    static void parse_into(double& slot, const std::string& flag, const std::string& text) {
        char* end = nullptr;
        errno = 0;
        slot = std::strtod(text.c_str(), &end);
        if (text.empty() || *end || errno) throw UsageError(flag + ": value " + text + " is not a number");
    }
    template <class U>
    static void parse_into(U& slot, const std::string& flag, const std::string& text) {
        static_assert(std::is_unsigned_v<U>);
        char* end = nullptr;
        errno = 0;
        const unsigned long long x = std::strtoull(text.c_str(), &end, 10);
        if (text.empty() || text[0] == '-' || *end || errno || x > std::numeric_limits<U>::max())
            throw UsageError(flag + ": value " + text + " is not a valid unsigned integer");
        slot = static_cast<U>(x);
    }

    void usage(std::ostream& out) const {
        out << "Usage: sparselda " << name << " [OPTIONS]\n" << help << "\n\nOptions:\n";
        for (const auto& o : opts) {
            out << "  " << o.flag << " <value>  " << o.help;
            if (!o.envname.empty()) out << " (env " << o.envname << ")";
            if (o.required) out << " REQUIRED";
            out << '\n';
        }
    }

    // argv[i..] -> slots; throws UsageError (exit 1) on unknown flags / missing values.
    void parse(int argc, char** argv, int i) {
        for (; i < argc; ++i) {
            std::string a = argv[i], val;
            if (a == "-h" || a == "--help") {
                usage(std::cout);
                std::exit(0);
            }
            const auto eq = a.find('=');
            bool inline_val = false;
            if (a.rfind("--", 0) == 0 && eq != std::string::npos) {
                val = a.substr(eq + 1);
                a = a.substr(0, eq);
                inline_val = true;
            }
            Option* o = find(a);
            if (!o) throw UsageError("The following argument was not expected: " + a);
            if (!inline_val) {
                if (i + 1 >= argc) throw UsageError(a + " requires a value");
                val = argv[++i];
            }
            o->set(val);
            o->is_flag_set = true;
        }
        for (auto& o : opts) {
            if (!o.is_flag_set && !o.envname.empty()) {
                if (const char* e = std::getenv(o.envname.c_str()); e && *e) {
                    o.set(e);
                    o.is_flag_set = true;
                }
            }
            if (o.required && !o.is_flag_set) throw UsageError(o.flag + " is required");
        }
    }
};

// FNV-1a 64 of a file, "0x%016llx" (main.cpp:22-38).
std::string file_digest(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw sl::IoError("cannot open " + path);
    std::uint64_t hash = 1469598103934665603ull;
    std::vector<char> buf(1 << 16);
    while (in) {
        in.read(buf.data(), static_cast<std::streamsize>(buf.size()));
        const std::streamsize got = in.gcount();
        for (std::streamsize i = 0; i < got; ++i) {
            hash ^= static_cast<unsigned char>(buf[static_cast<std::size_t>(i)]);
            hash *= 1099511628211ull;
        }
    }
    char out[32];
    std::snprintf(out, sizeof(out), "0x%016llx", static_cast<unsigned long long>(hash));
    return out;
}

sl::Corpus load_docword_file(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw sl::IoError("cannot open docword file " + path);
    return sl::load_docword(in);
}

std::vector<std::string> load_vocab_file(const std::string& path, std::uint32_t expected) {
    std::ifstream in(path);
    if (!in) throw sl::IoError("cannot open vocab file " + path);
    std::vector<std::string> vocab;
    std::string term;
    while (std::getline(in, term)) {
        if (!term.empty() && term.back() == '\r') term.pop_back();
        vocab.push_back(term);
    }
    if (vocab.size() != expected)
        throw sl::ValidationError("vocab file has " + std::to_string(vocab.size()) + " entries, model expects " +
                                  std::to_string(expected));
    return vocab;
}

// ----------------------------------------------------------------- train --
struct TrainArgs {
    std::string docword, vocab, heldout, out_dir = "run", manifest_path, sampler = "sparse";
    std::uint32_t topics = 0, iters = 100, chunks = 0, eval_every = 1, burn_in = 20;
    double alpha = 0.0, beta = 0.01;
    unsigned workers = 0;
    std::uint64_t seed = 0, mem_budget = 1ull << 30;
    bool seed_given = false;
    int device = -1;
};

// --from-manifest: every flag not given on the command line takes the manifest's value
// (main.cpp:86-121).
void apply_manifest_defaults(const Command& cmd, TrainArgs& a) {
    std::ifstream in(a.manifest_path);
    if (!in) throw sl::IoError("cannot open manifest " + a.manifest_path);
    std::stringstream ss;
    ss << in.rdbuf();
    const std::string text = ss.str();
    JsonParser jp{text};
    const Json m = jp.value();
    const Json& cfg = m.at("config");
    const Json& inputs = m.at("inputs");
    auto has = [](const Json& src, const char* k) { return src.contains(k) && !src.at(k).is_null(); };
    if (!cmd.count("--docword") && has(inputs.at("docword"), "path")) a.docword = inputs.at("docword").at("path").str();
    if (!cmd.count("--vocab") && has(inputs.at("vocab"), "path")) a.vocab = inputs.at("vocab").at("path").str();
    if (inputs.contains("heldout") && !inputs.at("heldout").is_null() && !cmd.count("--heldout") &&
        has(inputs.at("heldout"), "path"))
        a.heldout = inputs.at("heldout").at("path").str();
    auto u32 = [&](const char* flag, const char* key, std::uint32_t& slot) {
        if (!cmd.count(flag) && has(cfg, key)) slot = static_cast<std::uint32_t>(cfg.at(key).uint());
    };
    u32("--topics", "topics", a.topics);
    if (!cmd.count("--alpha") && has(cfg, "alpha")) a.alpha = cfg.at("alpha").num();
    if (!cmd.count("--beta") && has(cfg, "beta")) a.beta = cfg.at("beta").num();
    u32("--iters", "iters", a.iters);
    u32("--chunks", "chunks", a.chunks);
    if (!cmd.count("--workers") && has(cfg, "workers")) a.workers = static_cast<unsigned>(cfg.at("workers").uint());
    if (!cmd.count("--mem-budget") && has(cfg, "mem_budget")) a.mem_budget = cfg.at("mem_budget").uint();
    u32("--eval-every", "eval_every", a.eval_every);
    u32("--burn-in", "burn_in", a.burn_in);
    if (!cmd.count("--sampler") && has(cfg, "sampler")) a.sampler = cfg.at("sampler").str();
    if (!cmd.count("--seed") && cfg.contains("seed")) {
        a.seed = cfg.at("seed").uint();
        a.seed_given = true;
    }
}

int run_train(const Command& cmd, TrainArgs& a) {
    if (!a.manifest_path.empty()) apply_manifest_defaults(cmd, a);
    if (a.docword.empty() || a.vocab.empty()) throw sl::ValidationError("train requires --docword and --vocab");
    if (!a.seed_given) {
        std::random_device rd;
        a.seed = (static_cast<std::uint64_t>(rd()) << 32) | rd();
    }
    const sl::Corpus corpus = sl::load_uci_files(a.docword, a.vocab);

    sl::TrainConfig cfg;
    cfg.num_topics = a.topics;
    cfg.alpha = a.alpha;
    cfg.beta = a.beta;
    cfg.iterations = a.iters;
    cfg.num_chunks = a.chunks;
    cfg.num_workers = a.workers;
    cfg.seed = a.seed;
    cfg.memory_budget = a.mem_budget;
    cfg.eval_every = a.eval_every;
    cfg.device = a.device;
    if (a.sampler == "sparse") cfg.sampler = sl::SamplerKind::kSparse;
    else if (a.sampler == "vanilla") cfg.sampler = sl::SamplerKind::kVanilla;
    else throw sl::ValidationError("--sampler must be sparse or vanilla");
    const sl::TrainConfig r = cfg.resolved(corpus);

    std::filesystem::create_directories(a.out_dir);
    const std::filesystem::path out_dir(a.out_dir);

    Json manifest;
    manifest["artifact_version"] = sl::kVersion;
    manifest["command"] = "train";
    Json& c = manifest["config"];
    c["topics"] = r.num_topics;
    c["alpha"] = r.alpha;
    c["beta"] = r.beta;
    c["iters"] = r.iterations;
    c["chunks"] = r.num_chunks;
    c["workers"] = static_cast<std::uint64_t>(r.num_workers);
    c["seed"] = r.seed;
    c["mem_budget"] = r.memory_budget;
    c["eval_every"] = r.eval_every;
    c["burn_in"] = a.burn_in;
    c["sampler"] = a.sampler;
    Json& in = manifest["inputs"];
    in["docword"]["path"] = a.docword;
    in["docword"]["digest"] = file_digest(a.docword);
    in["vocab"]["path"] = a.vocab;
    in["vocab"]["digest"] = file_digest(a.vocab);
    if (!a.heldout.empty()) {
        in["heldout"]["path"] = a.heldout;
        in["heldout"]["digest"] = file_digest(a.heldout);
    } else {
        in["heldout"] = nullptr;
    }
    {
        std::ofstream out(out_dir / "manifest.json");
        if (!out) throw sl::IoError("cannot write manifest in " + a.out_dir);
        std::string text;
        dump(manifest, text, 0);
        out << text << '\n';
    }

    std::optional<sl::Corpus> heldout;
    if (!a.heldout.empty()) {
        heldout = load_docword_file(a.heldout);
        if (heldout->vocab_size != corpus.vocab_size)
            throw sl::ValidationError("held-out vocabulary size differs from training corpus");
    }
    std::ofstream metrics(out_dir / "metrics.log", std::ios::trunc);
    if (!metrics) throw sl::IoError("cannot write metrics log in " + a.out_dir);
    const sl::MetricsSink sink = [&metrics](const sl::MetricsEntry& e) {
        metrics << sl::format_metrics_line(e) << '\n';
        metrics.flush();
    };
    sl::HeldoutProbe probe;
    if (heldout) {
        probe = [&](sl::ModelState& m) {
            return sl::heldout_ll(m, *heldout, a.burn_in, r.num_workers, r.seed).per_token_ll;
        };
    }
    sl::ModelState state = sl::train(corpus, r, sink, probe);
    sl::save_checkpoint(out_dir / "model.ckpt", state);
    std::cout << "trained " << state.num_tokens << " tokens, K=" << state.num_topics << ", " << r.iterations
              << " iterations -> " << (out_dir / "model.ckpt").string() << '\n';
    return 0;
}

// ------------------------------------------------------------- eval/topics --
struct EvalArgs {
    std::string model, heldout;
    std::uint32_t burn_in = 20;
    unsigned workers = 0;
    std::uint64_t seed = 0;
    bool seed_given = false;
    int device = -1;
};

int run_eval(const EvalArgs& a) {
    const sl::Checkpoint ck = sl::load_checkpoint(a.model);
    sl::ModelState model = sl::model_from_checkpoint(ck, a.workers);
    const sl::Corpus held = load_docword_file(a.heldout);
    if (held.vocab_size != model.vocab_size) throw sl::ValidationError("held-out vocabulary size differs from model");
    const std::uint64_t seed = a.seed_given ? a.seed : ck.seed;
    std::cout << sl::format_eval_line(sl::heldout_ll(model, held, a.burn_in, a.workers, seed)) << '\n';
    return 0;
}

struct TopicsArgs {
    std::string model, vocab;
    std::uint32_t top_n = 10;
};

int run_topics(const TopicsArgs& a) {
    const sl::Checkpoint ck = sl::load_checkpoint(a.model);
    std::vector<std::string> vocab;
    if (!a.vocab.empty()) vocab = load_vocab_file(a.vocab, ck.vocab_size);
    if (a.top_n > ck.vocab_size) throw sl::ValidationError("top_words n exceeds vocabulary size");
    const sl::ModelState model = sl::model_from_checkpoint(ck);
    sl::print_topics(std::cout, model, vocab, a.top_n);
    return 0;
}

void top_usage(std::ostream& out) {
    out << "Sparsity-aware LDA trainer (B200 engine)\nUsage: sparselda SUBCOMMAND [OPTIONS]\n\n"
           "Subcommands:\n  train   Train a topic model\n  eval    Held-out log-likelihood of a checkpoint\n"
           "  topics  Top words per topic\n";
}

}  // namespace

int main(int argc, char** argv) {
    TrainArgs ta;
    Command train{"train", "Train a topic model", {}};
    train.add("--docword", ta.docword, "UCI bag-of-words docword file").envname = "SPARSELDA_DOCWORD";
    train.add("--vocab", ta.vocab, "Vocabulary file, one term per line").envname = "SPARSELDA_VOCAB";
    train.add("--topics", ta.topics, "Number of topics K");
    train.add("--alpha", ta.alpha, "Doc-topic smoothing (default 50/K)");
    train.add("--beta", ta.beta, "Word-topic smoothing (0.01)");
    train.add("--iters", ta.iters, "Training iterations (100)");
    train.add("--chunks", ta.chunks, "Chunk count (0 = auto from --mem-budget)");
    train.add("--workers", ta.workers, "Worker threads (0 = hardware)").envname = "SPARSELDA_WORKERS";
    train.add("--seed", ta.seed, "RNG seed (generated when absent)").envname = "SPARSELDA_SEED";
    train.add("--heldout", ta.heldout, "Held-out docword file");
    train.add("--eval-every", ta.eval_every, "Iterations between held-out evaluations (1)");
    train.add("--burn-in", ta.burn_in, "Held-out burn-in sweeps (20)");
    train.add("--out", ta.out_dir, "Output directory (run)").envname = "SPARSELDA_OUT";
    train.add("--mem-budget", ta.mem_budget, "Chunk memory budget in bytes (1073741824)").envname = "SPARSELDA_MEM_BUDGET";
    train.add("--sampler", ta.sampler, "sparse | vanilla (sparse)");
    train.add("--from-manifest", ta.manifest_path, "Reproduce a run from its manifest");
    unsigned train_dev = 0;
    train.add("--device", train_dev, "CUDA device ordinal (0)");

    EvalArgs ea;
    Command eval{"eval", "Held-out log-likelihood of a checkpoint", {}};
    eval.add("--model", ea.model, "Checkpoint file").required = true;
    eval.add("--heldout", ea.heldout, "Held-out docword file").required = true;
    eval.add("--burn-in", ea.burn_in, "Burn-in sweeps (20)");
    eval.add("--workers", ea.workers, "Worker threads (0 = hardware)").envname = "SPARSELDA_WORKERS";
    eval.add("--seed", ea.seed, "RNG seed (default: checkpoint seed)");

    TopicsArgs tpa;
    Command topics{"topics", "Top words per topic", {}};
    topics.add("--model", tpa.model, "Checkpoint file").required = true;
    topics.add("--top-n", tpa.top_n, "Words per topic (10)");
    topics.add("--vocab", tpa.vocab, "Vocabulary file for surface forms");

    try {
        if (argc < 2) throw UsageError("A subcommand is required");
        const std::string sub = argv[1];
        if (sub == "-h" || sub == "--help") {
            top_usage(std::cout);
            return 0;
        }
        if (sub == "train") {
            train.parse(argc, argv, 2);
            ta.seed_given = train.count("--seed") > 0;
            ta.device = train.count("--device") ? static_cast<int>(train_dev) : -1;
            return run_train(train, ta);
        }
        if (sub == "eval") {
            eval.parse(argc, argv, 2);
            ea.seed_given = eval.count("--seed") > 0;
            return run_eval(ea);
        }
        if (sub == "topics") {
            topics.parse(argc, argv, 2);
            return run_topics(tpa);
        }
        throw UsageError("The following argument was not expected: " + sub);
    } catch (const UsageError& e) {
        std::cerr << e.what() << "\nRun with --help for more information.\n";
        return 1;
    } catch (const sl::ValidationError& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 1;
    } catch (const sl::IoError& e) {
        std::cerr << "io error: " << e.what() << '\n';
        return 2;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 1;
    }
}
