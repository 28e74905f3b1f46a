// corpus_gen.cpp -- the synthetic corpora of SURVEY.md §8(d) (slda_generate_*, declared in
// include/saberlda.h).  Host-only, multi-threaded, deterministic in (params, seed) whatever the
// thread count.  Compiled into libsaberlda.so, and on its own (SLDA_GEN_STANDALONE, by
// oracle/Makefile) into oracle/libcorpusgen.so so that bench.py's reference arm builds the
// same corpus without loading the product.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/saberlda.h"

#ifdef SLDA_GEN_STANDALONE
namespace {
thread_local std::string g_gen_error;
}
void slda_set_error_internal(const std::string& msg) { g_gen_error = msg; }
extern "C" const char* slda_gen_last_error(void) { return g_gen_error.c_str(); }
#else
void slda_set_error_internal(const std::string& msg);  // engine.cu
#endif

namespace {


// Counter-based Philox4x32-10 stream (same generator as rng.hpp:14-83), so a
// corpus is a pure function of (params, seed) whatever the thread count.
struct Stream {
    uint32_t key[2];
    uint32_t ctr[4];
    uint64_t buf[2];
    int cached = 0;
    Stream(uint64_t seed, uint32_t kind, uint64_t element)
        : key{static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32)},
          ctr{kind, static_cast<uint32_t>(element), static_cast<uint32_t>(element >> 32), 0u} {}
    void refill() {
        uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3], k0 = key[0], k1 = key[1];
        for (int r = 0; r < 10; ++r) {
            const uint64_t p0 = static_cast<uint64_t>(0xD2511F53u) * c0;
            const uint64_t p1 = static_cast<uint64_t>(0xCD9E8D57u) * c2;
            const uint32_t n0 = static_cast<uint32_t>(p1 >> 32) ^ c1 ^ k0;
            const uint32_t n2 = static_cast<uint32_t>(p0 >> 32) ^ c3 ^ k1;
            c1 = static_cast<uint32_t>(p1);
            c3 = static_cast<uint32_t>(p0);
            c0 = n0;
            c2 = n2;
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        ++ctr[3];
        buf[1] = (static_cast<uint64_t>(c1) << 32) | c0;
        buf[0] = (static_cast<uint64_t>(c3) << 32) | c2;
        cached = 2;
    }
    double uniform() {  // [0, 1)
        if (cached == 0) refill();
        return static_cast<double>(buf[--cached] >> 11) * 0x1.0p-53;
    }
    double open_uniform() {  // (0, 1)
        double u;
        do u = uniform(); while (u == 0.0);
        return u;
    }
    double normal() {
        const double u1 = open_uniform(), u2 = uniform();
        return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
    }
    // Marsaglia-Tsang; shape < 1 via the U^(1/a) boost.
    double gamma(double a) {
        if (a < 1.0) return gamma(a + 1.0) * std::pow(open_uniform(), 1.0 / a);
        const double d = a - 1.0 / 3.0, c = 1.0 / std::sqrt(9.0 * d);
        for (;;) {
            double x, v;
            do {
                x = normal();
                v = 1.0 + c * x;
            } while (v <= 0.0);
            v = v * v * v;
            const double u = open_uniform();
            if (std::log(u) < 0.5 * x * x + d - d * v + d * std::log(v)) return d * v;
        }
    }
};

enum : uint32_t { kKindLength = 1, kKindTheta = 2, kKindTokens = 3, kKindPerm = 4 };

unsigned resolve_threads(uint32_t t) {
    if (t) return t;
    const unsigned hw = std::thread::hardware_concurrency();
    return hw ? hw : 1;
}

template <class Body>
void parallel_blocks(uint64_t n, unsigned workers, Body&& body) {
    if (n == 0) return;
    workers = static_cast<unsigned>(std::min<uint64_t>(workers, n));
    if (workers <= 1) {
        body(uint64_t{0}, n);
        return;
    }
    std::vector<std::thread> pool;
    const uint64_t base = n / workers, extra = n % workers;
    uint64_t begin = 0;
    for (unsigned w = 0; w < workers; ++w) {
        const uint64_t end = begin + base + (w < extra ? 1 : 0);
        pool.emplace_back([&body, begin, end] { body(begin, end); });
        begin = end;
    }
    for (auto& t : pool) t.join();
}

struct Params {
    uint32_t family, D, V, KT;
    uint64_t T;
    double s, dir, sigma;
    uint64_t seed;
    unsigned threads;
};

Params resolve(const slda_gen_params* p) {
    if (!p) throw std::invalid_argument("null params");
    Params r;
    r.family = p->family;
    r.D = p->num_docs;
    r.V = p->vocab_size;
    r.T = p->num_tokens;
    r.KT = p->latent_topics ? p->latent_topics : 100;
    r.s = p->zipf_s > 0 ? p->zipf_s : 1.0;
    r.dir = p->doc_dirichlet > 0 ? p->doc_dirichlet : 0.1;
    r.sigma = p->length_sigma > 0 ? p->length_sigma : 0.6;
    r.seed = p->seed ? p->seed : 20161008ull;
    r.threads = resolve_threads(p->threads);
    if (r.family > 1) throw std::invalid_argument("family must be 0 (G) or 1 (U)");
    if (r.D == 0 || r.V == 0) throw std::invalid_argument("num_docs and vocab_size must be >= 1");
    if (r.family == 0 && r.T < r.D) throw std::invalid_argument("family G needs T >= D (every length >= 1)");
    return r;
}

std::vector<uint32_t> doc_lengths(const Params& p) {
    std::vector<uint32_t> len(p.D);
    if (p.family == 0) {
        // lognormal(0, sigma), rescaled so the lengths sum to T exactly, each >= 1.
        std::vector<double> raw(p.D);
        parallel_blocks(p.D, p.threads, [&](uint64_t b, uint64_t e) {
            for (uint64_t d = b; d < e; ++d) raw[d] = std::exp(p.sigma * Stream(p.seed, kKindLength, d).normal());
        });
        double sum = 0;
        for (double x : raw) sum += x;
        uint64_t total = 0;
        for (uint32_t d = 0; d < p.D; ++d) {
            const double x = std::floor(raw[d] * static_cast<double>(p.T) / sum);
            len[d] = static_cast<uint32_t>(std::max(1.0, std::min(x, 4.0e9)));
            total += len[d];
        }
        uint32_t d = 0;
        while (total < p.T) {
            ++len[d];
            ++total;
            d = d + 1 == p.D ? 0 : d + 1;
        }
        d = 0;
        while (total > p.T) {
            if (len[d] > 1) {
                --len[d];
                --total;
            }
            d = d + 1 == p.D ? 0 : d + 1;
        }
    } else {
        // Poisson(T/D) by inversion, >= 1 (fixtures.cpp:50-67 shape).
        const double mean = static_cast<double>(p.T) / p.D;
        parallel_blocks(p.D, p.threads, [&](uint64_t b, uint64_t e) {
            for (uint64_t d = b; d < e; ++d) {
                Stream rng(p.seed, kKindLength, d);
                uint32_t k;
                if (mean < 500) {
                    const double L = std::exp(-mean);
                    double prod = rng.open_uniform();
                    k = 0;
                    while (prod > L) {
                        ++k;
                        prod *= rng.open_uniform();
                    }
                } else {
                    k = static_cast<uint32_t>(std::max(0.0, std::round(mean + std::sqrt(mean) * rng.normal())));
                }
                len[d] = std::max<uint32_t>(1, k);
            }
        });
    }
    return len;
}

}  // namespace

extern "C" {

int slda_generate_corpus_size(const slda_gen_params* params, uint64_t* num_tokens) {
    try {
        const Params p = resolve(params);
        if (p.family == 0) {
            *num_tokens = p.T;
        } else {
            uint64_t t = 0;
            for (uint32_t l : doc_lengths(p)) t += l;
            *num_tokens = t;
        }
        return SLDA_OK;
    } catch (const std::exception& e) {
        slda_set_error_internal(e.what());
        return SLDA_ERR_VALIDATION;
    }
}

int slda_generate_doc_lengths(const slda_gen_params* params, uint32_t* lengths) {
    try {
        const Params p = resolve(params);
        const std::vector<uint32_t> len = doc_lengths(p);
        std::memcpy(lengths, len.data(), len.size() * 4);
        return SLDA_OK;
    } catch (const std::exception& e) {
        slda_set_error_internal(e.what());
        return SLDA_ERR_VALIDATION;
    }
}

int slda_generate_corpus(const slda_gen_params* params, uint32_t* tokens, uint64_t capacity) {
    if (!params) return SLDA_ERR_VALIDATION;
    return slda_generate_docs(params, 0, params->num_docs, tokens, capacity);
}

int slda_generate_docs(const slda_gen_params* params, uint32_t doc_begin, uint32_t doc_end,
                       uint32_t* tokens, uint64_t capacity) {
    try {
        const Params p = resolve(params);
        if (doc_begin > doc_end || doc_end > p.D) throw std::invalid_argument("invalid document range");
        const std::vector<uint32_t> len = doc_lengths(p);
        // Offsets relative to the first token of doc_begin.
        std::vector<uint64_t> off(static_cast<size_t>(p.D) + 1, 0);
        for (uint32_t d = doc_begin; d < doc_end; ++d) off[d + 1] = off[d] + len[d];
        if (off[doc_end] > capacity) throw std::invalid_argument("token buffer too small");
        const uint64_t nd = doc_end - doc_begin;
        if (p.family == 1) {
            parallel_blocks(nd, p.threads, [&](uint64_t b, uint64_t e) {
                for (uint64_t d = doc_begin + b; d < doc_begin + e; ++d) {
                    Stream rng(p.seed, kKindTokens, d);
                    for (uint64_t t = off[d]; t < off[d + 1]; ++t) {
                        uint32_t w = static_cast<uint32_t>(rng.uniform() * p.V);
                        tokens[3 * t] = static_cast<uint32_t>(d);
                        tokens[3 * t + 1] = w < p.V ? w : p.V - 1;
                        tokens[3 * t + 2] = SLDA_INVALID_TOPIC;
                    }
                }
            });
            return SLDA_OK;
        }
        // Family G: latent topic j is Zipf(s) over its own seeded permutation of the
        // vocabulary; doc theta ~ Dirichlet(dir) over KT latent topics.
        std::vector<double> cdf(p.V);
        double acc = 0;
        for (uint32_t r = 0; r < p.V; ++r) {
            acc += std::pow(static_cast<double>(r + 1), -p.s);
            cdf[r] = acc;
        }
        for (double& c : cdf) c /= acc;
        std::vector<uint32_t> perm(static_cast<size_t>(p.KT) * p.V);
        parallel_blocks(p.KT, p.threads, [&](uint64_t b, uint64_t e) {
            for (uint64_t j = b; j < e; ++j) {
                uint32_t* pj = perm.data() + j * p.V;
                for (uint32_t i = 0; i < p.V; ++i) pj[i] = i;
                Stream rng(p.seed, kKindPerm, j);
                for (uint32_t i = p.V - 1; i > 0; --i) {
                    uint32_t k = static_cast<uint32_t>(rng.uniform() * (i + 1));
                    if (k > i) k = i;
                    std::swap(pj[i], pj[k]);
                }
            }
        });
        parallel_blocks(nd, p.threads, [&](uint64_t b, uint64_t e) {
            std::vector<double> theta(p.KT);
            for (uint64_t d = doc_begin + b; d < doc_begin + e; ++d) {
                Stream trng(p.seed, kKindTheta, d);
                double tsum = 0;
                for (uint32_t j = 0; j < p.KT; ++j) {
                    tsum += trng.gamma(p.dir);
                    theta[j] = tsum;
                }
                Stream rng(p.seed, kKindTokens, d);
                for (uint64_t t = off[d]; t < off[d + 1]; ++t) {
                    const double pick = rng.uniform() * tsum;
                    uint32_t j = static_cast<uint32_t>(std::upper_bound(theta.begin(), theta.end(), pick) - theta.begin());
                    if (j >= p.KT) j = p.KT - 1;
                    const double u = rng.uniform();
                    uint32_t r = static_cast<uint32_t>(std::upper_bound(cdf.begin(), cdf.end(), u) - cdf.begin());
                    if (r >= p.V) r = p.V - 1;
                    tokens[3 * t] = static_cast<uint32_t>(d);
                    tokens[3 * t + 1] = perm[static_cast<size_t>(j) * p.V + r];
                    tokens[3 * t + 2] = SLDA_INVALID_TOPIC;
                }
            }
        });
        return SLDA_OK;
    } catch (const std::exception& e) {
        slda_set_error_internal(e.what());
        return SLDA_ERR_VALIDATION;
    }
}

}  // extern "C"
