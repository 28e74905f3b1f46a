// kernels.cu -- sm_100a kernels of one ESCA iteration and its setup.
//
// Reference paths are relative to /root/reference/proj.  Each kernel names the
// reference function it replaces.  See DESIGN.md for layouts and rooflines.
#include "common.cuh"
#include "kernels.hpp"

#include <cstdlib>
#include <string>

namespace slda {

namespace {

inline uint32_t grid_for(uint64_t n, uint32_t threads, uint32_t cap = 148u * 32u) {
    const uint64_t g = (n + threads - 1) / threads;
    return static_cast<uint32_t>(g == 0 ? 1 : (g > cap ? cap : g));
}

}  // namespace

// ============================================================================
// K3 sampler -- process_segment (trainer.cpp:265-291) + sample_token<float>
// (sampler.hpp:166-204) + the C_wk accumulation of accumulate_word_topic
// (counts.cpp:127-132).  One CTA per heavy-first work unit of one word; the
// word's phi row and its L8 level are staged in shared memory; each warp stages
// its 32 tokens' C_dk rows cooperatively (coalesced), and each lane samples one
// token so that the sparse mass S and the in-place prefix run as the reference's
// sequential f32 chains.
// ============================================================================

// phi row lookup: shared memory (staged row) or, when the row is too large to stage
// (kGlobalPhi, K >~ 45K), the global row through L1/L2.
template <bool kGlobalPhi>
__device__ __forceinline__ float entry_mass(uint32_t e, uint32_t tbits, uint32_t tmask, const float* phi) {
    const float p = kGlobalPhi ? __ldg(phi + (e & tmask)) : phi[e & tmask];
    return __fmul_rn(__uint2float_rn(e >> tbits), p);
}

template <bool kGlobalPhi>
__device__ __forceinline__ float acc_quad(float s, const uint4& q, uint32_t tbits, uint32_t tmask,
                                          const float* phi) {
    s = __fadd_rn(s, entry_mass<kGlobalPhi>(q.x, tbits, tmask, phi));
    s = __fadd_rn(s, entry_mass<kGlobalPhi>(q.y, tbits, tmask, phi));
    s = __fadd_rn(s, entry_mass<kGlobalPhi>(q.z, tbits, tmask, phi));
    return __fadd_rn(s, entry_mass<kGlobalPhi>(q.w, tbits, tmask, phi));
}

// One 32-byte sector (8 C_dk entries) per lane: a 256-bit load (LDG.E.256 on sm_100a),
// not allocated in L1 (rows are streamed; the reuse is in L2).
struct Sector {
    uint4 lo, hi;
};
__device__ __forceinline__ Sector ldg_sector(const uint4* p) {
    Sector s;
    asm("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(s.lo.x), "=r"(s.lo.y), "=r"(s.lo.z), "=r"(s.lo.w), "=r"(s.hi.x), "=r"(s.hi.y),
                   "=r"(s.hi.z), "=r"(s.hi.w)
                 : "l"(p));
    return s;
}

__device__ __forceinline__ Sector zero_sector() { return Sector{make_uint4(0u, 0u, 0u, 0u), make_uint4(0u, 0u, 0u, 0u)}; }

// Compact C_dk rows (K <= kCompactMaxK): 16-bit slots, two per 32-bit word.  Word 0 =
// nsect | nnz << 16.  Then the entries in ascending topic order: a count-1 entry is one slot
// holding its topic; a count >= 2 entry is a whole word (topic | 0x8000, count) at an even
// slot, a null slot (0xFFFF) padding the odd slot before it when needed; the row ends with
// null slots up to a sector (16 slots).  Pairs never straddle a word, so every word decodes
// on its own (sector checkpoints carry no parse state), and a count-1 entry needs no count
// conversion: f32(1) * phi == phi.  Versus the 32-bit wide format this halves the bytes of
// count-1 entries, the majority while documents are spread over many topics.
constexpr uint32_t kNull16 = 0xFFFFu;

// lower_bound over the word's L4 prefix (== WaryTree::sample, acceptance.cpp:140-200):
// binary search of the staged L8 level (first 8-block whose last prefix >= x), then one
// 32-byte sector of L4.  Returns the first index with L4 >= x (x <= total).
__device__ __forceinline__ uint32_t tree_search(float x, const float* s_l8, uint32_t n_l8, const float* l4row) {
    uint32_t lo = 0, hi = n_l8 - 1;  // s_l8[n_l8 - 1] == total >= x
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (s_l8[mid] >= x) hi = mid; else lo = mid + 1;
    }
    const Sector b = ldg_sector(reinterpret_cast<const uint4*>(l4row + lo * kLeaf));
    const uint32_t below = (__uint_as_float(b.lo.x) < x) + (__uint_as_float(b.lo.y) < x) +
                           (__uint_as_float(b.lo.z) < x) + (__uint_as_float(b.lo.w) < x) +
                           (__uint_as_float(b.hi.x) < x) + (__uint_as_float(b.hi.y) < x) +
                           (__uint_as_float(b.hi.z) < x) + (__uint_as_float(b.hi.w) < x);
    return lo * kLeaf + below;
}

// Per-warp staging of C_dk rows.  Lane-private random row reads cap at ~1.5 TB/s on B200
// (L1TEX: one line per lane per load); the warp-cooperative layout (adjacent lanes read
// adjacent sectors of one row) is coalesced per row and measured at 3.7-6 TB/s
// (scripts/microbench_rows.cu).  A group is G sectors (8G entries) of each of the warp's 32
// rows, loaded by 32/G rows per instruction (scripts/mb_pattern.cu: G=4 moves the same row
// bytes with ~20% fewer L1TEX wavefronts than G=2).  The (32G+16)-byte row stride keeps the
// cooperative stores and each lane's 128-bit reads of its own row bank-conflict free.
template <int G>
struct Stage {
    static constexpr uint32_t kRowsPerInst = 32 / G;
    static constexpr uint32_t kRow = 32 * G + 16;
    static constexpr uint32_t kWarp = 32 * kRow;
};
// Per-sector running sums for the first kCkSectors sectors (96 entries): the prefix pass
// of the sparse branch re-reads one sector instead of the row.  (12: at K = 10K two
// 512-thread CTAs fit one SM.)
constexpr uint32_t kCkSectors = 12;

__device__ __forceinline__ void sts_sector(unsigned char* p, const Sector& q) {
    *reinterpret_cast<uint4*>(p) = q.lo;
    *reinterpret_cast<uint4*>(p + 16) = q.hi;
}

// Cooperative load of sectors [gs, gs + G) of each of the warp's 32 rows (registers),
// and its store into the stage.  Per row kRowsPerInst*j + grp: rq = quad offset, ns = sector
// limit (0: skip), gs = first sector.  Sectors past a row's limit are neither loaded nor
// stored (the owning lane never reads them), so finished rows cost no L1TEX wavefronts.
template <int G>
__device__ __forceinline__ void load_group(const uint4* A4, const uint32_t (&rq)[G], const uint32_t (&ns)[G],
                                           const uint32_t (&gs)[G], uint32_t sub, Sector (&q)[G]) {
#pragma unroll
    for (uint32_t j = 0; j < G; ++j) {
        const uint32_t sec = gs[j] + sub;
        q[j] = sec < ns[j] ? ldg_sector(A4 + rq[j] + 2 * sec) : zero_sector();
    }
}
template <int G>
__device__ __forceinline__ void store_group(const Sector (&q)[G], const uint32_t (&ns)[G], const uint32_t (&gs)[G],
                                            uint32_t sub, uint32_t grp, unsigned char* stage) {
#pragma unroll
    for (uint32_t j = 0; j < G; ++j)
        if (gs[j] + sub < ns[j])
            sts_sector(stage + (Stage<G>::kRowsPerInst * j + grp) * Stage<G>::kRow + sub * 32, q[j]);
}
template <int G>
__device__ __forceinline__ void stage_group(const uint4* A4, const uint32_t (&rq)[G], const uint32_t (&ns)[G],
                                            const uint32_t (&gs)[G], uint32_t sub, uint32_t grp,
                                            unsigned char* stage) {
    Sector q[G];
    load_group<G>(A4, rq, ns, gs, sub, q);
    store_group<G>(q, ns, gs, sub, grp, stage);
}

// ---- Row decoding for the sampler (both row formats) ----------------------------------------
template <bool kGlobalPhi>
__device__ __forceinline__ float ld_phi(const float* phi, uint32_t t) {
    return kGlobalPhi ? __ldg(phi + t) : phi[t];
}

// Compact format word: up to two entries (see compact_chunk).  f32(1) * phi == phi, so a
// count-1 entry adds phi[topic] directly, exactly as the reference's s += f32(1) * phi.
// Branch-free word decode (lanes of a warp see different word kinds): the first slot is a
// pair (topic|0x8000, count), a single, or null; the second slot is a single or null unless
// the word is a pair.  Absent entries contribute +0 (s + +0 == s for the running sums, which
// are >= +0) and their gathers are predicated off.
struct WordEntries {
    uint32_t t0, t1;   // topics
    float c0;          // count of the first entry (1 for a single)
    bool v0, v1;       // entries present
};
__device__ __forceinline__ WordEntries decode_word(uint32_t w) {
    const uint32_t h0 = w & 0xFFFFu, h1 = w >> 16;
    const bool pair = (h0 & 0x8000u) != 0;
    WordEntries e;
    e.v0 = h0 != kNull16;
    e.t0 = h0 & 0x7FFFu;
    e.c0 = pair ? __uint2float_rn(h1) : 1.0f;
    e.v1 = !pair && h1 != kNull16;
    e.t1 = h1;
    return e;
}

template <bool kGlobalPhi>
__device__ __forceinline__ float acc_word_compact(float s, uint32_t w, const float* phi) {
    const WordEntries e = decode_word(w);
    float p0 = 0.0f, p1 = 0.0f;
    if (e.v0) p0 = ld_phi<kGlobalPhi>(phi, e.t0);
    if (e.v1) p1 = ld_phi<kGlobalPhi>(phi, e.t1);
    s = __fadd_rn(s, __fmul_rn(e.c0, p0));  // f32(1) * phi == phi; f32(c) * phi as the reference
    return __fadd_rn(s, p1);
}

template <bool kGlobalPhi>
__device__ __forceinline__ void scan_word_compact(float& run, bool& need, uint32_t& topic, float xs, uint32_t w,
                                                  const float* phi) {
    const WordEntries e = decode_word(w);
    float p0 = 0.0f, p1 = 0.0f;
    if (e.v0) p0 = ld_phi<kGlobalPhi>(phi, e.t0);
    if (e.v1) p1 = ld_phi<kGlobalPhi>(phi, e.t1);
    run = __fadd_rn(run, __fmul_rn(e.c0, p0));
    if (need && e.v0 && run >= xs) { topic = e.t0; need = false; }
    run = __fadd_rn(run, p1);
    if (need && e.v1 && run >= xs) { topic = e.t1; need = false; }
}

// First pass over one staged sector (32 bytes) of a row.  Sector 0 starts with the header
// (compact: skipped; wide: a count-0 entry that adds +0).
template <bool kGlobalPhi, bool kCompact>
__device__ __forceinline__ float acc_sector(float s, const unsigned char* p, uint32_t sec, uint32_t tbits,
                                            uint32_t tmask, const float* phi) {
    const uint4 lo = *reinterpret_cast<const uint4*>(p);
    const uint4 hi = *reinterpret_cast<const uint4*>(p + 16);
    if (kCompact) {
        if (sec != 0) s = acc_word_compact<kGlobalPhi>(s, lo.x, phi);
        s = acc_word_compact<kGlobalPhi>(s, lo.y, phi);
        s = acc_word_compact<kGlobalPhi>(s, lo.z, phi);
        s = acc_word_compact<kGlobalPhi>(s, lo.w, phi);
        s = acc_word_compact<kGlobalPhi>(s, hi.x, phi);
        s = acc_word_compact<kGlobalPhi>(s, hi.y, phi);
        s = acc_word_compact<kGlobalPhi>(s, hi.z, phi);
        return acc_word_compact<kGlobalPhi>(s, hi.w, phi);
    }
    s = acc_quad<kGlobalPhi>(s, lo, tbits, tmask, phi);
    return acc_quad<kGlobalPhi>(s, hi, tbits, tmask, phi);
}

// Prefix re-scan of one staged sector: first running sum >= xs.
template <bool kGlobalPhi, bool kCompact>
__device__ __forceinline__ void scan_sector(float& run, bool& need, uint32_t& topic, float xs,
                                            const unsigned char* p, uint32_t sec, uint32_t tbits,
                                            uint32_t tmask, const float* phi) {
    const uint4 lo = *reinterpret_cast<const uint4*>(p);
    const uint4 hi = *reinterpret_cast<const uint4*>(p + 16);
    const uint32_t es[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
#pragma unroll
    for (int w = 0; w < 8; ++w) {
        if (kCompact) {
            if (w > 0 || sec != 0) scan_word_compact<kGlobalPhi>(run, need, topic, xs, es[w], phi);
        } else {
            run = __fadd_rn(run, entry_mass<kGlobalPhi>(es[w], tbits, tmask, phi));
            if (need && run >= xs) {
                topic = es[w] & tmask;
                need = false;
            }
        }
    }
}

template <int NT, int G, int MINB, bool kGlobalPhi, bool kCompact>
__global__ void __launch_bounds__(NT, MINB) sampler_kernel(SamplerArgs a) {
    using St = Stage<G>;
    extern __shared__ __align__(16) float sm[];
    const uint32_t v = a.units[blockIdx.x].word;
    const float* s_bhat = kGlobalPhi ? a.bhat + static_cast<size_t>(v) * a.K_pad : sm;
    float* s_l8 = kGlobalPhi ? sm : sm + a.K_pad;  // l8_stride (L4[8j+7], padded with the total)
    float* s_ck = s_l8 + a.l8_stride;       // [kCkSectors][NT]
    unsigned char* s_stage = reinterpret_cast<unsigned char*>(s_ck + kCkSectors * NT);

    const Unit unit = a.units[blockIdx.x];
    const float* l4row = a.l4 + static_cast<size_t>(v) * a.K_pad;
    const float total = __ldg(l4row + a.K_pad - 1);  // padded with the row total
    {
        if (!kGlobalPhi) {
            const float4* gb = reinterpret_cast<const float4*>(a.bhat + static_cast<size_t>(v) * a.K_pad);
            float4* sb = reinterpret_cast<float4*>(sm);
            for (uint32_t i = threadIdx.x; i < a.K_pad / 4; i += NT) sb[i] = __ldg(gb + i);
        }
        const float4* gl = reinterpret_cast<const float4*>(a.l8 + static_cast<size_t>(v) * a.l8_stride);
        float4* sl = reinterpret_cast<float4*>(s_l8);
        for (uint32_t i = threadIdx.x; i < a.l8_stride / 4; i += NT) sl[i] = __ldg(gl + i);
    }
    const float qv = __ldg(a.q + v);
    uint32_t* brow = a.B + static_cast<size_t>(v) * a.K_pad;
    const uint32_t tbits = a.tbits;
    const uint32_t tmask = (1u << tbits) - 1u;
    const uint4* A4 = reinterpret_cast<const uint4*>(a.A);
    float* ck = s_ck + threadIdx.x;
    // Cooperative layout: lane -> row kRowsPerInst*j + lane%kRowsPerInst, sector
    // lane/kRowsPerInst.  A quarter warp then stores 8 different rows at the same sector
    // offset, which the (32G+16)-byte row stride spreads over all 32 banks.
    const uint32_t lane = lane_id(), sub = lane / St::kRowsPerInst, grp = lane % St::kRowsPerInst;
    unsigned char* stage = s_stage + (threadIdx.x >> 5) * St::kWarp;
    const unsigned char* mine = stage + lane * St::kRow;  // this lane's staged sectors
    unsigned long long entries = 0;
    __syncthreads();

    const uint32_t rounds = (unit.length + NT - 1) / NT;  // CTA-uniform
    for (uint32_t r = 0; r < rounds; ++r) {
        const uint32_t i = r * NT + threadIdx.x;
        const bool active = i < unit.length;
        const uint2 t = active ? __ldg(a.tok + unit.offset + i) : make_uint2(0u, 0u);  // {row quads, slot}
        uint32_t rq[G], ns[G], gs[G];
#pragma unroll
        for (uint32_t j = 0; j < G; ++j) {
            rq[j] = __shfl_sync(0xffffffffu, t.x, St::kRowsPerInst * j + grp);
            ns[j] = __shfl_sync(0xffffffffu, active ? G : 0u, St::kRowsPerInst * j + grp);  // speculative
            gs[j] = 0;
        }
        __syncwarp();
        stage_group<G>(A4, rq, ns, gs, sub, grp, stage);
        __syncwarp();

        // Wide row = [header (nnz-1, count 0) | entries | zero-count padding to 8]: header and
        // padding add +0 to every running sum.  Compact row: word 0 = nsect | nnz << 16.
        const uint32_t w0 = reinterpret_cast<const uint4*>(mine)->x;
        const uint32_t nnz = active ? (kCompact ? w0 >> 16 : (w0 & tmask) + 1u) : 0u;
        const uint32_t nsect = active ? (kCompact ? w0 & 0xFFFFu : (nnz + 8u) >> 3) : 0u;
        entries += nnz;
#pragma unroll
        for (uint32_t j = 0; j < G; ++j) ns[j] = __shfl_sync(0xffffffffu, nsect, St::kRowsPerInst * j + grp);
        const uint32_t ngroups = (nsect + G - 1) / G;
        const uint32_t max_groups = __reduce_max_sync(0xffffffffu, ngroups);

        float ub = 0.0f, up = 0.0f;
        if (active) {
            const uint64_t id = a.ids ? __ldg(a.ids + t.y) : a.id_base + t.y;
            draw2_f32(a.seed, a.stream_kind, id, ub, up);
        }

        // make_branch_context: S = sum_i f32(cnt_i) * bhat[top_i], sequential f32.
        // Group g+1 is loaded into registers while group g is consumed from the stage.
        float s = 0.0f;
        for (uint32_t g = 0; g < max_groups; ++g) {
            Sector next[G];
            const bool more = g + 1 < max_groups;
            if (more) {
#pragma unroll
                for (uint32_t j = 0; j < G; ++j) gs[j] = G * (g + 1);
                load_group<G>(A4, rq, ns, gs, sub, next);
            }
#pragma unroll
            for (uint32_t u = 0; u < G; ++u) {
                const uint32_t sec = G * g + u;
                if (sec < nsect) {
                    s = acc_sector<kGlobalPhi, kCompact>(s, mine + 32 * u, sec, tbits, tmask, s_bhat);
                    if (sec < kCkSectors) ck[sec * NT] = s;
                }
            }
            if (more) {
                __syncwarp();
                store_group<G>(next, ns, gs, sub, grp, stage);
                __syncwarp();
            }
        }

        uint32_t topic = 0;
        bool need = false;  // sparse branch still searching its prefix
        uint32_t sec = 0;
        float run = 0.0f, xs = 0.0f;
        if (active) {
            if (ub < __fdiv_rn(s, __fadd_rn(s, qv))) {
                // Sparse branch: first running prefix >= p*S (prefix_search, sampler.hpp:18-41).
                xs = __fmul_rn(up, s);
                if (xs == 0.0f) {
                    // every prefix is >= 0: the first real entry (word 1 in both formats)
                    const uint32_t e1 = __ldg(reinterpret_cast<const uint32_t*>(A4 + t.x) + 1);
                    topic = kCompact ? (e1 & 0x7FFFu) : (e1 & tmask);
                } else {
                    // The first sector whose end sum reaches xs holds the crossing; its re-scan
                    // restarts from the previous checkpoint, the same f32 value the first pass
                    // held there, so it is bit-identical.
                    const uint32_t stored = nsect < kCkSectors ? nsect : kCkSectors;
                    uint32_t lo = 0, hi = stored;  // first checkpoint >= xs (or stored)
                    while (lo < hi) {
                        const uint32_t mid = (lo + hi) >> 1;
                        if (ck[mid * NT] >= xs) hi = mid; else lo = mid + 1;
                    }
                    sec = lo;
                    run = lo > 0 ? ck[(lo - 1) * NT] : 0.0f;
                    need = true;
                }
            } else {
                // Word branch: WaryTree::sample(p * total) (sampler.hpp:100-106).
                float x = __fmul_rn(up, total);
                if (!(x <= total)) x = total;
                const uint32_t k = tree_search(x, s_l8, a.n_l8, l4row);
                topic = k < a.K ? k : a.K - 1;
            }
        }
        // Cooperative re-staging of the crossing sector of every searching lane.
        while (__any_sync(0xffffffffu, need)) {
            const uint32_t first = need ? sec : 0u;
            const uint32_t lim = need ? sec + 1 : 0u;
#pragma unroll
            for (uint32_t j = 0; j < G; ++j) {
                gs[j] = __shfl_sync(0xffffffffu, first, St::kRowsPerInst * j + grp);
                ns[j] = __shfl_sync(0xffffffffu, lim, St::kRowsPerInst * j + grp);
            }
            __syncwarp();
            stage_group<G>(A4, rq, ns, gs, sub, grp, stage);
            __syncwarp();
            if (need) {
                scan_sector<kGlobalPhi, kCompact>(run, need, topic, xs, mine, sec, tbits, tmask, s_bhat);
                ++sec;
            }
        }
        if (active) {
            a.z[t.y] = static_cast<uint16_t>(topic);
            atomicAdd(brow + topic, 1u);
        }
    }
    if (a.row_entries) {
        // One atomic per warp.
        for (int o = 16; o > 0; o >>= 1) entries += __shfl_xor_sync(0xffffffffu, entries, o);
        if (lane == 0) atomicAdd(a.row_entries, entries);
    }
}

// ---- K3' streaming sampler: the same draws, bit for bit, with lane refill -----------------------
// The round-based kernel above advances a warp's 32 tokens in lock step: every round waits for
// its longest row, re-reads the crossing sector with a second dependent round trip, and loads a
// speculative group for every row.  Here each lane owns a sequence of tokens instead: the
// warp streams G-sector groups of its lanes' CURRENT rows (cooperative, coalesced, next group
// prefetched in registers); a lane whose row ends takes the next token of the unit at once
// (warp ballot over a 32-token pool, CTA-wide dynamic batches), so the stream never waits for
// the longest row.  The branch decision needs the whole row (S), so a finished token's last
// step is deferred by one step: the one sector it still needs -- the sparse branch's crossing
// sector (found from the per-sector checkpoints) or the tree branch's L4 block -- is loaded
// lane-private in step t and resolved in step t+1, under the next step's consumption.
// Arithmetic (make_branch_context, prefix_search, WaryTree::sample) is unchanged.
template <int NT, int G>
__global__ void __launch_bounds__(NT, NT <= 128 ? 3 : 2) sampler_stream_kernel(SamplerArgs a) {
    using St = Stage<G>;
    extern __shared__ __align__(16) float sm[];
    __shared__ uint32_t s_next;  // next unclaimed 32-token batch (index within the unit)
    const Unit unit = a.units[blockIdx.x];
    const uint32_t v = unit.word;
    float* s_bhat = sm;
    float* s_l8 = sm + a.K_pad;
    float* s_ck = s_l8 + a.l8_stride;  // [kCkSectors][NT]
    unsigned char* s_stage = reinterpret_cast<unsigned char*>(s_ck + kCkSectors * NT);
    const float* l4row = a.l4 + static_cast<size_t>(v) * a.K_pad;
    const float total = __ldg(l4row + a.K_pad - 1);
    {
        const float4* gb = reinterpret_cast<const float4*>(a.bhat + static_cast<size_t>(v) * a.K_pad);
        float4* sb = reinterpret_cast<float4*>(sm);
        for (uint32_t i = threadIdx.x; i < a.K_pad / 4; i += NT) sb[i] = __ldg(gb + i);
        const float4* gl = reinterpret_cast<const float4*>(a.l8 + static_cast<size_t>(v) * a.l8_stride);
        float4* sl = reinterpret_cast<float4*>(s_l8);
        for (uint32_t i = threadIdx.x; i < a.l8_stride / 4; i += NT) sl[i] = __ldg(gl + i);
    }
    if (threadIdx.x == 0) s_next = NT;  // warp w starts with batch [32w, 32w + 32)
    const float qv = __ldg(a.q + v);
    uint32_t* brow = a.B + static_cast<size_t>(v) * a.K_pad;
    const uint32_t tbits = a.tbits, tmask = (1u << tbits) - 1u;
    const uint4* A4 = reinterpret_cast<const uint4*>(a.A);
    const uint2* toks = a.tok + unit.offset;
    const uint32_t len = unit.length;
    const uint32_t lane = lane_id(), sub = lane / St::kRowsPerInst, grp = lane % St::kRowsPerInst;
    unsigned char* stage = s_stage + (threadIdx.x >> 5) * St::kWarp;
    const unsigned char* mine = stage + lane * St::kRow;
    float* ck = s_ck + threadIdx.x;
    unsigned long long entries = 0;
    __syncthreads();

    // Token pool: pool = batch at pool_base (lane l holds token pool_base + l), nxt = the batch
    // after it; pc = tokens of the pool already handed out.
    uint32_t pool_base = (threadIdx.x >> 5) * 32u;
    uint2 pool = pool_base + lane < len ? __ldg(toks + pool_base + lane) : make_uint2(0u, 0u);
    auto claim = [&]() -> uint32_t {
        uint32_t b = 0;
        if (lane == 0) b = atomicAdd(&s_next, 32u);
        return __shfl_sync(0xffffffffu, b, 0);
    };
    uint32_t next_base = claim();
    uint2 nxt = next_base + lane < len ? __ldg(toks + next_base + lane) : make_uint2(0u, 0u);
    uint32_t pc = 0;

    // Current row (the one staged this step).
    bool cur = false, hdr = false;  // hdr: the staged group is the row's first (header unread)
    uint32_t c_rq = 0, c_slot = 0, c_ns = 0, c_base = 0;
    float s = 0.0f;
    // Pending resolution: 0 none, 1 sparse (scan sector p_sec from run p_run for xs), 2 tree
    // (L4 block p_sec), 3 sparse with xs == 0 (the first real entry).
    uint32_t p_kind = 0, p_slot = 0, p_sec = 0, p_rq = 0, p_ns = 0;
    float p_run = 0.0f, p_x = 0.0f;
    Sector psec = zero_sector();

    // Hands out tokens to the lanes in `need` (ballot), in lane order.
    auto take = [&](bool want, uint32_t& rq, uint32_t& slot) -> bool {
        const uint32_t need = __ballot_sync(0xffffffffu, want);
        const uint32_t idx = pc + __popc(need & ((1u << lane) - 1u));
        const uint2 ra = make_uint2(__shfl_sync(0xffffffffu, pool.x, idx & 31u),
                                    __shfl_sync(0xffffffffu, pool.y, idx & 31u));
        const uint2 rb = make_uint2(__shfl_sync(0xffffffffu, nxt.x, idx & 31u),
                                    __shfl_sync(0xffffffffu, nxt.y, idx & 31u));
        const uint32_t gi = idx < 32u ? pool_base + idx : next_base + (idx - 32u);
        const bool got = want && idx < 64u && gi < len;
        rq = idx < 32u ? ra.x : rb.x;
        slot = idx < 32u ? ra.y : rb.y;
        pc += __popc(need);
        if (pc >= 32u) {  // pool consumed: the next batch becomes the pool
            pc -= 32u;
            pool = nxt;
            pool_base = next_base;
            next_base = claim();
            nxt = next_base + lane < len ? __ldg(toks + next_base + lane) : make_uint2(0u, 0u);
        }
        return got;
    };

    // First tokens and their first groups.
    uint32_t t_rq = 0, t_slot = 0;
    cur = take(true, t_rq, t_slot);
    c_rq = t_rq;
    c_slot = t_slot;
    hdr = cur;
    {
        uint32_t rq[G], ns[G], gs[G];
#pragma unroll
        for (uint32_t j = 0; j < G; ++j) {
            rq[j] = __shfl_sync(0xffffffffu, c_rq, St::kRowsPerInst * j + grp);
            ns[j] = __shfl_sync(0xffffffffu, cur ? G : 0u, St::kRowsPerInst * j + grp);
            gs[j] = 0;
        }
        stage_group<G>(A4, rq, ns, gs, sub, grp, stage);
        __syncwarp();
    }

    while (__any_sync(0xffffffffu, cur || p_kind != 0)) {
        // Header of a row whose first group is staged: [nnz-1 | entries | zero pad].
        if (cur && hdr) {
            const uint32_t nnz = (reinterpret_cast<const uint4*>(mine)->x & tmask) + 1u;
            c_ns = (nnz + 8u) >> 3;
            entries += nnz;
            hdr = false;
        }
        // Next step's group per lane: the rest of this row, or the first group of a new token.
        const bool ends = cur && c_base + G >= c_ns;
        uint32_t n_rq = 0, n_slot = 0;
        const bool got = take(ends, n_rq, n_slot);
        uint32_t l_rq = 0, l_start = 0, l_lim = 0;
        if (cur && !ends) {
            l_rq = c_rq; l_start = c_base + G; l_lim = c_ns;
        } else if (got) {
            l_rq = n_rq; l_start = 0; l_lim = G;  // speculative first group (header inside)
        }
        uint32_t rq[G], ns[G], gs[G];
#pragma unroll
        for (uint32_t j = 0; j < G; ++j) {
            const uint32_t src = St::kRowsPerInst * j + grp;
            rq[j] = __shfl_sync(0xffffffffu, l_rq, src);
            gs[j] = __shfl_sync(0xffffffffu, l_start, src);
            ns[j] = __shfl_sync(0xffffffffu, l_lim, src);
        }
        Sector nx[G];
        load_group<G>(A4, rq, ns, gs, sub, nx);

        // make_branch_context over this step's sectors (sequential f32 chain).
        if (cur) {
#pragma unroll
            for (uint32_t u = 0; u < G; ++u) {
                const uint32_t sec = c_base + u;
                if (sec < c_ns) {
                    s = acc_sector<false, false>(s, mine + 32 * u, sec, tbits, tmask, s_bhat);
                    if (sec < kCkSectors) ck[sec * NT] = s;
                }
            }
        }

        // Resolve the token finished in the previous step (its sector arrived meanwhile).
        if (p_kind != 0) {
            uint32_t topic;
            if (p_kind == 2) {
                const float x = p_x;
                const uint32_t below = (__uint_as_float(psec.lo.x) < x) + (__uint_as_float(psec.lo.y) < x) +
                                       (__uint_as_float(psec.lo.z) < x) + (__uint_as_float(psec.lo.w) < x) +
                                       (__uint_as_float(psec.hi.x) < x) + (__uint_as_float(psec.hi.y) < x) +
                                       (__uint_as_float(psec.hi.z) < x) + (__uint_as_float(psec.hi.w) < x);
                const uint32_t k = p_sec * kLeaf + below;
                topic = k < a.K ? k : a.K - 1;
            } else if (p_kind == 3) {
                topic = psec.lo.y & tmask;  // word 1 of sector 0: the first real entry
            } else {
                // prefix_search (sampler.hpp:18-41) from the checkpoint: first running sum >= xs.
                float run = p_run;
                bool need = true;
                topic = 0;
                uint32_t sec = p_sec;
                Sector q = psec;
                while (true) {
                    const uint32_t es[8] = {q.lo.x, q.lo.y, q.lo.z, q.lo.w, q.hi.x, q.hi.y, q.hi.z, q.hi.w};
#pragma unroll
                    for (int w = 0; w < 8; ++w) {
                        run = __fadd_rn(run, entry_mass<false>(es[w], tbits, tmask, s_bhat));
                        if (need && run >= p_x) { topic = es[w] & tmask; need = false; }
                    }
                    if (!need || ++sec >= p_ns) break;
                    q = ldg_sector(A4 + p_rq + 2 * sec);  // crossing beyond the checkpoints (rare)
                }
            }
            a.z[p_slot] = static_cast<uint16_t>(topic);
            atomicAdd(brow + topic, 1u);
            p_kind = 0;
        }

        // A finished row: sample_token (sampler.hpp:183-204) up to its last sector read.
        if (ends) {
            float ub, up;
            const uint64_t id = a.ids ? __ldg(a.ids + c_slot) : a.id_base + c_slot;
            draw2_f32(a.seed, a.stream_kind, id, ub, up);
            p_slot = c_slot;
            if (ub < __fdiv_rn(s, __fadd_rn(s, qv))) {
                const float xs = __fmul_rn(up, s);
                if (xs == 0.0f) {
                    p_kind = 3;
                    p_sec = 0;
                    psec = ldg_sector(A4 + c_rq);
                } else {
                    const uint32_t stored = c_ns < kCkSectors ? c_ns : kCkSectors;
                    uint32_t lo = 0, hi = stored;  // first checkpoint >= xs (or stored)
                    while (lo < hi) {
                        const uint32_t mid = (lo + hi) >> 1;
                        if (ck[mid * NT] >= xs) hi = mid; else lo = mid + 1;
                    }
                    p_kind = 1;
                    p_sec = lo;
                    p_run = lo > 0 ? ck[(lo - 1) * NT] : 0.0f;
                    p_x = xs;
                    p_rq = c_rq;
                    p_ns = c_ns;
                    psec = ldg_sector(A4 + c_rq + 2 * lo);
                }
            } else {
                float x = __fmul_rn(up, total);  // WaryTree::sample(p * total)
                if (!(x <= total)) x = total;
                uint32_t lo = 0, hi = a.n_l8 - 1;
                while (lo < hi) {
                    const uint32_t mid = (lo + hi) >> 1;
                    if (s_l8[mid] >= x) hi = mid; else lo = mid + 1;
                }
                p_kind = 2;
                p_sec = lo;
                p_x = x;
                psec = ldg_sector(reinterpret_cast<const uint4*>(l4row + lo * kLeaf));
            }
            // The next token (if any) starts with the group loaded above.
            cur = got;
            c_rq = n_rq;
            c_slot = n_slot;
            c_base = 0;
            hdr = got;
            s = 0.0f;
        } else if (cur) {
            c_base += G;
        }
        __syncwarp();
        store_group<G>(nx, ns, gs, sub, grp, stage);
        __syncwarp();
    }
    if (a.row_entries) {
        for (int o = 16; o > 0; o >>= 1) entries += __shfl_xor_sync(0xffffffffu, entries, o);
        if (lane == 0) atomicAdd(a.row_entries, entries);
    }
}

// ---- K3'' quad-lane sampler: four lanes per token, no staging ----------------------------------
// The lane-per-token kernels must move every C_dk row through shared memory (cooperative
// coalesced loads land a row's sectors in OTHER lanes' registers), and their phi gathers run
// with a third of the lanes idle.  Here a warp samples 8 tokens at a time with 4 lanes each:
// one instruction loads one 128-byte line (4 sectors, 32 entries) of each of the 8 rows -- the
// rows are line-aligned -- straight into the registers of the 4 lanes that consume it, so
// there is no stage store/load at all, and every lane gathers phi for its own sector's 8
// entries (full-warp gathers).  The reference's sequential f32 chain (make_branch_context,
// sampler.hpp:166-178) is kept exactly: the products are formed in parallel, then the running
// sum visits the 4 sectors of a line in order -- lane j adds its 8 products to the value lane
// j-1 handed it (shuffle) -- so every intermediate is the reference's.  The per-sector sums
// double as the prefix_search checkpoints (a few hundred bytes per warp instead of a stage).
template <int NT, int MINB, int L, bool kCompact>
__global__ void __launch_bounds__(NT, MINB) sampler_quad_kernel(SamplerArgs a) {
    constexpr uint32_t NW = NT / 32;
    constexpr uint32_t TPR = 32u / L;  // tokens per round (L lanes each, L sectors per group)
    constexpr uint32_t kCk = 16;       // checkpointed sectors per token (128 entries)
    constexpr uint32_t kCkStride = 17; // odd: different tokens' checkpoints fall in different banks
    extern __shared__ __align__(16) float sm[];
    __shared__ uint32_t s_next;  // next unclaimed 32-token batch of the unit
    const Unit unit = a.units[blockIdx.x];
    const uint32_t v = unit.word;
    float* s_bhat = sm;
    float* s_l8 = sm + a.K_pad;
    float* s_ck = s_l8 + a.l8_stride;  // [NW][32 tokens][kCkStride]
    const float* l4row = a.l4 + static_cast<size_t>(v) * a.K_pad;
    const float total = __ldg(l4row + a.K_pad - 1);
    {
        const float4* gb = reinterpret_cast<const float4*>(a.bhat + static_cast<size_t>(v) * a.K_pad);
        float4* sb = reinterpret_cast<float4*>(sm);
        for (uint32_t i = threadIdx.x; i < a.K_pad / 4; i += NT) sb[i] = __ldg(gb + i);
        const float4* gl = reinterpret_cast<const float4*>(a.l8 + static_cast<size_t>(v) * a.l8_stride);
        float4* sl = reinterpret_cast<float4*>(s_l8);
        for (uint32_t i = threadIdx.x; i < a.l8_stride / 4; i += NT) sl[i] = __ldg(gl + i);
    }
    const float qv = __ldg(a.q + v);
    uint32_t* brow = a.B + static_cast<size_t>(v) * a.K_pad;
    const uint32_t tbits = a.tbits, tmask = (1u << tbits) - 1u;
    const uint4* A4 = reinterpret_cast<const uint4*>(a.A);
    const uint32_t lane = lane_id(), t = lane / L, sub = lane % L, lead = lane & ~(L - 1u);
    const uint32_t warp = threadIdx.x >> 5;
    float* ckw = s_ck + warp * 32u * kCkStride;
    unsigned long long entries = 0;
    if (threadIdx.x == 0) s_next = NW * 32u;
    __syncthreads();

    // A batch of 32 tokens per warp: L rounds of 32/L tokens x L lanes stream the rows and form
    // S; then lane l finishes token l of the batch (draws, branch, prefix search / tree).  The
    // first batch of warp w is tokens [32w, 32w + 32); later ones are claimed dynamically, so
    // the CTA's warps finish the unit together.
    for (uint32_t base = warp * 32u; base < unit.length;) {
        const bool mine = base + lane < unit.length;
        const uint2 tk = mine ? __ldg(a.tok + unit.offset + base + lane) : make_uint2(0u, 0u);  // {row quads, slot}
        float S = 0.0f;
        uint32_t my_ns = 0;
#pragma unroll 1
        for (uint32_t r = 0; r < L; ++r) {
            const uint32_t ti = TPR * r + t;  // this lane group's token within the batch
            if (__all_sync(0xffffffffu, base + TPR * r >= unit.length)) break;
            const bool act = base + ti < unit.length;
            const uint4* row = A4 + __shfl_sync(0xffffffffu, tk.x, ti);
            Sector c = zero_sector();
            if (act) c = ldg_sector(row + 2 * sub);
            const uint32_t hw = __shfl_sync(0xffffffffu, c.lo.x, lead);  // header: word 0 of sector 0
            // wide: [nnz-1 | entries | pad to 8]; compact: word 0 = nsect | nnz << 16
            const uint32_t nnz = act ? (kCompact ? hw >> 16 : (hw & tmask) + 1u) : 0u;
            const uint32_t nsect = act ? (kCompact ? hw & 0xFFFFu : (nnz + 8u) >> 3) : 0u;
            if (sub == 0) entries += nnz;
            const uint32_t max_groups = __reduce_max_sync(0xffffffffu, (nsect + L - 1u) / L);
            float* ck = ckw + ti * kCkStride;
            float run = 0.0f;
            // Products of this lane's sector, then the chain over the line's 4 sectors in order.
            auto consume = [&](const Sector& q, uint32_t g) {
                const uint32_t sec = L * g + sub;
                constexpr int NP = kCompact ? 16 : 8;  // products per sector
                float p[NP];
                if (sec < nsect) {
                    const uint32_t es[8] = {q.lo.x, q.lo.y, q.lo.z, q.lo.w, q.hi.x, q.hi.y, q.hi.z, q.hi.w};
                    if (kCompact) {
                        // Each word: (c0 * phi[t0]) then phi[t1]; absent entries are +0 (acc_word_compact).
#pragma unroll
                        for (int w = 0; w < 8; ++w) {
                            const WordEntries e = decode_word(es[w]);
                            const bool hdr = w == 0 && sec == 0;  // the header word
                            float p0 = 0.0f, p1 = 0.0f;
                            if (e.v0 && !hdr) p0 = s_bhat[e.t0];
                            if (e.v1 && !hdr) p1 = s_bhat[e.t1];
                            p[2 * w] = __fmul_rn(e.c0, p0);
                            p[2 * w + 1] = p1;
                        }
                    } else {
#pragma unroll
                        for (int w = 0; w < 8; ++w) p[w] = entry_mass<false>(es[w], tbits, tmask, s_bhat);
                    }
                }
#pragma unroll
                for (uint32_t j = 0; j < L; ++j) {
                    if (sub == j && sec < nsect) {
#pragma unroll
                        for (int w = 0; w < NP; ++w) run = __fadd_rn(run, p[w]);
                        if (sec < kCk) ck[sec] = run;
                    }
                    run = __shfl_sync(0xffffffffu, run, lead | j);
                }
            };
            for (uint32_t g = 0; g < max_groups; g += 2) {  // two groups per trip: no register copies
                Sector n = c;
                if (L * (g + 1) + sub < nsect) n = ldg_sector(row + 2 * (L * (g + 1) + sub));
                consume(c, g);
                if (g + 1 >= max_groups) break;
                if (L * (g + 2) + sub < nsect) c = ldg_sector(row + 2 * (L * (g + 2) + sub));
                consume(n, g + 1);
            }
            // Token ti's S and sector count to its owning lane (lane ti).
            const uint32_t src = ((lane - TPR * r) & (TPR - 1u)) * L;
            const float xS = __shfl_sync(0xffffffffu, run, src);
            const uint32_t xn = __shfl_sync(0xffffffffu, nsect, src);
            if (lane / TPR == r) {
                S = xS;
                my_ns = xn;
            }
        }
        __syncwarp();
        // sample_token (sampler.hpp:183-204), one token per lane.
        if (mine) {
            float ub, up;
            const uint64_t id = a.ids ? __ldg(a.ids + tk.y) : a.id_base + tk.y;
            draw2_f32(a.seed, a.stream_kind, id, ub, up);
            const uint4* row = A4 + tk.x;
            uint32_t topic = 0;
            if (ub < __fdiv_rn(S, __fadd_rn(S, qv))) {
                const float xs = __fmul_rn(up, S);
                if (xs == 0.0f) {
                    const uint32_t e1 = __ldg(reinterpret_cast<const uint32_t*>(row) + 1);  // first real entry
                    topic = kCompact ? (e1 & 0x7FFFu) : (e1 & tmask);
                } else {
                    const float* ck = ckw + lane * kCkStride;
                    const uint32_t stored = my_ns < kCk ? my_ns : kCk;
                    uint32_t lo = 0, hi = stored;  // first checkpoint >= xs (or stored)
                    while (lo < hi) {
                        const uint32_t mid = (lo + hi) >> 1;
                        if (ck[mid] >= xs) hi = mid; else lo = mid + 1;
                    }
                    float r = lo > 0 ? ck[lo - 1] : 0.0f;
                    for (uint32_t sc = lo; sc < my_ns; ++sc) {  // one sector unless past the checkpoints
                        const Sector q = ldg_sector(row + 2 * sc);
                        const uint32_t es[8] = {q.lo.x, q.lo.y, q.lo.z, q.lo.w, q.hi.x, q.hi.y, q.hi.z, q.hi.w};
                        bool found = false;
                        if (kCompact) {
                            bool need = true;
#pragma unroll
                            for (int w = 0; w < 8; ++w)
                                if (w > 0 || sc != 0) scan_word_compact<false>(r, need, topic, xs, es[w], s_bhat);
                            found = !need;
                        } else {
#pragma unroll
                            for (int w = 0; w < 8; ++w) {
                                r = __fadd_rn(r, entry_mass<false>(es[w], tbits, tmask, s_bhat));
                                if (!found && r >= xs) { topic = es[w] & tmask; found = true; }
                            }
                        }
                        if (found) break;
                    }
                }
            } else {
                float x = __fmul_rn(up, total);  // WaryTree::sample(p * total)
                if (!(x <= total)) x = total;
                const uint32_t k = tree_search(x, s_l8, a.n_l8, l4row);
                topic = k < a.K ? k : a.K - 1;
            }
            a.z[tk.y] = static_cast<uint16_t>(topic);
            atomicAdd(brow + topic, 1u);
        }
        uint32_t nb = 0;
        if (lane == 0) nb = atomicAdd(&s_next, 32u);
        base = __shfl_sync(0xffffffffu, nb, 0);
    }
    if (a.row_entries) {
        for (int o = 16; o > 0; o >>= 1) entries += __shfl_xor_sync(0xffffffffu, entries, o);
        if (lane == 0) atomicAdd(a.row_entries, entries);
    }
}

// The same algorithm with the next round's first line prefetched in each round's last group
// slot and the next batch claimed a batch ahead; the per-unit scalars live in shared memory to
// make room in the 64-register budget (C3 K=10K: 95.5 -> 92.8 ms; C2: 19.8 -> 20.5 ms).
template <int NT, int MINB, int L, bool kCompact, bool kPrefetchNext = true>
__global__ void __launch_bounds__(NT, MINB) sampler_quad_pf_kernel(SamplerArgs a) {
    constexpr uint32_t NW = NT / 32;
    constexpr uint32_t TPR = 32u / L;  // tokens per round (L lanes each, L sectors per group)
    constexpr uint32_t kCk = 16;       // checkpointed sectors per token (128 entries)
    constexpr uint32_t kCkStride = 17; // odd: different tokens' checkpoints fall in different banks
    extern __shared__ __align__(16) float sm[];
    __shared__ uint32_t s_next;  // next unclaimed 32-token batch of the unit
    __shared__ float s_total, s_qv;  // the word's tree total and Q_v (read in the sampling step only)
    const Unit unit = a.units[blockIdx.x];
    const uint32_t v = unit.word;
    float* s_bhat = sm;
    float* s_l8 = sm + a.K_pad;
    float* s_ck = s_l8 + a.l8_stride;  // [NW][32 tokens][kCkStride]
    {
        const float4* gb = reinterpret_cast<const float4*>(a.bhat + static_cast<size_t>(v) * a.K_pad);
        float4* sb = reinterpret_cast<float4*>(sm);
        for (uint32_t i = threadIdx.x; i < a.K_pad / 4; i += NT) sb[i] = __ldg(gb + i);
        const float4* gl = reinterpret_cast<const float4*>(a.l8 + static_cast<size_t>(v) * a.l8_stride);
        float4* sl = reinterpret_cast<float4*>(s_l8);
        for (uint32_t i = threadIdx.x; i < a.l8_stride / 4; i += NT) sl[i] = __ldg(gl + i);
    }
    const uint32_t tbits = a.tbits, tmask = (1u << tbits) - 1u;
    const uint4* A4 = reinterpret_cast<const uint4*>(a.A);
    const uint32_t lane = lane_id(), t = lane / L, sub = lane % L, lead = lane & ~(L - 1u);
    const uint32_t warp = threadIdx.x >> 5;
    float* ckw = s_ck + warp * 32u * kCkStride;
    uint32_t entries = 0;
    if (threadIdx.x == 0) {
        s_next = NW * 32u;
        s_total = __ldg(a.l4 + static_cast<size_t>(v) * a.K_pad + a.K_pad - 1);  // padded with the total
        s_qv = __ldg(a.q + v);
    }
    __syncthreads();

    // A batch of 32 tokens per warp: L rounds of 32/L tokens x L lanes stream the rows and form
    // S; then lane l finishes token l of the batch (draws, branch, prefix search / tree).  The
    // first batch of warp w is tokens [32w, 32w + 32); later ones are claimed dynamically, so
    // the CTA's warps finish the unit together.
    // The next batch is claimed when a batch starts, and each round's last group slot loads
    // the NEXT round's first line (its header sets that round's length), so rounds never start
    // on an exposed load.
    uint32_t base = warp * 32u;
    uint2 tk = base + lane < unit.length ? __ldg(a.tok + unit.offset + base + lane) : make_uint2(0u, 0u);
    Sector c = zero_sector();
    if (kPrefetchNext) {
        const uint32_t rq0 = __shfl_sync(0xffffffffu, tk.x, t);
        if (base + t < unit.length) c = ldg_sector(A4 + rq0 + 2 * sub);
    }
    while (base < unit.length) {
        const bool mine = base + lane < unit.length;
        uint32_t nb = 0;
        uint2 tk_nx = make_uint2(0u, 0u);
        if (kPrefetchNext) {  // claim the next batch now and load its token records
            if (lane == 0) nb = atomicAdd(&s_next, 32u);
            nb = __shfl_sync(0xffffffffu, nb, 0);
            if (nb + lane < unit.length) tk_nx = __ldg(a.tok + unit.offset + nb + lane);
        }
        float S = 0.0f;
        uint32_t my_ns = 0;
#pragma unroll 1
        for (uint32_t r = 0; r < L; ++r) {
            const uint32_t ti = TPR * r + t;  // this lane group's token within the batch
            if (__all_sync(0xffffffffu, base + TPR * r >= unit.length)) break;
            const bool act = base + ti < unit.length;
            const uint4* row = A4 + __shfl_sync(0xffffffffu, tk.x, ti);
            if (!kPrefetchNext) {  // this round's first line, loaded now
                c = zero_sector();
                if (act) c = ldg_sector(row + 2 * sub);
            }
            const uint32_t hw = __shfl_sync(0xffffffffu, c.lo.x, lead);  // header: word 0 of sector 0
            // wide: [nnz-1 | entries | pad to 8]; compact: word 0 = nsect | nnz << 16
            const uint32_t nnz = act ? (kCompact ? hw >> 16 : (hw & tmask) + 1u) : 0u;
            const uint32_t nsect = act ? (kCompact ? hw & 0xFFFFu : (nnz + 8u) >> 3) : 0u;
            if (sub == 0) entries += nnz;
            const uint32_t max_groups = __reduce_max_sync(0xffffffffu, (nsect + L - 1u) / L);
            float* ck = ckw + ti * kCkStride;
            float run = 0.0f;
            // Products of this lane's sector, then the chain over the line's 4 sectors in order.
            auto consume = [&](const Sector& q, uint32_t g) {
                const uint32_t sec = L * g + sub;
                constexpr int NP = kCompact ? 16 : 8;  // products per sector
                float p[NP];
                if (sec < nsect) {
                    const uint32_t es[8] = {q.lo.x, q.lo.y, q.lo.z, q.lo.w, q.hi.x, q.hi.y, q.hi.z, q.hi.w};
                    if (kCompact) {
                        // Each word: (c0 * phi[t0]) then phi[t1]; absent entries are +0 (acc_word_compact).
#pragma unroll
                        for (int w = 0; w < 8; ++w) {
                            const WordEntries e = decode_word(es[w]);
                            const bool hdr = w == 0 && sec == 0;  // the header word
                            float p0 = 0.0f, p1 = 0.0f;
                            if (e.v0 && !hdr) p0 = s_bhat[e.t0];
                            if (e.v1 && !hdr) p1 = s_bhat[e.t1];
                            p[2 * w] = __fmul_rn(e.c0, p0);
                            p[2 * w + 1] = p1;
                        }
                    } else {
#pragma unroll
                        for (int w = 0; w < 8; ++w) p[w] = entry_mass<false>(es[w], tbits, tmask, s_bhat);
                    }
                }
#pragma unroll
                for (uint32_t j = 0; j < L; ++j) {
                    if (sub == j && sec < nsect) {
#pragma unroll
                        for (int w = 0; w < NP; ++w) run = __fadd_rn(run, p[w]);
                        if (sec < kCk) ck[sec] = run;
                    }
                    run = __shfl_sync(0xffffffffu, run, lead | j);
                }
            };
            // Group g+1 (or the next round's first line) loads while group g is consumed; two
            // groups per trip so no registers are copied.
            auto fetch = [&](uint32_t g, Sector& dst) {
                if (g < max_groups) {  // warp-uniform
                    if (L * g + sub < nsect) dst = ldg_sector(row + 2 * (L * g + sub));
                } else if (kPrefetchNext) {
                    const bool last = r + 1 == L || base + TPR * (r + 1) >= unit.length;
                    const uint32_t nrq = __shfl_sync(0xffffffffu, last ? tk_nx.x : tk.x, last ? t : ti + TPR);
                    if (last ? nb + t < unit.length : base + ti + TPR < unit.length)
                        dst = ldg_sector(A4 + nrq + 2 * sub);
                }
            };
            if (max_groups == 0) {
                fetch(0, c);
            } else {
                Sector n = c;
                for (uint32_t g = 0;; g += 2) {
                    fetch(g + 1, n);
                    consume(c, g);
                    if (g + 1 >= max_groups) { c = n; break; }
                    fetch(g + 2, c);
                    consume(n, g + 1);
                    if (g + 2 >= max_groups) break;
                }
            }
            // Token ti's S and sector count to its owning lane (lane ti).
            const uint32_t src = ((lane - TPR * r) & (TPR - 1u)) * L;
            const float xS = __shfl_sync(0xffffffffu, run, src);
            const uint32_t xn = __shfl_sync(0xffffffffu, nsect, src);
            if (lane / TPR == r) {
                S = xS;
                my_ns = xn;
            }
        }
        __syncwarp();
        // sample_token (sampler.hpp:183-204), one token per lane.
        if (mine) {
            const float qv = s_qv, total = s_total;
            const float* l4row = a.l4 + static_cast<size_t>(v) * a.K_pad;
            float ub, up;
            const uint64_t id = a.ids ? __ldg(a.ids + tk.y) : a.id_base + tk.y;
            draw2_f32(a.seed, a.stream_kind, id, ub, up);
            const uint4* row = A4 + tk.x;
            uint32_t topic = 0;
            if (ub < __fdiv_rn(S, __fadd_rn(S, qv))) {
                const float xs = __fmul_rn(up, S);
                if (xs == 0.0f) {
                    const uint32_t e1 = __ldg(reinterpret_cast<const uint32_t*>(row) + 1);  // first real entry
                    topic = kCompact ? (e1 & 0x7FFFu) : (e1 & tmask);
                } else {
                    const float* ck = ckw + lane * kCkStride;
                    const uint32_t stored = my_ns < kCk ? my_ns : kCk;
                    uint32_t lo = 0, hi = stored;  // first checkpoint >= xs (or stored)
                    while (lo < hi) {
                        const uint32_t mid = (lo + hi) >> 1;
                        if (ck[mid] >= xs) hi = mid; else lo = mid + 1;
                    }
                    float r = lo > 0 ? ck[lo - 1] : 0.0f;
                    for (uint32_t sc = lo; sc < my_ns; ++sc) {  // one sector unless past the checkpoints
                        const Sector q = ldg_sector(row + 2 * sc);
                        const uint32_t es[8] = {q.lo.x, q.lo.y, q.lo.z, q.lo.w, q.hi.x, q.hi.y, q.hi.z, q.hi.w};
                        bool found = false;
                        if (kCompact) {
                            bool need = true;
#pragma unroll
                            for (int w = 0; w < 8; ++w)
                                if (w > 0 || sc != 0) scan_word_compact<false>(r, need, topic, xs, es[w], s_bhat);
                            found = !need;
                        } else {
#pragma unroll
                            for (int w = 0; w < 8; ++w) {
                                r = __fadd_rn(r, entry_mass<false>(es[w], tbits, tmask, s_bhat));
                                if (!found && r >= xs) { topic = es[w] & tmask; found = true; }
                            }
                        }
                        if (found) break;
                    }
                }
            } else {
                float x = __fmul_rn(up, total);  // WaryTree::sample(p * total)
                if (!(x <= total)) x = total;
                const uint32_t k = tree_search(x, s_l8, a.n_l8, l4row);
                topic = k < a.K ? k : a.K - 1;
            }
            a.z[tk.y] = static_cast<uint16_t>(topic);
            atomicAdd(a.B + static_cast<size_t>(v) * a.K_pad + topic, 1u);
        }
        if (kPrefetchNext) {
            base = nb;
            tk = tk_nx;
        } else {
            if (lane == 0) nb = atomicAdd(&s_next, 32u);
            base = __shfl_sync(0xffffffffu, nb, 0);
            tk = base + lane < unit.length ? __ldg(a.tok + unit.offset + base + lane) : make_uint2(0u, 0u);
        }
    }
    if (a.row_entries) {
        for (int o = 16; o > 0; o >>= 1) entries += __shfl_xor_sync(0xffffffffu, entries, o);
        if (lane == 0) atomicAdd(a.row_entries, static_cast<unsigned long long>(entries));
    }
}

size_t sampler_smem(const SamplerArgs& a, int nt, int g, bool global_phi) {
    const size_t stage_row = 32u * static_cast<size_t>(g) + 16u;
    return sizeof(float) * ((global_phi ? 0 : static_cast<size_t>(a.K_pad)) + a.l8_stride) +
           (sizeof(float) * kCkSectors + stage_row) * static_cast<size_t>(nt);
}

template <int NT, int G, int MINB, bool Gl, bool C>
cudaError_t launch_sampler_t(const SamplerArgs& a, uint32_t n_units, cudaStream_t s) {
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(sampler_kernel<NT, G, MINB, Gl, C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             227 * 1024);
        configured = true;
    }
    sampler_kernel<NT, G, MINB, Gl, C><<<n_units, NT, sampler_smem(a, NT, G, Gl), s>>>(a);
    return cudaGetLastError();
}

template <int NT, int G>
cudaError_t launch_stream_t(const SamplerArgs& a, uint32_t n_units, cudaStream_t s) {
    static bool configured = false;
    if (!configured) {
        // 227 KB per block minus the kernel's static shared memory (the batch counter).
        const cudaError_t e = cudaFuncSetAttribute(sampler_stream_kernel<NT, G>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    sampler_stream_kernel<NT, G><<<n_units, NT, sampler_smem(a, NT, G, false), s>>>(a);
    return cudaGetLastError();
}

int sampler_shape_from_name(const char* name) {
    const std::string v(name ? name : "");
    return v == "g2" ? 0 : v == "g4" ? 1 : v == "g4x512" ? 2 : v == "s4" ? 3 : v == "s2" ? 4 : v == "s4x128" ? 5
         : v == "q512" ? 6 : v == "q256" ? 7 : v == "q512r" ? 8 : v == "q256r" ? 9
         : v == "p512" ? 10 : v == "p256" ? 11 : v == "o512" ? 12 : -1;
}

size_t sampler_quad_smem(const SamplerArgs& a, int nt) {
    return sizeof(float) * (static_cast<size_t>(a.K_pad) + a.l8_stride + static_cast<size_t>(nt / 32) * 32u * 17u);
}

template <int NT, int MINB, int L, bool C, bool PF>
cudaError_t launch_quad_t1(const SamplerArgs& a, uint32_t n_units, cudaStream_t s) {
    static bool configured = false;
    auto kern = PF ? sampler_quad_pf_kernel<NT, MINB, L, C> : sampler_quad_kernel<NT, MINB, L, C>;
    if (!configured) {
        // 227 KB per block minus the kernel's static shared memory (the batch counter).
        const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    kern<<<n_units, NT, sampler_quad_smem(a, NT), s>>>(a);
    return cudaGetLastError();
}
// PF: the next round's first line is prefetched in each round's last group slot (C3 K=10K:
// 95.5 -> 92.8 ms; short-phi C2: 19.8 -> 20.5 ms, so only the 512-thread shape uses it).
template <int NT, int MINB, int L = 4, bool PF = (NT >= 512)>
cudaError_t launch_quad_t(const SamplerArgs& a, uint32_t n_units, cudaStream_t s) {
    return a.compact ? launch_quad_t1<NT, MINB, L, true, PF>(a, n_units, s)
                     : launch_quad_t1<NT, MINB, L, false, PF>(a, n_units, s);
}

// Launch shape (SLDA_SAMPLER overrides for experiments; default by phi row size):
//   "g2"     : round-based, 256/512-thread CTAs, 2-sector groups, 64 registers
//   "g4"     : round-based, 256-thread CTAs, 4-sector groups, up to 128 registers
//   "g4x512" : round-based, 512-thread CTAs, 4-sector groups (one CTA / SM at K = 10K)
//   "s4", "s2", "s4x128" : streaming lane refill (sampler_stream_kernel)
//   "q512", "q256"       : quad-lane (sampler_quad_kernel, L=4 lanes per token), 64 registers
//   "p512", "p256"       : pair-lane (L=2; C2 20.7 vs 21.5 ms, C3 107.9 vs 100.0 ms)
//   "o512"               : octet-lane (L=8; slower at both)
//   "q512r", "q256r"     : quad-lane with a relaxed register bound (fewer warps; slower)
cudaError_t launch_sampler(const SamplerArgs& a, uint32_t n_units, cudaStream_t s) {
    if (n_units == 0) return cudaSuccess;
    const size_t phi_bytes = sizeof(float) * (static_cast<size_t>(a.K_pad) + a.l8_stride);
    // Default: the quad-lane kernel wherever two 512-thread (or four 256-thread) CTAs fit an SM
    // (C3 K=10K: 100.0 vs 102.6 ms for 4-sector groups; C2 K=1K: 21.5 vs 23.5 ms for 2-sector
    // groups), else 4-sector groups (large phi rows), else 2-sector groups.
    int shape = a.shape;
    if (shape < 0) {
        if (phi_bytes <= 24 * 1024 && 4 * sampler_quad_smem(a, 256) <= 227 * 1024) shape = 7;
        else if (2 * sampler_quad_smem(a, 512) <= 227 * 1024) shape = 6;
    }
    if (shape < 0) shape = phi_bytes > 24 * 1024 ? 1 : 0;
    const bool fits512 = sampler_smem(a, 512, 2, false) <= 227 * 1024;
    if (!fits512) {
        // Rows that do not fit shared memory (K > kCompactMaxK, so always the wide format):
        // gather phi through L1/L2.
        if (a.compact) return cudaErrorInvalidConfiguration;
        return launch_sampler_t<512, 2, 2, true, false>(a, n_units, s);
    }
    if (shape == 6 && sampler_quad_smem(a, 512) <= 227 * 1024)
        return launch_quad_t<512, 2>(a, n_units, s);
    if (shape == 7 && sampler_quad_smem(a, 256) <= 227 * 1024)
        return launch_quad_t<256, 4>(a, n_units, s);
    if (shape == 8 && sampler_quad_smem(a, 512) <= 227 * 1024)
        return launch_quad_t<512, 1>(a, n_units, s);
    if (shape == 9 && sampler_quad_smem(a, 256) <= 227 * 1024)
        return launch_quad_t<256, 3>(a, n_units, s);
    if (shape == 10 && sampler_quad_smem(a, 512) <= 227 * 1024)
        return launch_quad_t<512, 2, 2>(a, n_units, s);
    if (shape == 11 && sampler_quad_smem(a, 256) <= 227 * 1024)
        return launch_quad_t<256, 4, 2>(a, n_units, s);
    if (shape == 12 && sampler_quad_smem(a, 512) <= 227 * 1024)
        return launch_quad_t<512, 2, 8>(a, n_units, s);
    if (!a.compact && shape == 3 && sampler_smem(a, 256, 4, false) <= 227 * 1024)
        return launch_stream_t<256, 4>(a, n_units, s);
    if (!a.compact && shape == 4 && sampler_smem(a, 256, 2, false) <= 227 * 1024)
        return launch_stream_t<256, 2>(a, n_units, s);
    if (!a.compact && shape == 5 && sampler_smem(a, 128, 4, false) <= 227 * 1024)
        return launch_stream_t<128, 4>(a, n_units, s);
    if (shape == 1 && sampler_smem(a, 256, 4, false) <= 227 * 1024)
        return a.compact ? launch_sampler_t<256, 4, 2, false, true>(a, n_units, s)
                         : launch_sampler_t<256, 4, 2, false, false>(a, n_units, s);
    if (shape == 2 && sampler_smem(a, 512, 4, false) <= 227 * 1024)
        return a.compact ? launch_sampler_t<512, 4, 1, false, true>(a, n_units, s)
                         : launch_sampler_t<512, 4, 1, false, false>(a, n_units, s);
    // Small phi rows: 256-thread CTAs.  Large (K = 10K): 512 threads share one staged row
    // (2 CTAs x 16 warps per SM).
    if (phi_bytes <= 24 * 1024)
        return a.compact ? launch_sampler_t<256, 2, 4, false, true>(a, n_units, s)
                         : launch_sampler_t<256, 2, 4, false, false>(a, n_units, s);
    return a.compact ? launch_sampler_t<512, 2, 2, false, true>(a, n_units, s)
                     : launch_sampler_t<512, 2, 2, false, false>(a, n_units, s);
}

// ============================================================================
// K4 SSC -- rebuild_doc_topic (counts.cpp:103-125) + segmented_count (:65-94).
// Topics are already doc-grouped (the sampler writes them by slot), so the
// shuffle is fused into the sampler's store.  Warp per document: bitonic sort
// in shared memory, then a ballot run-length pass emitting (topic asc, count).
// Long documents: CTA per document, K-bin histogram + ordered compaction.
// ============================================================================

constexpr int kSscWarps = 8;

// Ascending bitonic sort of N = 32*R keys held striped across the warp (key i in lane
// i % 32, register i / 32): cross-lane stages exchange through shuffles, in-lane stages
// swap registers.  Integer keys, so any correct sort is bit-identical to std::sort.
// In-lane stage (partner distance j = 32*RJ): registers r and r|RJ.
template <int R, int RJ>
__device__ __forceinline__ void bitonic_inlane(uint32_t (&key)[R], uint32_t lane, uint32_t k) {
#pragma unroll
    for (uint32_t r = 0; r < R; ++r) {
        if ((r & RJ) == 0) {
            const uint32_t i = r * 32 + lane;
            const bool up = (i & k) == 0;
            const uint32_t a = key[r], b = key[r | RJ];
            const uint32_t lo = min(a, b), hi = max(a, b);
            key[r] = up ? lo : hi;
            key[r | RJ] = up ? hi : lo;
        }
    }
}

// Stage loops are not unrolled (only the register dimension is), which keeps the five
// instantiations within the instruction cache.
template <int R>
__device__ __forceinline__ void warp_bitonic(uint32_t (&key)[R], uint32_t lane) {
#pragma unroll 1
    for (uint32_t k = 2; k <= 32u * R; k <<= 1) {
#pragma unroll 1
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            if (j >= 32) {
                switch (j >> 5) {
                    case 1: bitonic_inlane<R, 1>(key, lane, k); break;
                    case 2: if (R > 2) bitonic_inlane<R, (R > 2 ? 2 : 1)>(key, lane, k); break;
                    case 4: if (R > 4) bitonic_inlane<R, (R > 4 ? 4 : 1)>(key, lane, k); break;
                    default: if (R > 8) bitonic_inlane<R, (R > 8 ? 8 : 1)>(key, lane, k); break;
                }
            } else {
                const bool lower = (lane & j) == 0;
#pragma unroll
                for (uint32_t r = 0; r < R; ++r) {
                    const uint32_t i = r * 32 + lane;
                    const bool up = (i & k) == 0;
                    const uint32_t other = __shfl_xor_sync(0xffffffffu, key[r], j);
                    key[r] = (up == lower) ? min(key[r], other) : max(key[r], other);
                }
            }
        }
    }
}

// ---- Compact C_dk rows: encoder (format: kNull16 above) -------------------------------------

// Appends up to 32 entries (lane-ordered; invalid lanes skipped) at slot `pos` (warp-uniform,
// advanced).  Slot positions come from a warp scan over the parity automaton
// single: (adv 1, parity flips), pair: (adv 2 + parity, parity -> 0).
__device__ __noinline__ void compact_chunk(uint16_t* row16, uint32_t& pos, bool valid, uint32_t topic,
                                           uint32_t count, uint32_t lane) {
    const bool pair = valid && count > 1;
    // f(p) for p in {0, 1}: advance a_p (8 bits each; <= 96 per chunk), parity out q_p,
    // packed as a0 | a1 << 8 | q0 << 16 | q1 << 17.  Identity for invalid lanes.
    uint32_t f = valid ? (pair ? (2u | 3u << 8) : (1u | 1u << 8 | 1u << 16)) : (1u << 17);
#pragma unroll
    for (uint32_t o = 1; o < 32; o <<= 1) {
        const uint32_t b = __shfl_up_sync(0xffffffffu, f, o);
        if (lane >= o) {  // earlier lanes (b) first, then this one (f)
            const uint32_t r0 = (b >> 16) & 1u, r1 = (b >> 17) & 1u;
            const uint32_t n0 = (b & 0xFFu) + ((r0 ? f >> 8 : f) & 0xFFu);
            const uint32_t n1 = ((b >> 8) & 0xFFu) + ((r1 ? f >> 8 : f) & 0xFFu);
            const uint32_t m0 = r0 ? (f >> 17) & 1u : (f >> 16) & 1u;
            const uint32_t m1 = r1 ? (f >> 17) & 1u : (f >> 16) & 1u;
            f = n0 | n1 << 8 | m0 << 16 | m1 << 17;
        }
    }
    const uint32_t p = pos & 1u;
    const uint32_t ex = __shfl_up_sync(0xffffffffu, f, 1);
    const uint32_t start = pos + (lane == 0 ? 0u : ((p ? ex >> 8 : ex) & 0xFFu));
    if (valid) {
        if (pair) {
            uint32_t s = start;
            if (s & 1u) row16[s++] = static_cast<uint16_t>(kNull16);
            row16[s] = static_cast<uint16_t>(0x8000u | topic);
            row16[s + 1] = static_cast<uint16_t>(count);
        } else {
            row16[start] = static_cast<uint16_t>(topic);
        }
    }
    const uint32_t tot = __shfl_sync(0xffffffffu, f, 31);
    pos += (p ? tot >> 8 : tot) & 0xFFu;
}

// Closes a compact row: null slots to the sector end, header word.
__device__ __forceinline__ void compact_finish(uint16_t* row16, uint32_t pos, uint32_t nnz, uint32_t lane) {
    const uint32_t end = (pos + 15u) & ~15u;
    for (uint32_t s = pos + lane; s < end; s += 32) row16[s] = static_cast<uint16_t>(kNull16);
    if (lane == 0) reinterpret_cast<uint32_t*>(row16)[0] = (end >> 4) | (nnz << 16);
}

// One document of n <= 32*R tokens: sort, run-length, write the C_dk row (header, entries,
// padding to a sector).  starts: per-warp scratch of >= n words.  Returns nnz.
template <int R, bool kCompact>
__device__ __forceinline__ uint32_t ssc_doc(const uint16_t* z, uint32_t n, uint32_t lane, uint32_t* starts,
                                            uint32_t* out_row, uint32_t tbits) {
    uint32_t key[R];
#pragma unroll
    for (uint32_t r = 0; r < R; ++r) {
        const uint32_t i = r * 32 + lane;
        key[r] = i < n ? static_cast<uint32_t>(z[i]) : 0xFFFFFFFFu;
    }
    warp_bitonic<R>(key, lane);
    // Run starts in sorted order (i == r*32 + lane).
    uint32_t nnz = 0;
#pragma unroll
    for (uint32_t r = 0; r < R; ++r) {
        const uint32_t i = r * 32 + lane;
        const uint32_t up1 = __shfl_up_sync(0xffffffffu, key[r], 1);
        const uint32_t last = __shfl_sync(0xffffffffu, key[r > 0 ? r - 1 : 0], 31);
        const uint32_t prev = lane != 0 ? up1 : (r == 0 ? 0xFFFFFFFEu : last);
        const bool start = i < n && (i == 0 || key[r] != prev);
        const uint32_t ballot = __ballot_sync(0xffffffffu, start);
        if (start) starts[nnz + __popc(ballot & ((1u << lane) - 1u))] = i;
        nnz += __popc(ballot);
        if (32u * (r + 1) >= n) break;
    }
    __syncwarp();
    // Entries: topic of the run's first key, count = distance to the next start.  The sorted
    // keys are gone from smem, so the topic is recovered from the start position's lane.
    uint16_t* row16 = reinterpret_cast<uint16_t*>(out_row);
    uint32_t pos = 2;  // compact: slots 0-1 are the header word
    for (uint32_t base = 0; base < nnz; base += 32) {
        const uint32_t e = base + lane;
        const uint32_t st = e < nnz ? starts[e] : 0u;
        const uint32_t en = e + 1 < nnz ? starts[e + 1] : n;
        // key at sorted position st lives in lane st % 32, register st / 32.
        uint32_t topic = 0;
#pragma unroll
        for (uint32_t r = 0; r < R; ++r) {
            const uint32_t kv = __shfl_sync(0xffffffffu, key[r], st & 31u);
            if ((st >> 5) == r) topic = kv;
        }
        if (kCompact) compact_chunk(row16, pos, e < nnz, topic, en - st, lane);
        else if (e < nnz) out_row[1 + e] = topic | ((en - st) << tbits);
    }
    if (kCompact) {
        compact_finish(row16, pos, nnz, lane);
    } else {
        const uint32_t padded = (nnz + 8u) & ~7u;
        for (uint32_t e = nnz + 1 + lane; e < padded; e += 32) out_row[e] = 0u;
        if (lane == 0) out_row[0] = nnz - 1u;
    }
    __syncwarp();
    return nnz;
}

template <bool kCompact>
__global__ void __launch_bounds__(kSscWarps * 32) ssc_warp_kernel(SscArgs a) {
    __shared__ uint32_t s_start[kSscWarps][kSscWarpCap];
    const uint32_t w = threadIdx.x >> 5, lane = lane_id();
    uint32_t* starts = s_start[w];
    unsigned long long nnz_acc = 0;
    const uint32_t gw = blockIdx.x * kSscWarps + w, nw = gridDim.x * kSscWarps;
    for (uint32_t d = gw; d < a.D; d += nw) {
        const uint32_t s0 = __ldg(a.doc_start + d);
        const uint32_t n = __ldg(a.doc_start + d + 1) - s0;
        if (n > kSscWarpCap || n == 0) continue;  // ssc_long_kernel / empty document
        uint32_t* row = a.A + __ldg(a.row4 + d) * 4u;
        const uint16_t* z = a.z + s0;
        uint32_t nnz;
        if (n <= 32) nnz = ssc_doc<1, kCompact>(z, n, lane, starts, row, a.tbits);
        else if (n <= 64) nnz = ssc_doc<2, kCompact>(z, n, lane, starts, row, a.tbits);
        else if (n <= 128) nnz = ssc_doc<4, kCompact>(z, n, lane, starts, row, a.tbits);
        else if (n <= 256) nnz = ssc_doc<8, kCompact>(z, n, lane, starts, row, a.tbits);
        else nnz = ssc_doc<16, kCompact>(z, n, lane, starts, row, a.tbits);
        nnz_acc += nnz;
    }
    if (lane == 0 && nnz_acc) atomicAdd(a.nnz_total, nnz_acc);
}

// SSC without a sort (wide rows): a two-level topic bitmap per warp.  Setting one bit per
// token in a K-bit map (and one per 32-topic word in a K/32-bit summary) and reading the
// map back in order yields the document's distinct topics in ascending order; each token's
// rank among them is a popcount, so the counts are smem atomics at that rank.  Per document
// this costs O(len + nnz) warp steps instead of the bitonic sort's O(len log^2 len), and
// the order-free integer counts are identical to segmented_count's (counts.cpp:65-94).
struct SscBitmapSmem {
    uint32_t* bm0;    // K_pad/32 words (bit k = topic k present), all zero between documents
    uint32_t* bm1;    // ceil(K_pad/1024) words (bit w = bm0[w] != 0)
    uint16_t* wpre;   // per bm0 word: rank of its first topic
    uint16_t* wlist;  // non-empty bm0 words in ascending order
    uint32_t* ent;    // per rank: topic (low 16 bits) | count (high 16 bits, smem atomics)
};

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t x, uint32_t lane) {
#pragma unroll
    for (uint32_t o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    return x;
}

template <int R, bool kCompact>
__device__ __forceinline__ uint32_t ssc_doc_bitmap(const uint16_t* z, uint32_t n, uint32_t lane,
                                                   const SscBitmapSmem& w, uint32_t n1, uint32_t* out_row,
                                                   uint32_t tbits) {
    uint32_t key[R];
#pragma unroll
    for (uint32_t r = 0; r < R; ++r) {
        const uint32_t i = r * 32 + lane;
        key[r] = i < n ? static_cast<uint32_t>(z[i]) : 0xFFFFFFFFu;
        if (key[r] != 0xFFFFFFFFu) {
            atomicOr(w.bm0 + (key[r] >> 5), 1u << (key[r] & 31u));
            atomicOr(w.bm1 + (key[r] >> 10), 1u << ((key[r] >> 5) & 31u));
        }
    }
    __syncwarp();
    // Non-empty bm0 words in ascending order (and clear the summary).
    uint32_t m = 0;
    for (uint32_t b = 0; b < n1; b += 32) {
        const uint32_t wi = b + lane;
        const uint32_t bits0 = wi < n1 ? w.bm1[wi] : 0u;
        const uint32_t c = __popc(bits0);
        const uint32_t incl = warp_incl_scan(c, lane);
        uint32_t pos = m + incl - c;
        for (uint32_t bits = bits0; bits; bits &= bits - 1u) w.wlist[pos++] = static_cast<uint16_t>((wi << 5) | (__ffs(bits) - 1));
        if (bits0) w.bm1[wi] = 0u;
        m += __shfl_sync(0xffffffffu, incl, 31);
    }
    __syncwarp();
    // Distinct topics in order, and each word's first rank.
    uint32_t nnz = 0;
    for (uint32_t b = 0; b < m; b += 32) {
        const uint32_t e = b + lane;
        const uint32_t wi = e < m ? w.wlist[e] : 0u;
        const uint32_t bits0 = e < m ? w.bm0[wi] : 0u;
        const uint32_t c = __popc(bits0);
        const uint32_t incl = warp_incl_scan(c, lane);
        uint32_t pos = nnz + incl - c;
        if (e < m) w.wpre[wi] = static_cast<uint16_t>(pos);
        for (uint32_t bits = bits0; bits; bits &= bits - 1u) w.ent[pos++] = (wi << 5) | (__ffs(bits) - 1);
        nnz += __shfl_sync(0xffffffffu, incl, 31);
    }
    __syncwarp();
#pragma unroll
    for (uint32_t r = 0; r < R; ++r) {
        if (key[r] != 0xFFFFFFFFu) {
            const uint32_t wi = key[r] >> 5;
            const uint32_t rank = w.wpre[wi] + __popc(w.bm0[wi] & ((1u << (key[r] & 31u)) - 1u));
            atomicAdd(w.ent + rank, 1u << 16);
        }
    }
    __syncwarp();
#pragma unroll
    for (uint32_t r = 0; r < R; ++r)
        if (key[r] != 0xFFFFFFFFu) w.bm0[key[r] >> 5] = 0u;
    if (kCompact) {  // 16-bit slots (compact_chunk), header written by compact_finish
        uint16_t* row16 = reinterpret_cast<uint16_t*>(out_row);
        uint32_t pos = 2;
        for (uint32_t b = 0; b < nnz; b += 32) {
            const uint32_t e = b + lane;
            const uint32_t x = e < nnz ? w.ent[e] : 0u;
            compact_chunk(row16, pos, e < nnz, x & 0xFFFFu, x >> 16, lane);
        }
        compact_finish(row16, pos, nnz, lane);
    } else {
        for (uint32_t e = lane; e < nnz; e += 32) {
            const uint32_t x = w.ent[e];
            out_row[1 + e] = (x & 0xFFFFu) | ((x >> 16) << tbits);
        }
        const uint32_t padded = (nnz + 8u) & ~7u;
        for (uint32_t e = nnz + 1 + lane; e < padded; e += 32) out_row[e] = 0u;
        if (lane == 0) out_row[0] = nnz - 1u;
    }
    __syncwarp();
    return nnz;
}

constexpr uint32_t kSscBmWarps = 8;

__host__ __device__ inline size_t ssc_bitmap_warp_bytes(uint32_t K_pad) {
    const size_t n0 = (K_pad + 31u) / 32u, n1 = (n0 + 31u) / 32u;
    const size_t b = 4 * n0 + 4 * n1 + 4 * kSscWarpCap + 2 * n0 + 2 * kSscWarpCap;
    return (b + 15u) & ~static_cast<size_t>(15u);
}

template <bool kCompact>
__global__ void __launch_bounds__(kSscBmWarps * 32) ssc_bitmap_kernel(SscArgs a) {
    extern __shared__ __align__(16) unsigned char s_raw[];
    const uint32_t wid = threadIdx.x >> 5, lane = lane_id();
    const uint32_t n0 = (a.K_pad + 31u) / 32u, n1 = (n0 + 31u) / 32u;
    const size_t wb = ssc_bitmap_warp_bytes(a.K_pad);
    unsigned char* base = s_raw + wid * wb;
    SscBitmapSmem w;
    w.bm0 = reinterpret_cast<uint32_t*>(base);
    w.bm1 = w.bm0 + n0;
    w.ent = w.bm1 + n1;
    w.wpre = reinterpret_cast<uint16_t*>(w.ent + kSscWarpCap);
    w.wlist = w.wpre + n0;
    for (uint32_t i = lane; i < n0 + n1; i += 32) w.bm0[i] = 0u;
    __syncwarp();
    unsigned long long nnz_acc = 0;
    const uint32_t gw = blockIdx.x * kSscBmWarps + wid, nw = gridDim.x * kSscBmWarps;
    for (uint32_t d = gw; d < a.D; d += nw) {
        const uint32_t s0 = __ldg(a.doc_start + d);
        const uint32_t n = __ldg(a.doc_start + d + 1) - s0;
        if (n > kSscWarpCap || n == 0) continue;  // ssc_long_kernel / empty document
        uint32_t* row = a.A + __ldg(a.row4 + d) * 4u;
        const uint16_t* z = a.z + s0;
        uint32_t nnz;
        if (n <= 32) nnz = ssc_doc_bitmap<1, kCompact>(z, n, lane, w, n1, row, a.tbits);
        else if (n <= 64) nnz = ssc_doc_bitmap<2, kCompact>(z, n, lane, w, n1, row, a.tbits);
        else if (n <= 128) nnz = ssc_doc_bitmap<4, kCompact>(z, n, lane, w, n1, row, a.tbits);
        else if (n <= 256) nnz = ssc_doc_bitmap<8, kCompact>(z, n, lane, w, n1, row, a.tbits);
        else nnz = ssc_doc_bitmap<16, kCompact>(z, n, lane, w, n1, row, a.tbits);
        nnz_acc += nnz;
    }
    if (lane == 0 && nnz_acc) atomicAdd(a.nnz_total, nnz_acc);
}

// Long documents: one CTA per document (grid-stride over the long-doc list).
template <bool kSmemHist, bool kCompact>
__global__ void __launch_bounds__(256) ssc_long_kernel(SscArgs a) {
    extern __shared__ __align__(16) uint32_t s_dyn[];
    __shared__ uint32_t s_scan[256];
    uint32_t* hist = kSmemHist ? s_dyn : a.hist_scratch + static_cast<size_t>(blockIdx.x) * a.K_pad;
    const uint32_t tid = threadIdx.x;
    const uint32_t per = (a.K_pad + 255u) / 256u;
    for (uint32_t li = blockIdx.x; li < a.n_long; li += gridDim.x) {
        const uint32_t d = a.long_docs[li];
        const uint32_t s0 = a.doc_start[d];
        const uint32_t n = a.doc_start[d + 1] - s0;
        const uint32_t row = a.row4[d] * 4u;
        for (uint32_t k = tid; k < a.K_pad; k += 256) hist[k] = 0;
        __syncthreads();
        for (uint32_t i = tid; i < n; i += 256) atomicAdd(hist + a.z[s0 + i], 1u);
        __syncthreads();
        const uint32_t b0 = tid * per, b1 = min(a.K_pad, b0 + per);
        uint32_t mine = 0;
        for (uint32_t k = b0; k < b1; ++k) mine += hist[k] != 0;
        s_scan[tid] = mine;
        __syncthreads();
        for (uint32_t off = 1; off < 256; off <<= 1) {
            const uint32_t add = tid >= off ? s_scan[tid - off] : 0;
            __syncthreads();
            s_scan[tid] += add;
            __syncthreads();
        }
        const uint32_t nnz = s_scan[255];
        if (kCompact) {
            // One warp walks the histogram in topic order and packs the slots.
            if (tid < 32) {
                uint16_t* row16 = reinterpret_cast<uint16_t*>(a.A + row);
                uint32_t pos = 2;
                for (uint32_t k0 = 0; k0 < a.K_pad; k0 += 32) {
                    const uint32_t c = hist[k0 + tid];
                    compact_chunk(row16, pos, c != 0, k0 + tid, c, tid);
                }
                compact_finish(row16, pos, nnz, tid);
            }
        } else {
            uint32_t pos = s_scan[tid] - mine;
            for (uint32_t k = b0; k < b1; ++k) {
                const uint32_t c = hist[k];
                if (c) a.A[row + 1 + pos++] = k | (c << a.tbits);
            }
            const uint32_t padded = (nnz + 8u) & ~7u;
            for (uint32_t r = nnz + 1 + tid; r < padded; r += 256) a.A[row + r] = 0u;
            if (tid == 0) a.A[row] = nnz - 1u;
        }
        if (tid == 0) atomicAdd(a.nnz_total, static_cast<unsigned long long>(nnz));
        __syncthreads();
    }
}

template <bool kCompact>
cudaError_t launch_ssc_t(const SscArgs& a, cudaStream_t s) {
    if (a.D > 0) {
        const size_t bm_smem = kSscBmWarps * ssc_bitmap_warp_bytes(a.K_pad);
        if (!a.use_sort && bm_smem <= 200 * 1024) {
            static bool configured = false;
            if (!configured) {
                cudaFuncSetAttribute(ssc_bitmap_kernel<kCompact>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     200 * 1024);
                configured = true;
            }
            // Short-lived CTAs (16 documents per warp) rather than a persistent grid: SSC runs
            // beside the M-step on a low-priority stream, and retiring CTAs let the scheduler
            // hand SMs to the higher-priority colsum/phi CTAs.
            const uint32_t blocks = static_cast<uint32_t>((a.D + kSscBmWarps * 16u - 1) / (kSscBmWarps * 16u));
            ssc_bitmap_kernel<kCompact><<<blocks, kSscBmWarps * 32, bm_smem, s>>>(a);
        } else {
            const uint32_t blocks = grid_for(a.D, kSscWarps, 148u * 8u);
            ssc_warp_kernel<kCompact><<<blocks, kSscWarps * 32, 0, s>>>(a);
        }
    }
    if (a.n_long > 0) {
        const size_t smem = sizeof(uint32_t) * a.K_pad;
        const uint32_t blocks = a.n_long < 148u * 2u ? a.n_long : 148u * 2u;
        if (smem <= 200 * 1024) {
            static bool configured = false;
            if (!configured) {
                cudaFuncSetAttribute(ssc_long_kernel<true, kCompact>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
                configured = true;
            }
            ssc_long_kernel<true, kCompact><<<blocks, 256, smem, s>>>(a);
        } else {
            ssc_long_kernel<false, kCompact><<<blocks, 256, 0, s>>>(a);
        }
    }
    return cudaGetLastError();
}

cudaError_t launch_ssc(const SscArgs& a, cudaStream_t s) {
    return a.compact ? launch_ssc_t<true>(a, s) : launch_ssc_t<false>(a, s);
}

// ============================================================================
// K5/K6 -- preprocess (counts.cpp:37-63) + rebuild_trees (trainer.cpp:237-248,
// sampler.hpp:58-90, :142-149).  colsum: integer column sums (order-free).
// phi: thread per word row, 32-column tiles transposed through shared memory
// so global traffic is coalesced while each thread runs the row's sequential
// f32 prefix (the L4 level) exactly as WaryTree::build.
// ============================================================================

__global__ void __launch_bounds__(256) colsum_kernel(const uint32_t* __restrict__ B, uint32_t row_begin,
                                                     uint32_t row_end, uint32_t cols4,
                                                     uint32_t rows_per_chunk,
                                                     unsigned long long* __restrict__ colsum) {
    __shared__ unsigned long long s_acc[256][4];
    const uint32_t c4 = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t r0 = row_begin + blockIdx.y * rows_per_chunk;
    const uint32_t r1 = min(row_end, r0 + rows_per_chunk);
    unsigned long long acc[4] = {0, 0, 0, 0};
    if (c4 < cols4) {
        const uint4* B4 = reinterpret_cast<const uint4*>(B);
        for (uint32_t r = r0 + threadIdx.y; r < r1; r += blockDim.y) {
            const uint4 b = __ldg(B4 + static_cast<size_t>(r) * cols4 + c4);
            acc[0] += b.x; acc[1] += b.y; acc[2] += b.z; acc[3] += b.w;
        }
    }
    const uint32_t tid = threadIdx.y * blockDim.x + threadIdx.x;
    for (int j = 0; j < 4; ++j) s_acc[tid][j] = acc[j];
    __syncthreads();
    if (threadIdx.y == 0 && c4 < cols4) {
        for (uint32_t y = 1; y < blockDim.y; ++y)
            for (int j = 0; j < 4; ++j) acc[j] += s_acc[y * blockDim.x + threadIdx.x][j];
        for (int j = 0; j < 4; ++j)
            if (acc[j]) atomicAdd(colsum + 4 * c4 + j, acc[j]);
    }
}

cudaError_t launch_colsum(const uint32_t* B, uint32_t row_begin, uint32_t row_end, uint32_t K_pad,
                          unsigned long long* colsum, cudaStream_t s) {
    if (row_end <= row_begin) return cudaSuccess;
    const uint32_t cols4 = K_pad / 4;
    const uint32_t bx = cols4 < 256 ? cols4 : 256;
    const uint32_t by = 256 / bx;
    const uint32_t gx = (cols4 + bx - 1) / bx;
    const uint32_t rows = row_end - row_begin;
    // ~4 waves of CTAs.
    uint32_t gy = (148u * 8u + gx - 1) / gx;
    uint32_t per = (rows + gy - 1) / gy;
    if (per < by) per = by;
    gy = (rows + per - 1) / per;
    colsum_kernel<<<dim3(gx, gy), dim3(bx, by), 0, s>>>(B, row_begin, row_end, cols4, per, colsum);
    return cudaGetLastError();
}

// denom_k = f64(colsum_k) + V*beta (counts.cpp:49-50); zero-count cells share
// bhat = f32(beta / denom_k), so the phi kernel divides only non-zero cells.
__global__ void denom_kernel(const unsigned long long* colsum, uint32_t K, uint32_t K_pad, uint32_t V,
                             double beta, double* denom, float* zv) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= K_pad) return;
    if (k < K) {
        const double d = __dadd_rn(static_cast<double>(colsum[k]),
                                   __dmul_rn(static_cast<double>(V), beta));
        denom[k] = d;
        zv[k] = __double2float_rn(__ddiv_rn(__dadd_rn(0.0, beta), d));
    } else {
        denom[k] = 1.0;
        zv[k] = 0.0f;
    }
}

cudaError_t launch_denom(const unsigned long long* colsum, uint32_t K, uint32_t K_pad, uint32_t V,
                         double beta, double* denom, float* zv, cudaStream_t s) {
    denom_kernel<<<(K_pad + 255) / 256, 256, 0, s>>>(colsum, K, K_pad, V, beta, denom, zv);
    return cudaGetLastError();
}

// One thread per word row (the L4 prefix is a sequential f32 chain); 32-column tiles are
// moved through shared memory for coalescing, and tile c+1 is loaded into registers while
// tile c is computed.
constexpr int kPhiRows = 128;
constexpr int kPhiCols = 32;
constexpr int kPhiLoads = kPhiRows * kPhiCols / kPhiRows;  // per thread per tile

__global__ void __launch_bounds__(kPhiRows, 4) phi_kernel(const uint32_t* __restrict__ B,
                                                        const double* __restrict__ denom,
                                                        const float* __restrict__ zv,
                                                        float* __restrict__ bhat, float* __restrict__ l4,
                                                        float* __restrict__ l8, float* __restrict__ q,
                                                        uint32_t row_begin, uint32_t row_end, uint32_t K,
                                                        uint32_t K_pad, uint32_t l8_stride, double beta,
                                                        float falpha) {
    // t_bh aliases t_in: thread r overwrites cell [r][c] only after reading it.
    __shared__ uint32_t t_in[kPhiRows][kPhiCols + 1];
    __shared__ float t_l4[kPhiRows][kPhiCols + 1];
    __shared__ double s_den[kPhiCols];
    __shared__ float s_zv[kPhiCols];
    float(*t_bh)[kPhiCols + 1] = reinterpret_cast<float(*)[kPhiCols + 1]>(t_in);
    const uint32_t r = threadIdx.x;
    const uint32_t v0 = row_begin + blockIdx.x * kPhiRows;
    const uint32_t v = v0 + r;
    float run = 0.0f;
    uint32_t next[kPhiLoads];
    auto load_tile = [&](uint32_t c0) {
#pragma unroll
        for (int it = 0; it < kPhiLoads; ++it) {
            const uint32_t idx = it * kPhiRows + r;
            const uint32_t rr = idx / kPhiCols, cc = idx % kPhiCols;
            const uint32_t vv = v0 + rr;
            next[it] = vv < row_end ? __ldg(B + static_cast<size_t>(vv) * K_pad + c0 + cc) : 0u;
        }
    };
    load_tile(0);
    for (uint32_t c0 = 0; c0 < K_pad; c0 += kPhiCols) {
#pragma unroll
        for (int it = 0; it < kPhiLoads; ++it) {
            const uint32_t idx = it * kPhiRows + r;
            t_in[idx / kPhiCols][idx % kPhiCols] = next[it];
        }
        if (r < kPhiCols) {  // this tile's column constants, off the dependent chain
            s_den[r] = __ldg(denom + c0 + r);
            s_zv[r] = __ldg(zv + c0 + r);
        }
        __syncthreads();
        if (c0 + kPhiCols < K_pad) load_tile(c0 + kPhiCols);
        // Eight independent divisions are issued before the sequential f32 prefix consumes them.
#pragma unroll
        for (uint32_t c8 = 0; c8 < kPhiCols; c8 += 8) {
            float bh[8];
#pragma unroll
            for (uint32_t u = 0; u < 8; ++u) {
                const uint32_t c = c8 + u;
                const uint32_t cnt = t_in[r][c];
                bh[u] = c0 + c >= K ? 0.0f
                        : cnt ? __double2float_rn(__ddiv_rn(__dadd_rn(static_cast<double>(cnt), beta), s_den[c]))
                              : s_zv[c];
            }
#pragma unroll
            for (uint32_t u = 0; u < 8; ++u) {
                const uint32_t c = c8 + u;
                if (c0 + c < K) run = __fadd_rn(run, bh[u]);
                t_bh[r][c] = bh[u];
                t_l4[r][c] = run;
            }
        }
        if (v < row_end) {  // L8: the prefix at every 8th column of this tile
            const float4 l8v = make_float4(t_l4[r][7], t_l4[r][15], t_l4[r][23], t_l4[r][31]);
            *reinterpret_cast<float4*>(l8 + static_cast<size_t>(v) * l8_stride + c0 / kLeaf) = l8v;
        }
        __syncthreads();
#pragma unroll
        for (int it = 0; it < kPhiLoads; ++it) {
            const uint32_t idx = it * kPhiRows + r;
            const uint32_t rr = idx / kPhiCols, cc = idx % kPhiCols;
            const uint32_t vv = v0 + rr;
            if (vv < row_end) {
                const size_t o = static_cast<size_t>(vv) * K_pad + c0 + cc;
                bhat[o] = t_bh[rr][cc];
                l4[o] = t_l4[rr][cc];
            }
        }
        __syncthreads();  // the next tile store overwrites t_in (== t_bh)
    }
    if (v < row_end) {
        for (uint32_t j = K_pad / kLeaf; j < l8_stride; ++j) l8[static_cast<size_t>(v) * l8_stride + j] = run;
        q[v] = __fmul_rn(falpha, run);  // trainer.cpp:245
    }
}

cudaError_t launch_phi(const uint32_t* B, const double* denom, const float* zv, float* bhat,
                       float* l4, float* l8, float* q, uint32_t row_begin, uint32_t row_end,
                       uint32_t K, uint32_t K_pad, uint32_t l8_stride, double beta, float falpha,
                       cudaStream_t s) {
    if (row_end <= row_begin) return cudaSuccess;
    const uint32_t blocks = (row_end - row_begin + kPhiRows - 1) / kPhiRows;
    phi_kernel<<<blocks, kPhiRows, 0, s>>>(B, denom, zv, bhat, l4, l8, q, row_begin, row_end, K, K_pad,
                                           l8_stride, beta, falpha);
    return cudaGetLastError();
}

// ============================================================================
// K1/K2 setup -- build_chunks (corpus.cpp:125-198), build_schedule (:200-210),
// init_assignments (corpus.cpp:87-96), count_chunk_into (trainer.cpp:223-235).
// ============================================================================

__global__ void deinterleave_kernel(const uint32_t* __restrict__ aos, uint64_t T, uint32_t doc_begin,
                                    uint32_t* doc_local, uint32_t* word, uint32_t* topic) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < T;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        doc_local[i] = aos[3 * i] - doc_begin;
        word[i] = aos[3 * i + 1];
        if (topic) topic[i] = aos[3 * i + 2];
    }
}

cudaError_t launch_deinterleave(const uint32_t* aos, uint64_t T, uint32_t doc_begin,
                                uint32_t* doc_local, uint32_t* word, uint32_t* topic,
                                cudaStream_t s) {
    if (T == 0) return cudaSuccess;
    deinterleave_kernel<<<grid_for(T, 256), 256, 0, s>>>(aos, T, doc_begin, doc_local, word, topic);
    return cudaGetLastError();
}

__global__ void check_sorted_kernel(const uint32_t* doc_local, uint64_t T, uint32_t* flag) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x + 1; i < T;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        if (doc_local[i] < doc_local[i - 1]) *flag = 1u;
    }
}

cudaError_t launch_check_sorted(const uint32_t* doc_local, uint64_t T, uint32_t* unsorted_flag,
                                cudaStream_t s) {
    if (T < 2) return cudaSuccess;
    check_sorted_kernel<<<grid_for(T, 256), 256, 0, s>>>(doc_local, T, unsorted_flag);
    return cudaGetLastError();
}

__global__ void doc_hist_kernel(const uint32_t* doc_local, uint64_t T, uint32_t* counts) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < T;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        atomicAdd(counts + doc_local[i], 1u);
}

cudaError_t launch_doc_hist(const uint32_t* doc_local, uint64_t T, uint32_t* counts, cudaStream_t s) {
    if (T == 0) return cudaSuccess;
    doc_hist_kernel<<<grid_for(T, 256), 256, 0, s>>>(doc_local, T, counts);
    return cudaGetLastError();
}

__global__ void iota_kernel(uint32_t* out, uint64_t n) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        out[i] = static_cast<uint32_t>(i);
}

cudaError_t launch_iota(uint32_t* out, uint64_t n, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    iota_kernel<<<grid_for(n, 256), 256, 0, s>>>(out, n);
    return cudaGetLastError();
}

__global__ void invert_perm_kernel(const uint32_t* input_of_slot, uint64_t T, uint32_t* slot_of_input) {
    for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < T;
         j += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        slot_of_input[input_of_slot[j]] = static_cast<uint32_t>(j);
}

cudaError_t launch_invert_perm(const uint32_t* input_of_slot, uint64_t T, uint32_t* slot_of_input,
                               cudaStream_t s) {
    if (T == 0) return cudaSuccess;
    invert_perm_kernel<<<grid_for(T, 256), 256, 0, s>>>(input_of_slot, T, slot_of_input);
    return cudaGetLastError();
}

// Execution-order sort key, laid out in slot order so that equal keys keep slot
// (== corpus) order under the stable radix sort:
//   word | (lmax - len_doc) | doc_local
// i.e. the reference's (word, doc, token_id) order (corpus.cpp:157-167) refined by
// descending document length inside each word segment, so the lanes of a sampler
// warp walk C_dk rows of similar length.  lbits == 0 gives the canonical order.
__global__ void make_keys_kernel(const uint32_t* word, const uint32_t* doc_local,
                                 const uint32_t* input_of_slot, const uint32_t* doc_len, uint64_t T,
                                 KeyLayout kl, unsigned long long* keys, uint32_t* vals) {
    for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < T;
         j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t i = input_of_slot ? input_of_slot[j] : j;
        const uint32_t d = doc_local[i];
        const unsigned long long lk = kl.lbits ? static_cast<unsigned long long>(kl.lmax - doc_len[d]) : 0ull;
        keys[j] = (static_cast<unsigned long long>(word[i]) << (kl.dbits + kl.lbits)) | (lk << kl.dbits) | d;
        vals[j] = static_cast<uint32_t>(j);
    }
}

cudaError_t launch_make_keys(const uint32_t* word, const uint32_t* doc_local, const uint32_t* input_of_slot,
                             const uint32_t* doc_len, uint64_t T, KeyLayout kl, unsigned long long* keys,
                             uint32_t* vals, cudaStream_t s) {
    if (T == 0) return cudaSuccess;
    make_keys_kernel<<<grid_for(T, 256), 256, 0, s>>>(word, doc_local, input_of_slot, doc_len, T, kl, keys, vals);
    return cudaGetLastError();
}

// tok = {C_dk row offset (quads), slot}; flags mark word-segment starts.
__global__ void make_tok_kernel(const unsigned long long* keys, const uint32_t* slots, const uint32_t* row4,
                                uint64_t T, KeyLayout kl, uint2* tok, uint32_t* seg_flag) {
    const unsigned long long dmask = (1ull << kl.dbits) - 1ull;
    const uint32_t ws = kl.dbits + kl.lbits;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < T;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const unsigned long long k = keys[i];
        tok[i] = make_uint2(row4[k & dmask], slots[i]);
        seg_flag[i] = (i == 0 || (keys[i - 1] >> ws) != (k >> ws)) ? 1u : 0u;
    }
}

cudaError_t launch_make_tok(const unsigned long long* keys, const uint32_t* slots, const uint32_t* row4,
                            uint64_t T, KeyLayout kl, uint2* tok, uint32_t* seg_flag, cudaStream_t s) {
    if (T == 0) return cudaSuccess;
    make_tok_kernel<<<grid_for(T, 256), 256, 0, s>>>(keys, slots, row4, T, kl, tok, seg_flag);
    return cudaGetLastError();
}

__global__ void emit_segments_kernel(const unsigned long long* keys, const uint32_t* seg_flag,
                                     const uint32_t* seg_index, uint64_t T, uint32_t wshift,
                                     uint32_t* seg_word, uint32_t* seg_off) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < T;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        if (seg_flag[i]) {
            const uint32_t s = seg_index[i];
            seg_word[s] = static_cast<uint32_t>(keys[i] >> wshift);
            seg_off[s] = static_cast<uint32_t>(i);
        }
    }
}

cudaError_t launch_emit_segments(const unsigned long long* keys, const uint32_t* seg_flag,
                                 const uint32_t* seg_index, uint64_t T, uint32_t wshift,
                                 uint32_t* seg_word, uint32_t* seg_off, cudaStream_t s) {
    if (T == 0) return cudaSuccess;
    emit_segments_kernel<<<grid_for(T, 256), 256, 0, s>>>(keys, seg_flag, seg_index, T, wshift, seg_word,
                                                         seg_off);
    return cudaGetLastError();
}

// build_schedule sort key: (length desc, word asc) -- corpus.cpp:201-205.
__global__ void segment_lengths_kernel(const uint32_t* seg_off, uint32_t nseg, uint64_t T,
                                       uint32_t* seg_len, unsigned long long* sched_keys,
                                       uint32_t* sched_vals, const uint32_t* seg_word,
                                       uint32_t* unit_count) {
    const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nseg) return;
    const uint64_t end = s + 1 < nseg ? seg_off[s + 1] : T;
    const uint32_t len = static_cast<uint32_t>(end - seg_off[s]);
    seg_len[s] = len;
    sched_keys[s] = (static_cast<unsigned long long>(0xFFFFFFFFu - len) << 32) | seg_word[s];
    sched_vals[s] = s;
    if (unit_count) unit_count[s] = (len + kUnitMaxTokens - 1) / kUnitMaxTokens;
}

cudaError_t launch_segment_lengths(const uint32_t* seg_off, uint32_t nseg, uint64_t T,
                                   uint32_t* seg_len, unsigned long long* sched_keys,
                                   uint32_t* sched_vals, const uint32_t* seg_word,
                                   uint32_t* unit_count, cudaStream_t s) {
    if (nseg == 0) return cudaSuccess;
    segment_lengths_kernel<<<(nseg + 255) / 256, 256, 0, s>>>(seg_off, nseg, T, seg_len, sched_keys,
                                                             sched_vals, seg_word, unit_count);
    return cudaGetLastError();
}

// unit_count here is indexed by schedule position (permuted by the caller).
__global__ void emit_units_kernel(const uint32_t* schedule, const uint32_t* seg_word,
                                  const uint32_t* seg_off, const uint32_t* seg_len,
                                  const uint32_t* unit_start, uint32_t nseg, Unit* units) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= nseg) return;
    const uint32_t s = schedule[p];
    const uint32_t len = seg_len[s];
    uint32_t u = unit_start[p];
    for (uint32_t o = 0; o < len; o += kUnitMaxTokens, ++u) {
        const uint32_t l = len - o < kUnitMaxTokens ? len - o : kUnitMaxTokens;
        units[u] = Unit{seg_word[s], seg_off[s] + o, l, 0u};
    }
}

cudaError_t launch_emit_units(const uint32_t* schedule, const uint32_t* seg_word,
                              const uint32_t* seg_off, const uint32_t* seg_len,
                              const uint32_t* unit_start, uint32_t nseg, Unit* units,
                              cudaStream_t s) {
    if (nseg == 0) return cudaSuccess;
    emit_units_kernel<<<(nseg + 255) / 256, 256, 0, s>>>(schedule, seg_word, seg_off, seg_len,
                                                        unit_start, nseg, units);
    return cudaGetLastError();
}

// C_dk row capacity in uint4 units: header + nnz_d entries with nnz_d <= len_d
// (test_counts.cpp:149-150), rounded up to 32 entries (one 128-byte line).
__global__ void row_quads_kernel(const uint32_t* doc_start, uint32_t D, uint32_t* quads) {
    const uint32_t d = blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= D) return;
    // Rounded up to a whole 128-byte line: every row starts line-aligned, so each 4-sector
    // group the sampler loads is exactly one L1 line (scripts/mb_pattern.cu: a third fewer
    // L1TEX wavefronts per loaded byte than 32-byte-aligned rows).
    quads[d] = ((((doc_start[d + 1] - doc_start[d] + 8u) >> 3) << 1) + 7u) & ~7u;
}

cudaError_t launch_row_quads(const uint32_t* doc_start, uint32_t D, uint32_t* quads, cudaStream_t s) {
    if (D == 0) return cudaSuccess;
    row_quads_kernel<<<(D + 255) / 256, 256, 0, s>>>(doc_start, D, quads);
    return cudaGetLastError();
}

__global__ void long_flags_kernel(const uint32_t* doc_start, uint32_t D, uint32_t* flags) {
    const uint32_t d = blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= D) return;
    flags[d] = (doc_start[d + 1] - doc_start[d]) > kSscWarpCap ? 1u : 0u;
}

cudaError_t launch_long_flags(const uint32_t* doc_start, uint32_t D, uint32_t* flags, cudaStream_t s) {
    if (D == 0) return cudaSuccess;
    long_flags_kernel<<<(D + 255) / 256, 256, 0, s>>>(doc_start, D, flags);
    return cudaGetLastError();
}

__global__ void init_topics_kernel(uint64_t T, const uint64_t* ids, uint64_t id_base, uint64_t seed,
                                   uint32_t K, uint16_t* z) {
    for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < T;
         j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t id = ids ? ids[j] : id_base + j;
        z[j] = static_cast<uint16_t>(uniform_topic(seed, kInitAssignStream, id, K));
    }
}

cudaError_t launch_init_topics(uint64_t T, const uint64_t* ids, uint64_t id_base, uint64_t seed,
                               uint32_t K, uint16_t* z, cudaStream_t s) {
    if (T == 0) return cudaSuccess;
    init_topics_kernel<<<grid_for(T, 256), 256, 0, s>>>(T, ids, id_base, seed, K, z);
    return cudaGetLastError();
}

__global__ void given_topics_kernel(const uint32_t* topic_in, const uint32_t* input_of_slot, uint64_t T,
                                    uint16_t* z) {
    for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < T;
         j += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        z[j] = static_cast<uint16_t>(topic_in[input_of_slot ? input_of_slot[j] : j]);
}

cudaError_t launch_given_topics(const uint32_t* topic_in, const uint32_t* input_of_slot, uint64_t T,
                                uint16_t* z, cudaStream_t s) {
    if (T == 0) return cudaSuccess;
    given_topics_kernel<<<grid_for(T, 256), 256, 0, s>>>(topic_in, input_of_slot, T, z);
    return cudaGetLastError();
}

__global__ void ids_by_slot_kernel(const uint64_t* ids_in, const uint32_t* input_of_slot, uint64_t T,
                                   uint64_t id_base, uint64_t* ids_out) {
    for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < T;
         j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t i = input_of_slot ? input_of_slot[j] : j;
        ids_out[j] = ids_in ? ids_in[i] : id_base + i;
    }
}

cudaError_t launch_ids_by_slot(const uint64_t* ids_in, const uint32_t* input_of_slot, uint64_t T,
                               uint64_t id_base, uint64_t* ids_out, cudaStream_t s) {
    if (T == 0) return cudaSuccess;
    ids_by_slot_kernel<<<grid_for(T, 256), 256, 0, s>>>(ids_in, input_of_slot, T, id_base, ids_out);
    return cudaGetLastError();
}

// count_chunk_into (trainer.cpp:223-235) in word order.  With freshly drawn topics
// (init_assignments) the topic is recomputed from the token id -- the same Philox draw as
// init_topics_kernel -- instead of gathered from z by slot (a random 2-byte read per token).
__global__ void __launch_bounds__(256) recount_kernel(const uint2* tok, const Unit* units,
                                                      const uint16_t* z, uint32_t* B, uint32_t K_pad,
                                                      RecountDraw draw) {
    const Unit u = units[blockIdx.x];
    uint32_t* brow = B + static_cast<size_t>(u.word) * K_pad;
    for (uint32_t i = threadIdx.x; i < u.length; i += blockDim.x) {
        const uint32_t slot = tok[u.offset + i].y;
        uint32_t topic;
        if (draw.K) {
            const uint64_t id = draw.ids ? draw.ids[slot] : draw.id_base + slot;
            topic = uniform_topic(draw.seed, kInitAssignStream, id, draw.K);
        } else {
            topic = z[slot];
        }
        atomicAdd(brow + topic, 1u);
    }
}

cudaError_t launch_recount(const uint2* tok, const Unit* units, uint32_t n_units, const uint16_t* z,
                           uint32_t* B, uint32_t K_pad, RecountDraw draw, cudaStream_t s) {
    if (n_units == 0) return cudaSuccess;
    recount_kernel<<<n_units, 256, 0, s>>>(tok, units, z, B, K_pad, draw);
    return cudaGetLastError();
}

__global__ void validate_kernel(const uint32_t* __restrict__ aos, uint64_t T, uint32_t doc_begin,
                                uint32_t doc_end, uint32_t V, uint32_t K, ValidateOut* out) {
    // Per-thread minima, then one atomic per warp and quantity (a corpus of sentinel topics
    // would otherwise serialise T atomics on one address).
    unsigned long long bad_doc = ~0ull, bad_word = ~0ull, first_invalid = ~0ull, first_big = ~0ull;
    uint32_t unsorted = 0;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < T;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t d = aos[3 * i], w = aos[3 * i + 1], t = aos[3 * i + 2];
        if ((d < doc_begin || d >= doc_end) && bad_doc == ~0ull) bad_doc = i;
        if (w >= V && bad_word == ~0ull) bad_word = i;
        if (t == kInvalidTopic) first_invalid = min(first_invalid, static_cast<unsigned long long>(i));
        else if (t >= K) first_big = min(first_big, static_cast<unsigned long long>(i));
        if (i > 0 && aos[3 * (i - 1)] > d) unsorted = 1u;
    }
    for (int o = 16; o > 0; o >>= 1) {
        bad_doc = min(bad_doc, __shfl_xor_sync(0xffffffffu, bad_doc, o));
        bad_word = min(bad_word, __shfl_xor_sync(0xffffffffu, bad_word, o));
        first_invalid = min(first_invalid, __shfl_xor_sync(0xffffffffu, first_invalid, o));
        first_big = min(first_big, __shfl_xor_sync(0xffffffffu, first_big, o));
        unsorted |= __shfl_xor_sync(0xffffffffu, unsorted, o);
    }
    if (lane_id() == 0) {
        if (bad_doc != ~0ull) atomicMin(&out->bad_doc, bad_doc);
        if (bad_word != ~0ull) atomicMin(&out->bad_word, bad_word);
        if (first_invalid != ~0ull) atomicMin(&out->first_invalid, first_invalid);
        if (first_big != ~0ull) atomicMin(&out->first_big, first_big);
        if (unsorted) out->unsorted = 1u;
    }
}

cudaError_t launch_validate(const uint32_t* aos, uint64_t T, uint32_t doc_begin, uint32_t doc_end,
                            uint32_t V, uint32_t K, ValidateOut* out, cudaStream_t s) {
    if (T == 0) return cudaSuccess;
    validate_kernel<<<grid_for(T, 256), 256, 0, s>>>(aos, T, doc_begin, doc_end, V, K, out);
    return cudaGetLastError();
}

__global__ void sched_counts_kernel(const uint32_t* schedule, const uint32_t* seg_len, uint32_t nseg,
                                    uint32_t* counts) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= nseg) return;
    counts[p] = (seg_len[schedule[p]] + kUnitMaxTokens - 1) / kUnitMaxTokens;
}

cudaError_t launch_sched_counts(const uint32_t* schedule, const uint32_t* seg_len, uint32_t nseg,
                                uint32_t* counts, cudaStream_t s) {
    if (nseg == 0) return cudaSuccess;
    sched_counts_kernel<<<(nseg + 255) / 256, 256, 0, s>>>(schedule, seg_len, nseg, counts);
    return cudaGetLastError();
}

}  // namespace slda

namespace slda {

// gather_assignments (trainer.cpp:203-213): slot-ordered u16 topics -> corpus-order u32.
// input_of_slot == null: doc-sorted corpus, slot == corpus position (a widening copy).
__global__ void assignments_kernel(const uint16_t* z, const uint32_t* input_of_slot, uint64_t T, uint32_t* out) {
    for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < T;
         j += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        out[input_of_slot ? input_of_slot[j] : j] = z[j];
}

cudaError_t launch_assignments(const uint16_t* z, const uint32_t* input_of_slot, uint64_t T, uint32_t* out,
                               cudaStream_t s) {
    if (T == 0) return cudaSuccess;
    assignments_kernel<<<grid_for(T, 256), 256, 0, s>>>(z, input_of_slot, T, out);
    return cudaGetLastError();
}

}  // namespace slda
