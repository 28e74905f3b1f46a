// sampler.cu -- K3: the ESCA sampling step on sm_100a.
//
// Reference paths are relative to /root/reference/proj.  Each kernel names the reference
// function it replaces.  See DESIGN.md §4 (kernels, rooflines) and §6 (measurements).
#include <cstdlib>
#include <string>

#include "row_format.cuh"

namespace slda {

// ============================================================================
// K3 sampler -- process_segment (trainer.cpp:265-291) + sample_token<float>
// (sampler.hpp:166-204) + the C_wk accumulation of accumulate_word_topic
// (counts.cpp:127-132).  One CTA per heavy-first work unit of one word; the
// word's phi row and its L8 level are staged in shared memory; each warp stages
// its 32 tokens' C_dk rows cooperatively (coalesced), and each lane samples one
// token so that the sparse mass S and the in-place prefix run as the reference's
// sequential f32 chains.
// ============================================================================

// Used where a 512-thread quad-lane CTA pair does not fit an SM but the phi row still fits shared
// memory (17.5K < K_pad <~ 45K).
// The new topic of execution position `exec` (slot `slot`): staged in execution order when the
// engine transposes afterwards (zmove.cu: full-sector stores), else straight to z by slot.
__device__ __forceinline__ void store_topic(const SamplerArgs& a, uint32_t exec, uint32_t slot, uint32_t topic) {
    if (a.zx)
        a.zx[a.zx_pos ? __ldg(a.zx_pos + exec) : exec] = static_cast<uint16_t>(topic);
    else
        a.z[slot] = static_cast<uint16_t>(topic);
}

template <int NT, int G, int MINB>
__global__ void __launch_bounds__(NT, MINB) sampler_kernel(SamplerArgs a) {
    using St = Stage<G>;
    extern __shared__ __align__(16) float sm[];
    const uint32_t v = a.units[blockIdx.x].word;
    const float* s_bhat = sm;
    float* s_l8 = sm + a.K_pad;  // l8_stride (L4[8j+7], padded with the total)
    float* s_ck = s_l8 + a.l8_stride;       // [kCkSectors][NT]
    unsigned char* s_stage = reinterpret_cast<unsigned char*>(s_ck + kCkSectors * NT);

    const Unit unit = a.units[blockIdx.x];
    const float total = __ldg(a.l8 + static_cast<size_t>(v) * a.l8_stride + a.n_l8 - 1);  // L8's last = the row total
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

        // Row = [header (nnz-1, count 0) | entries | zero-count padding to 8]: header and
        // padding add +0 to every running sum.
        const uint32_t w0 = reinterpret_cast<const uint4*>(mine)->x;
        const uint32_t nnz = active ? (w0 & tmask) + 1u : 0u;
        const uint32_t nsect = active ? (nnz + 8u) >> 3 : 0u;
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
                    s = acc_sector(s, mine + 32 * u, tbits, tmask, s_bhat);
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
                    // every prefix is >= 0: the first real entry (word 1)
                    const uint32_t e1 = __ldg(reinterpret_cast<const uint32_t*>(A4 + t.x) + 1);
                    topic = e1 & tmask;
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
                const uint32_t k = tree_search<false>(x, s_l8, a.n_l8, s_bhat);
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
                scan_sector(run, need, topic, xs, mine, tbits, tmask, s_bhat);
                ++sec;
            }
        }
        if (active) {
            store_topic(a, unit.offset + i, t.y, topic);
            atomicAdd(brow + topic, 1u);
        }
    }
    if (a.row_entries) {
        // One atomic per warp.
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
template <int NT, int MINB, int L, bool kC16 = false>
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
    const float total = __ldg(a.l8 + static_cast<size_t>(v) * a.l8_stride + a.n_l8 - 1);  // L8's last = the row total
    __shared__ __align__(8) unsigned long long s_bar;  // phi/L8 staging (TMA bulk copies)
    tma_stage_rows(sm, a.bhat + static_cast<size_t>(v) * a.K_pad, a.K_pad * 4u, s_l8,
                   a.l8 + static_cast<size_t>(v) * a.l8_stride, a.l8_stride * 4u, &s_bar);
    const float qv = __ldg(a.q + v);
    uint32_t* brow = a.B + static_cast<size_t>(v) * a.K_pad;
    // kC16: counts in the high half-word (tbits == 16): the count decode folds into one I2F.U16.H1.
    const uint32_t tbits = kC16 ? 16u : a.tbits, tmask = kC16 ? 0xFFFFu : (1u << a.tbits) - 1u;
    const uint4* A4 = reinterpret_cast<const uint4*>(a.A);
    const uint32_t lane = lane_id(), t = lane / L, sub = lane % L, lead = lane & ~(L - 1u);
    const uint32_t warp = threadIdx.x >> 5;
    float* ckw = s_ck + warp * 32u * kCkStride;
    unsigned long long entries = 0;
    if (threadIdx.x == 0) s_next = NW * 32u;
    __syncthreads();
    tma_wait_rows(&s_bar);

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
            // [nnz-1 | entries | pad to 8]
            const uint32_t nnz = act ? (hw & tmask) + 1u : 0u;
            const uint32_t nsect = act ? (nnz + 8u) >> 3 : 0u;
            if (sub == 0) entries += nnz;
            const uint32_t max_groups = __reduce_max_sync(0xffffffffu, (nsect + L - 1u) / L);
            float* ck = ckw + ti * kCkStride;
            float run = 0.0f;
            // Products of this lane's sector, then the chain over the line's 4 sectors in order.
            auto consume = [&](const Sector& q, uint32_t g) {
                const uint32_t sec = L * g + sub;
                constexpr int NP = 8;  // products per sector
                // Sectors past the row are loaded as zeros (in-range bhat[0] gathers, broadcast),
                // so the products need no branch; only valid sectors' products are accumulated.
                float p[NP];
                {
                    const uint32_t es[8] = {q.lo.x, q.lo.y, q.lo.z, q.lo.w, q.hi.x, q.hi.y, q.hi.z, q.hi.w};
#pragma unroll
                    for (int w = 0; w < 8; ++w) p[w] = entry_mass<false>(es[w], tbits, tmask, s_bhat);
                }
                // Branch-free rounds: every lane runs the 8 FADDs (an instruction costs the same
                // with 8 or 32 lanes active) and only lane j of each group keeps the result.
                const bool valid = sec < nsect;
#pragma unroll
                for (uint32_t j = 0; j < L; ++j) {
                    float r2 = run;
#pragma unroll
                    for (int w = 0; w < NP; ++w) r2 = __fadd_rn(r2, p[w]);
                    const bool mine = sub == j && valid;
                    run = mine ? r2 : run;
                    if (mine && sec < kCk) ck[sec] = run;
                    run = __shfl_sync(0xffffffffu, run, lead | j);
                }
            };
            for (uint32_t g = 0; g < max_groups; g += 2) {  // two groups per trip: no register copies
                Sector n = c;
                n = L * (g + 1) + sub < nsect ? ldg_sector(row + 2 * (L * (g + 1) + sub)) : zero_sector();
                consume(c, g);
                if (g + 1 >= max_groups) break;
                c = L * (g + 2) + sub < nsect ? ldg_sector(row + 2 * (L * (g + 2) + sub)) : zero_sector();
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
                    topic = e1 & tmask;
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
#pragma unroll
                        for (int w = 0; w < 8; ++w) {
                            r = __fadd_rn(r, entry_mass<false>(es[w], tbits, tmask, s_bhat));
                            if (!found && r >= xs) { topic = es[w] & tmask; found = true; }
                        }
                        if (found) break;
                    }
                }
            } else {
                float x = __fmul_rn(up, total);  // WaryTree::sample(p * total)
                if (!(x <= total)) x = total;
                const uint32_t k = tree_search<false>(x, s_l8, a.n_l8, s_bhat);
                topic = k < a.K ? k : a.K - 1;
            }
            store_topic(a, unit.offset + base + lane, tk.y, topic);
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

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(gmem), "r"(valid ? 16 : 0)
                 : "memory");
}

// The same algorithm with the next round's first line prefetched -- by cp.async into a 1 KB
// per-warp shared-memory buffer when a round starts, a whole round ahead (kAsyncNext, C3 sampler
// 70.3 -> 68.3 ms), or into registers in each round's last group slot -- and the next batch
// claimed a batch ahead; the per-unit scalars live in shared memory to
// make room in the 64-register budget (C3 K=10K: 95.5 -> 92.8 ms; C2: 19.8 -> 20.5 ms).
// kGlobalPhi: the phi row does not fit shared memory (K >~ 45K): only L8 is staged and the
// products gather phi through L1/L2.
template <int NT, int MINB, int L, bool kC16 = false, bool kPrefetchNext = true, bool kGlobalPhi = false,
          bool kAsyncNext = false>
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
    const float* s_bhat = kGlobalPhi ? a.bhat + static_cast<size_t>(v) * a.K_pad : sm;
    float* s_l8 = kGlobalPhi ? sm : sm + a.K_pad;
    float* s_ck = s_l8 + a.l8_stride;  // [NW][32 tokens][kCkStride]
    // kAsyncNext: the next round's first line of each token lands here by cp.async (32 B per lane),
    // issued when a round starts -- a whole round ahead, in no registers.
    unsigned char* s_line = reinterpret_cast<unsigned char*>(s_ck + NW * 32u * kCkStride) + (threadIdx.x >> 5) * 1024u +
                            (threadIdx.x & 31u) * 32u;
    __shared__ __align__(8) unsigned long long s_bar;  // phi/L8 staging (TMA bulk copies)
    tma_stage_rows(sm, a.bhat + static_cast<size_t>(v) * a.K_pad, kGlobalPhi ? 0u : a.K_pad * 4u, s_l8,
                   a.l8 + static_cast<size_t>(v) * a.l8_stride, a.l8_stride * 4u, &s_bar);
    // kC16: counts in the high half-word (tbits == 16): the count decode folds into one I2F.U16.H1.
    const uint32_t tbits = kC16 ? 16u : a.tbits, tmask = kC16 ? 0xFFFFu : (1u << a.tbits) - 1u;
    const uint4* A4 = reinterpret_cast<const uint4*>(a.A);
    const uint32_t lane = lane_id(), t = lane / L, sub = lane % L, lead = lane & ~(L - 1u);
    const uint32_t warp = threadIdx.x >> 5;
    float* ckw = s_ck + warp * 32u * kCkStride;
    uint32_t entries = 0;
    if (threadIdx.x == 0) {
        s_next = NW * 32u;
        s_total = __ldg(a.l8 + static_cast<size_t>(v) * a.l8_stride + a.n_l8 - 1);  // L8's last = the row total
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
    tma_wait_rows(&s_bar);  // phi + L8 landed (the first lines are already in flight)
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
            if (kAsyncNext) {  // the next round's first line (next batch's after the last round)
                const bool last = r + 1 == L || base + TPR * (r + 1) >= unit.length;
                const uint32_t nrq = __shfl_sync(0xffffffffu, last ? tk_nx.x : tk.x, last ? t : ti + TPR);
                const bool ok = last ? nb + t < unit.length : base + ti + TPR < unit.length;
                const uint4* src = ok ? A4 + nrq + 2 * sub : A4;
                cp_async16(s_line, src, ok);
                cp_async16(s_line + 16, src + 1, ok);
                asm volatile("cp.async.commit_group;\n" ::: "memory");
            }
            const uint32_t hw = __shfl_sync(0xffffffffu, c.lo.x, lead);  // header: word 0 of sector 0
            // [nnz-1 | entries | pad to 8]
            const uint32_t nnz = act ? (hw & tmask) + 1u : 0u;
            const uint32_t nsect = act ? (nnz + 8u) >> 3 : 0u;
            if (sub == 0) entries += nnz;
            const uint32_t max_groups = __reduce_max_sync(0xffffffffu, (nsect + L - 1u) / L);
            float* ck = ckw + ti * kCkStride;
            float run = 0.0f;
            // Products of this lane's sector, then the chain over the line's 4 sectors in order.
            auto consume = [&](const Sector& q, uint32_t g) {
                const uint32_t sec = L * g + sub;
                constexpr int NP = 8;  // products per sector
                // Sectors past the row are loaded as zeros (in-range bhat[0] gathers, broadcast),
                // so the products need no branch; only valid sectors' products are accumulated.
                float p[NP];
                {
                    const uint32_t es[8] = {q.lo.x, q.lo.y, q.lo.z, q.lo.w, q.hi.x, q.hi.y, q.hi.z, q.hi.w};
#pragma unroll
                    for (int w = 0; w < 8; ++w) p[w] = entry_mass<kGlobalPhi>(es[w], tbits, tmask, s_bhat);
                }
                // Branch-free rounds: every lane runs the 8 FADDs (an instruction costs the same
                // with 8 or 32 lanes active) and only lane j of each group keeps the result.
                const bool valid = sec < nsect;
#pragma unroll
                for (uint32_t j = 0; j < L; ++j) {
                    float r2 = run;
#pragma unroll
                    for (int w = 0; w < NP; ++w) r2 = __fadd_rn(r2, p[w]);
                    const bool mine = sub == j && valid;
                    run = mine ? r2 : run;
                    if (mine && sec < kCk) ck[sec] = run;
                    run = __shfl_sync(0xffffffffu, run, lead | j);
                }
            };
            // Group g+1 (or the next round's first line) loads while group g is consumed; two
            // groups per trip so no registers are copied.
            auto fetch = [&](uint32_t g, Sector& dst) {
                if (g < max_groups) {  // warp-uniform
                    dst = L * g + sub < nsect ? ldg_sector(row + 2 * (L * g + sub)) : zero_sector();
                } else if (kPrefetchNext && !kAsyncNext) {
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
            if (kAsyncNext) {
                asm volatile("cp.async.wait_group 0;\n" ::: "memory");
                c.lo = *reinterpret_cast<const uint4*>(s_line);
                c.hi = *reinterpret_cast<const uint4*>(s_line + 16);
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
            float ub, up;
            const uint64_t id = a.ids ? __ldg(a.ids + tk.y) : a.id_base + tk.y;
            draw2_f32(a.seed, a.stream_kind, id, ub, up);
            const uint4* row = A4 + tk.x;
            uint32_t topic = 0;
            if (ub < __fdiv_rn(S, __fadd_rn(S, qv))) {
                const float xs = __fmul_rn(up, S);
                if (xs == 0.0f) {
                    const uint32_t e1 = __ldg(reinterpret_cast<const uint32_t*>(row) + 1);  // first real entry
                    topic = e1 & tmask;
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
#pragma unroll
                        for (int w = 0; w < 8; ++w) {
                            r = __fadd_rn(r, entry_mass<kGlobalPhi>(es[w], tbits, tmask, s_bhat));
                            if (!found && r >= xs) { topic = es[w] & tmask; found = true; }
                        }
                        if (found) break;
                    }
                }
            } else {
                float x = __fmul_rn(up, total);  // WaryTree::sample(p * total)
                if (!(x <= total)) x = total;
                const uint32_t k = tree_search<kGlobalPhi>(x, s_l8, a.n_l8, s_bhat);
                topic = k < a.K ? k : a.K - 1;
            }
            store_topic(a, unit.offset + base + lane, tk.y, topic);
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

// Dynamic shared memory opt-in, set on every launch: the attribute is per device context, so
// a process-wide "configured" flag would leave a second engine on another GPU without it.
template <class Kern>
cudaError_t smem_optin(Kern kern, size_t bytes) {
    return bytes > 48 * 1024
               ? cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes))
               : cudaSuccess;
}

size_t sampler_smem(const SamplerArgs& a, int nt, int g) {
    const size_t stage_row = 32u * static_cast<size_t>(g) + 16u;
    return sizeof(float) * (static_cast<size_t>(a.K_pad) + a.l8_stride) +
           (sizeof(float) * kCkSectors + stage_row) * static_cast<size_t>(nt);
}

// Round-based 4-sector-group kernel (17.5K < K_pad <~ 45K).
cudaError_t launch_round(const SamplerArgs& a, uint32_t n_units, cudaStream_t s) {
    const size_t smem = sampler_smem(a, 256, 4);
    if (const cudaError_t e = smem_optin(sampler_kernel<256, 4, 2>, smem); e != cudaSuccess) return e;
    sampler_kernel<256, 4, 2><<<n_units, 256, smem, s>>>(a);
    return cudaGetLastError();
}

size_t sampler_quad_smem(const SamplerArgs& a, int nt) {
    return sizeof(float) * (static_cast<size_t>(a.K_pad) + a.l8_stride + static_cast<size_t>(nt / 32) * 32u * 17u);
}

template <int NT, int MINB, bool PF, bool C16>
cudaError_t launch_quad_t1(const SamplerArgs& a, uint32_t n_units, cudaStream_t s) {
    // The cp.async line buffer (1 KB per warp) only where two CTAs per SM still fit (K_pad <~ 13.5K
    // at 512 threads); above, the register prefetch.
    const bool an = PF && a.async_next &&
                    2 * (sampler_quad_smem(a, NT) + static_cast<size_t>(NT / 32) * 1024u) <= 227u * 1024u;
    auto kern = an ? sampler_quad_pf_kernel<NT, MINB, 4, C16, true, false, true>
              : PF ? sampler_quad_pf_kernel<NT, MINB, 4, C16> : sampler_quad_kernel<NT, MINB, 4, C16>;
    const size_t smem = sampler_quad_smem(a, NT) + (an ? static_cast<size_t>(NT / 32) * 1024u : 0u);
    if (const cudaError_t e = smem_optin(kern, smem); e != cudaSuccess) return e;
    kern<<<n_units, NT, smem, s>>>(a);
    return cudaGetLastError();
}
// PF: the next round's first line is prefetched in each round's last group slot (C3 K=10K:
// 95.5 -> 92.8 ms; short-phi C2: 19.8 -> 20.5 ms, so only the 512-thread shape uses it).
template <int NT, int MINB, bool PF = (NT >= 512)>
cudaError_t launch_quad_t(const SamplerArgs& a, uint32_t n_units, cudaStream_t s) {
    return a.tbits == 16 ? launch_quad_t1<NT, MINB, PF, true>(a, n_units, s)
                         : launch_quad_t1<NT, MINB, PF, false>(a, n_units, s);
}

// phi rows too large for shared memory (K_pad * 4 > ~180 KB): quad-lane kernel with only L8 staged.
cudaError_t launch_quad_global(const SamplerArgs& a, uint32_t n_units, cudaStream_t s) {
    // (no cp.async line buffer here: the shared memory it takes comes out of the L1 that serves the
    // phi gathers -- C5 K=50K sampler 59.6 -> 66.0 ms with it)
    auto kern = a.tbits == 16 ? sampler_quad_pf_kernel<512, 2, 4, true, true, true>
                              : sampler_quad_pf_kernel<512, 2, 4, false, true, true>;
    const size_t smem = sizeof(float) * (static_cast<size_t>(a.l8_stride) + 16u * 32u * 17u);
    if (const cudaError_t e = smem_optin(kern, smem); e != cudaSuccess) return e;
    kern<<<n_units, 512, smem, s>>>(a);
    return cudaGetLastError();
}

int sampler_shape_from_name(const char* name) {
    const std::string v(name ? name : "");
    return v == "round" ? kShapeRound : v == "quad512" ? kShapeQuad512 : v == "quad256" ? kShapeQuad256
         : v == "global" ? kShapeGlobal : -1;
}

// ---- SamplerKind::kVanilla: the reference's O(K) baseline mode ---------------------------------
// vanilla_sample<float> over the dense count row (sampler.hpp:222-236, trainer.cpp:281-285): the
// sequential f32 prefix running_k = running_{k-1} + (f32(n_dk) + alpha) * bhat_k over all K topics,
// the draw f32(u0) * running_K, and prefix_search (first prefix >= draw).  The dense row is the
// document's C_dk row densified on the fly (DenseDocTopic cell k == count of topic k,
// trainer.cpp:49-63).  Lane per token, CTA per work unit (one word: its phi row staged in
// shared memory when it fits); the search re-runs the same chain and stops at the first prefix
// >= the draw, which equals the binary lower_bound on a non-decreasing prefix.  A baseline mode
// (O(K) per token, as in the reference), not a tuned path.
template <int NT, bool kGlobalPhi>
__global__ void __launch_bounds__(NT) sampler_vanilla_kernel(SamplerArgs a) {
    extern __shared__ __align__(16) float s_phi[];
    const Unit unit = a.units[blockIdx.x];
    const uint32_t v = unit.word;
    const float* gphi = a.bhat + static_cast<size_t>(v) * a.K_pad;
    if (!kGlobalPhi) {
        for (uint32_t i = threadIdx.x; i < a.K_pad / 4; i += NT)
            reinterpret_cast<float4*>(s_phi)[i] = __ldg(reinterpret_cast<const float4*>(gphi) + i);
        __syncthreads();
    }
    const float* phi = kGlobalPhi ? gphi : s_phi;
    uint32_t* brow = a.B + static_cast<size_t>(v) * a.K_pad;
    const uint32_t tbits = a.tbits, tmask = (1u << tbits) - 1u;
    const float alpha = a.alpha;
    unsigned long long entries = 0;
    for (uint32_t i = threadIdx.x; i < unit.length; i += NT) {
        const uint2 t = __ldg(a.tok + unit.offset + i);
        const uint32_t* row = a.A + static_cast<size_t>(t.x) * 4u;  // [nnz-1 | entries ...]
        const uint32_t nnz = (__ldg(row) & tmask) + 1u;
        entries += nnz;
        // The chain: running over k = 0..K-1, the row's entries consumed in ascending topic order.
        auto chain_step = [&](float run, uint32_t k, uint32_t& p, uint32_t& e) {
            uint32_t c = 0;
            if (p <= nnz && (e & tmask) == k) {
                c = e >> tbits;
                ++p;
                e = p <= nnz ? __ldg(row + p) : 0u;
            }
            const float w = __fadd_rn(__uint2float_rn(c), alpha);
            return __fadd_rn(run, __fmul_rn(w, kGlobalPhi ? __ldg(phi + k) : phi[k]));
        };
        float total = 0.0f;
        {
            uint32_t p = 1, e = __ldg(row + 1);
            for (uint32_t k = 0; k < a.K; ++k) total = chain_step(total, k, p, e);
        }
        float u0 = 0.0f, u1 = 0.0f;
        const uint64_t id = a.ids ? __ldg(a.ids + t.y) : a.id_base + t.y;
        draw2_f32(a.seed, a.stream_kind, id, u0, u1);
        const float x = __fmul_rn(u0, total);
        uint32_t topic = a.K - 1;  // x > total cannot happen (u0 <= 1); kept as the clamp
        {
            uint32_t p = 1, e = __ldg(row + 1);
            float run = 0.0f;
            for (uint32_t k = 0; k < a.K; ++k) {
                run = chain_step(run, k, p, e);
                if (run >= x) {
                    topic = k;
                    break;
                }
            }
        }
        store_topic(a, unit.offset + i, t.y, topic);
        atomicAdd(brow + topic, 1u);
    }
    if (a.row_entries) {
        for (int o = 16; o > 0; o >>= 1) entries += __shfl_xor_sync(0xffffffffu, entries, o);
        if ((threadIdx.x & 31u) == 0) atomicAdd(a.row_entries, entries);
    }
}

cudaError_t launch_vanilla(const SamplerArgs& a, uint32_t n_units, cudaStream_t s) {
    const size_t phi_bytes = sizeof(float) * static_cast<size_t>(a.K_pad);
    if (phi_bytes <= 200 * 1024) {
        if (const cudaError_t e = smem_optin(sampler_vanilla_kernel<256, false>, phi_bytes); e != cudaSuccess) return e;
        sampler_vanilla_kernel<256, false><<<n_units, 256, phi_bytes, s>>>(a);
    } else {
        sampler_vanilla_kernel<256, true><<<n_units, 256, 0, s>>>(a);
    }
    return cudaGetLastError();
}

// Launch shape by phi row size (SLDA_SAMPLER=round|quad512|quad256|global forces one where it fits):
//   quad256 : K_pad*4 <= 24 KB (C2 K=1K, C5 K=100): 256-thread quad-lane CTAs, 4 per SM
//   quad512 : two 512-thread quad-lane CTAs fit an SM (K_pad <= ~17.5K; C3 K=10K)
//   round   : the phi row still fits shared memory (K_pad <= ~45K): round-based 4-sector groups
//   global  : larger rows (C5 K=50K): quad-lane, phi gathered through L1/L2, L8 staged
int sampler_shape(const SamplerArgs& a) {
    if (a.vanilla) return kShapeVanilla;
    const size_t phi_bytes = sizeof(float) * (static_cast<size_t>(a.K_pad) + a.l8_stride);
    constexpr size_t kSm = 227 * 1024;
    const bool q256 = phi_bytes <= 24 * 1024 && 4 * sampler_quad_smem(a, 256) <= kSm;
    const bool q512 = 2 * sampler_quad_smem(a, 512) <= kSm;
    const bool round = sampler_smem(a, 256, 4) <= kSm;
    int shape = a.shape;
    if (shape == kShapeQuad256 && sampler_quad_smem(a, 256) > kSm) shape = -1;
    if (shape == kShapeQuad512 && sampler_quad_smem(a, 512) > kSm) shape = -1;
    if (shape == kShapeRound && !round) shape = -1;
    if (shape < 0) shape = q256 ? kShapeQuad256 : q512 ? kShapeQuad512 : round ? kShapeRound : kShapeGlobal;
    return shape;
}

cudaError_t launch_sampler(const SamplerArgs& a, uint32_t n_units, cudaStream_t s) {
    if (n_units == 0) return cudaSuccess;
    switch (sampler_shape(a)) {
        case kShapeVanilla: return launch_vanilla(a, n_units, s);
        case kShapeQuad256: return launch_quad_t<256, 4>(a, n_units, s);
        case kShapeQuad512: return launch_quad_t<512, 2>(a, n_units, s);
        case kShapeRound: return launch_round(a, n_units, s);
        default: return launch_quad_global(a, n_units, s);
    }
}

}  // namespace slda
