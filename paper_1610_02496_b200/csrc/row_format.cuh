// row_format.cuh -- device-side C_dk row access of the sampler kernels (sampler.cu): sector
// loads, the entry decoder, the per-warp cooperative staging, and the tree search.
// Layouts: DESIGN.md §3.
#pragma once

#include "common.cuh"
#include "kernels.hpp"

namespace slda {

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

__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

__device__ __forceinline__ Sector zero_sector() { return Sector{make_uint4(0u, 0u, 0u, 0u), make_uint4(0u, 0u, 0u, 0u)}; }

// lower_bound over the word's L4 prefix (== WaryTree::sample, acceptance.cpp:140-200):
// binary search of the staged L8 level (first 8-block whose last prefix >= x), then the block's
// 8 prefixes re-derived from the previous block's end: L4 is the sequential f32 chain
// L4[c] = L4[c-1] + phi[c] (WaryTree::build) and L8[j-1] == L4[8j-1] exactly, so continuing the
// chain over the phi row (shared memory, or global when it is too large to stage) gives the
// very values the reference's tree holds -- no L4 array is stored or read.  Returns the first
// index with L4 >= x (x <= total; L8[j] = L4[8j+7] >= x ends the scan).
template <bool kGlobalPhi>
__device__ __forceinline__ uint32_t tree_search(float x, const float* s_l8, uint32_t n_l8, const float* phi) {
    uint32_t lo = 0, hi = n_l8 - 1;  // s_l8[n_l8 - 1] == total >= x
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (s_l8[mid] >= x) hi = mid; else lo = mid + 1;
    }
    float run = lo ? s_l8[lo - 1] : 0.0f;
    const float4* p4 = reinterpret_cast<const float4*>(phi + lo * kLeaf);
    const float4 a = kGlobalPhi ? __ldg(p4) : p4[0];
    const float4 b = kGlobalPhi ? __ldg(p4 + 1) : p4[1];
    const float f[7] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z};
    uint32_t i = 0;
#pragma unroll
    for (int k = 0; k < 7; ++k) {
        run = __fadd_rn(run, f[k]);
        i += run < x;  // non-decreasing: the count of prefixes below x is the first index >= x
    }
    return lo * kLeaf + i;
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

// ---- Row decoding for the round-based sampler ----------------------------------------------
// First pass over one staged sector (32 bytes) of a row.  Sector 0 starts with the header, a
// count-0 entry that adds +0.
__device__ __forceinline__ float acc_sector(float s, const unsigned char* p, uint32_t tbits, uint32_t tmask,
                                            const float* phi) {
    const uint4 lo = *reinterpret_cast<const uint4*>(p);
    const uint4 hi = *reinterpret_cast<const uint4*>(p + 16);
    s = acc_quad<false>(s, lo, tbits, tmask, phi);
    return acc_quad<false>(s, hi, tbits, tmask, phi);
}

// Prefix re-scan of one staged sector: first running sum >= xs.
__device__ __forceinline__ void scan_sector(float& run, bool& need, uint32_t& topic, float xs, const unsigned char* p,
                                            uint32_t tbits, uint32_t tmask, const float* phi) {
    const uint4 lo = *reinterpret_cast<const uint4*>(p);
    const uint4 hi = *reinterpret_cast<const uint4*>(p + 16);
    const uint32_t es[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
#pragma unroll
    for (int w = 0; w < 8; ++w) {
        run = __fadd_rn(run, entry_mass<false>(es[w], tbits, tmask, phi));
        if (need && run >= xs) {
            topic = es[w] & tmask;
            need = false;
        }
    }
}


// ---- phi row + L8 level staged by the TMA engine -----------------------------------------------
// One thread arms an mbarrier with the byte count and issues two bulk copies (cp.async.bulk,
// global -> shared, completing on the mbarrier); the CTA waits on the barrier's phase 0.  No
// registers or LSU instructions are spent on the 45 KB (K = 10K) staging, and the copies run
// while the CTA's warps start their first token loads.  Sizes are multiples of 16 bytes
// (K_pad % 32 == 0, l8_stride % 4 == 0) and both rows are 128-byte aligned.
__device__ __forceinline__ void tma_stage_rows(float* s_phi, const float* g_phi, uint32_t phi_bytes, float* s_l8,
                                               const float* g_l8, uint32_t l8_bytes, unsigned long long* bar) {
    const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(phi_bytes + l8_bytes)
                     : "memory");
        if (phi_bytes)  // 0: phi is read from global memory (rows too large for shared memory)
            asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(s_phi))), "l"(g_phi), "r"(phi_bytes),
                         "r"(b)
                         : "memory");
        asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(s_l8))), "l"(g_l8), "r"(l8_bytes), "r"(b)
                     : "memory");
    }
}
__device__ __forceinline__ void tma_wait_rows(unsigned long long* bar) {
    const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
    asm volatile("{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t"
                 "@!P1 bra WAIT_%=;\n\t}" ::"r"(b)
                 : "memory");
}

}  // namespace slda
