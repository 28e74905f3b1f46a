// ssc.cu -- K4: shuffle-and-segmented-count rebuild of the C_dk rows on sm_100a.
//
// Reference paths are relative to /root/reference/proj.  See DESIGN.md §4.
#include <cstdlib>
#include <string>

#include "row_format.cuh"

namespace slda {

// ============================================================================
// K4 SSC -- rebuild_doc_topic (counts.cpp:103-125) + segmented_count (:65-94).
// Topics are already doc-grouped (the sampler writes them by slot), so the
// shuffle is fused into the sampler's store.  Warp per document: a lane-ranged
// topic bitmap (below).  Long documents: CTA per document, K-bin histogram +
// ordered compaction.
// ============================================================================

// SSC without a sort: a lane-ranged topic bitmap per warp.  Each token sets its topic's bit
// in a K-bit map; lane l owns the contiguous map words [4*cq*l, 4*cq*(l+1)), so one warp
// exclusive scan of the lanes' popcounts, plus a running prefix inside each lane's range,
// gives every map word the rank of its first topic (wpre).  A token's rank among the
// document's distinct topics is then wpre[word] + popc(word & below-bit mask): the counts
// are smem atomics at that rank and the topic is a plain store there (all duplicates store
// the same value), so the ordered (topic, count) row falls out with no sort and no emit
// loop.  Per document this costs O(len + K/1024) warp steps; the integer counts are order
// free, identical to segmented_count's (counts.cpp:65-94), and the row is topic-ascending
// like rebuild_doc_topic's CSR row (counts.cpp:103-125).
//
// cq (16-byte map chunks per lane) is odd, so the lanes' LDS.128 chunk reads (stride 16*cq
// bytes) hit distinct 4-bank groups in every quarter-warp phase.
struct SscWarpSmem {
    uint32_t* bm;    // 128*cq words (bit k = topic k present), all zero between documents
    uint16_t* wpre;  // per map word: rank of its first topic
    uint16_t* top;   // per rank: topic
    uint32_t* cnt;   // per rank: count (zero between documents); packed: two 16-bit counts per word
};

__host__ __device__ inline uint32_t ssc_chunks_per_lane(uint32_t K_pad) {
    const uint32_t words = (K_pad + 31u) / 32u;
    const uint32_t cq = (words + 127u) / 128u;
    return cq | 1u;
}

// Per-warp shared memory: the map (512 cq B), the word ranks (256 cq B), and per-rank topics and
// counts for up to `cap` distinct topics (nnz <= document length <= cap).
__host__ __device__ inline size_t ssc_warp_bytes(uint32_t K_pad, uint32_t cap = kSscWarpCap) {
    const size_t cq = ssc_chunks_per_lane(K_pad);
    const size_t cnt_bytes = (cap > kSscWarpCap ? 2 : 4) * static_cast<size_t>(cap);  // packed past 512
    const size_t b = 512 * cq + 256 * cq + 2 * static_cast<size_t>(cap) + cnt_bytes;
    return (b + 15u) & ~static_cast<size_t>(15u);
}


__device__ __forceinline__ uint32_t warp_excl_scan(uint32_t x, uint32_t lane, uint32_t& total) {
    uint32_t incl = x;
#pragma unroll
    for (uint32_t o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    total = __shfl_sync(0xffffffffu, incl, 31);
    return incl - x;
}

// Topics of one document striped over the warp (topic i in lane i % 32, register i / 32),
// 0xFFFFFFFF past the end.
template <int R>
__device__ __forceinline__ void ssc_load_keys(const uint16_t* z, uint32_t n, uint32_t lane, uint32_t* key) {
#pragma unroll
    for (uint32_t r = 0; r < R; ++r) {
        const uint32_t i = r * 32 + lane;
        key[r] = i < n ? static_cast<uint32_t>(__ldg(z + i)) : 0xFFFFFFFFu;
    }
}

// One document of n <= cap tokens: its first 128 topics are in key[] (prefetched), the rest are
// re-read from z (L1) by a runtime loop, so one code body serves every length (several
// length-specialised bodies overflow the instruction cache: ncu no_instruction stalls).  The
// loop issues four loads before their shared-memory updates (the medium pass is all loop).
// kPacked: counts (<= cap <= 65535) two per word, so the medium pass fits more warps per SM.
template <bool kPacked>
__device__ __forceinline__ uint32_t ssc_doc(const uint32_t* key, const uint16_t* z, uint32_t n, uint32_t lane,
                                            const SscWarpSmem& w, uint32_t cq, uint32_t* out_row, uint32_t tbits) {
    auto set_bit = [&](uint32_t k) { atomicOr(w.bm + (k >> 5), 1u << (k & 31u)); };
    auto count = [&](uint32_t k) {
        const uint32_t wi = k >> 5;
        const uint32_t rank = w.wpre[wi] + __popc(w.bm[wi] & ((1u << (k & 31u)) - 1u));
        if (kPacked)
            atomicAdd(w.cnt + (rank >> 1), 1u << ((rank & 1u) * 16u));
        else
            atomicAdd(w.cnt + rank, 1u);
        w.top[rank] = static_cast<uint16_t>(k);
    };
    auto rest = [&](auto&& f) {
#pragma unroll 1
        for (uint32_t i = 128 + lane; i < n; i += 128) {
            uint32_t t[4];
#pragma unroll
            for (uint32_t r = 0; r < 4; ++r) t[r] = i + 32 * r < n ? __ldg(z + i + 32 * r) : 0xFFFFFFFFu;
#pragma unroll
            for (uint32_t r = 0; r < 4; ++r)
                if (t[r] != 0xFFFFFFFFu) f(t[r]);
        }
    };
#pragma unroll
    for (uint32_t r = 0; r < 4; ++r)
        if (key[r] != 0xFFFFFFFFu) set_bit(key[r]);
    rest(set_bit);
    __syncwarp();
    // Lane-range popcounts -> warp exclusive scan -> per-word first ranks.  Up to kScanRegs
    // chunks per lane stay in registers between the two passes (K <= 12288: one read of the map).
    constexpr uint32_t kScanRegs = 3;
    const uint4* mine = reinterpret_cast<const uint4*>(w.bm) + lane * cq;
    uint2* wp = reinterpret_cast<uint2*>(w.wpre) + lane * cq;
    auto ranks = [](uint4 v, uint32_t& run) {
        const uint32_t r1 = run + __popc(v.x), r2 = r1 + __popc(v.y), r3 = r2 + __popc(v.z);
        const uint2 out = make_uint2(run | (r1 << 16), r2 | (r3 << 16));
        run = r3 + __popc(v.w);
        return out;
    };
    uint32_t nnz;
    if (cq <= kScanRegs) {
        uint4 v[kScanRegs];
        uint32_t c = 0;
#pragma unroll
        for (uint32_t j = 0; j < kScanRegs; ++j) {
            v[j] = j < cq ? mine[j] : make_uint4(0u, 0u, 0u, 0u);
            c += __popc(v[j].x) + __popc(v[j].y) + __popc(v[j].z) + __popc(v[j].w);
        }
        uint32_t run = warp_excl_scan(c, lane, nnz);
#pragma unroll
        for (uint32_t j = 0; j < kScanRegs; ++j)
            if (j < cq) wp[j] = ranks(v[j], run);
    } else {
        uint32_t c = 0;
#pragma unroll 1
        for (uint32_t j = 0; j < cq; ++j) {
            const uint4 v = mine[j];
            c += __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
        }
        uint32_t run = warp_excl_scan(c, lane, nnz);
#pragma unroll 1
        for (uint32_t j = 0; j < cq; ++j) wp[j] = ranks(mine[j], run);
    }
    __syncwarp();
#pragma unroll
    for (uint32_t r = 0; r < 4; ++r)
        if (key[r] != 0xFFFFFFFFu) count(key[r]);
    rest(count);
    __syncwarp();
    // Emit the row; the map is cleared once per distinct topic (nnz stores, not len).
#pragma unroll 1
    for (uint32_t e = lane; e < nnz; e += 32) {
        const uint32_t k = kPacked ? (w.cnt[e >> 1] >> ((e & 1u) * 16u)) & 0xFFFFu : w.cnt[e];
        const uint32_t t = w.top[e];
        w.cnt[kPacked ? e >> 1 : e] = 0u;  // (packed: both lanes of a word read it before either clears)
        w.bm[t >> 5] = 0u;
        out_row[1 + e] = t | (k << tbits);
    }
    const uint32_t padded = (nnz + 8u) & ~7u;
    if (nnz + 1 + lane < padded) out_row[nnz + 1 + lane] = 0u;  // < 8 pad words
    if (lane == 0) out_row[0] = nnz - 1u;
    __syncwarp();
    return nnz;
}

// Warps per CTA: short-lived 4-warp CTAs hand SMs back to the concurrent M-step sooner
// (bitmap SSC, C3, SSC alone / whole iteration: 2 -> 6.22 / 99.85 ms, 4 -> 6.26 / 99.87,
// 8 -> 6.45 / 100.16, 16 -> 6.57 / 100.40).
constexpr uint32_t kSscWarps = 4;

// kCap = kSscWarpCap: every document (those longer are skipped); kCap = kSscMidCap: the
// long-document list, those of at most kCap tokens.
template <uint32_t kCap, int MINB>
__global__ void __launch_bounds__(kSscWarps * 32, MINB) ssc_warp_kernel(SscArgs a) {
    constexpr bool kList = kCap > kSscWarpCap;
    extern __shared__ __align__(16) unsigned char s_raw[];
    const uint32_t wid = threadIdx.x >> 5, lane = lane_id();
    const uint32_t cq = ssc_chunks_per_lane(a.K_pad);
    unsigned char* base = s_raw + wid * ssc_warp_bytes(a.K_pad, kCap);
    SscWarpSmem w;
    w.bm = reinterpret_cast<uint32_t*>(base);
    w.wpre = reinterpret_cast<uint16_t*>(w.bm + 128 * cq);
    w.cnt = reinterpret_cast<uint32_t*>(w.wpre + 128 * cq);
    w.top = reinterpret_cast<uint16_t*>(w.cnt + (kList ? kCap / 2 : kCap));
    {
        uint4* b4 = reinterpret_cast<uint4*>(w.bm);
        for (uint32_t i = lane; i < 32 * cq; i += 32) b4[i] = make_uint4(0u, 0u, 0u, 0u);
        for (uint32_t i = lane; i < (kList ? kCap / 2 : kCap); i += 32) w.cnt[i] = 0u;
    }
    __syncwarp();
    unsigned long long nnz_acc = 0;
    const uint32_t gw = blockIdx.x * kSscWarps + wid, nw = gridDim.x * kSscWarps;
    const uint32_t ndocs = kList ? a.n_long - a.n_huge : a.D;
    const uint32_t* list = a.long_docs + a.n_huge;
    // Software pipeline over the warp's documents: the next document's extent, row offset and
    // (up to 128) topics are loaded while this one is counted.
    auto meta = [&](uint32_t dd, uint32_t& s0, uint32_t& n, uint32_t& rq) {
        s0 = 0; n = 0; rq = 0;
        if (dd < ndocs) {
            const uint32_t doc = kList ? __ldg(list + dd) : dd;
            s0 = __ldg(a.doc_start + doc);
            n = __ldg(a.doc_start + doc + 1) - s0;
            rq = __ldg(a.row4 + doc);
        }
    };
    uint32_t s0, n, rq, key[4];
    meta(gw, s0, n, rq);
    ssc_load_keys<4>(a.z + s0, n <= kCap ? n : 0u, lane, key);
    for (uint32_t d = gw; d < ndocs; d += nw) {
        const uint32_t cs0 = s0, cn = n;
        uint32_t* row = a.A + rq * 4u;
        // (the prefetched keys cover the first 128 topics of documents up to kCap)
        const uint32_t k0 = key[0], k1 = key[1], k2 = key[2], k3 = key[3];
        meta(d + nw, s0, n, rq);
        ssc_load_keys<4>(a.z + s0, n <= kCap ? n : 0u, lane, key);
        if (cn > kCap || cn == 0) continue;  // a longer document's kernel / empty document
        const uint32_t ck[4] = {k0, k1, k2, k3};
        const uint32_t nnz = ssc_doc<kList>(ck, a.z + cs0, cn, lane, w, cq, row, a.tbits);
        nnz_acc += nnz;
    }
    if (lane == 0 && nnz_acc) atomicAdd(a.nnz_total, nnz_acc);
}

// Long documents: one CTA per document (grid-stride over the long-doc list).
template <bool kSmemHist>
__global__ void __launch_bounds__(256) ssc_long_kernel(SscArgs a) {
    extern __shared__ __align__(16) uint32_t s_dyn[];
    __shared__ uint32_t s_scan[256];
    uint32_t* hist = kSmemHist ? s_dyn : a.hist_scratch + static_cast<size_t>(blockIdx.x) * a.K_pad;
    const uint32_t tid = threadIdx.x;
    const uint32_t per = (a.K_pad + 255u) / 256u;
    for (uint32_t li = blockIdx.x; li < a.n_huge; li += gridDim.x) {
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
        {
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

cudaError_t launch_ssc(const SscArgs& a, cudaStream_t s) {
    if (a.D > 0) {
        const size_t bm_smem = kSscWarps * ssc_warp_bytes(a.K_pad);  // <= 59 KB for K <= 65536
        auto kern = ssc_warp_kernel<kSscWarpCap, 8>;
        if (const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                       static_cast<int>(bm_smem));
            e != cudaSuccess)
            return e;
        // Short-lived CTAs (16 documents per warp) rather than a persistent grid: SSC runs
        // beside the M-step on a low-priority stream, and retiring CTAs let the scheduler
        // hand SMs to the higher-priority colsum/phi CTAs.
        const uint32_t blocks = static_cast<uint32_t>((a.D + kSscWarps * 16u - 1) / (kSscWarps * 16u));
        kern<<<blocks, kSscWarps * 32, bm_smem, s>>>(a);
    }
    if (a.n_long > a.n_huge) {  // medium documents: warps with kSscMidCap rank arrays
        const size_t mid_smem = kSscWarps * ssc_warp_bytes(a.K_pad, kSscMidCap);  // <= 84 KB
        auto kern = ssc_warp_kernel<kSscMidCap, 4>;
        if (const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                       static_cast<int>(mid_smem));
            e != cudaSuccess)
            return e;
        const uint32_t blocks = (a.n_long - a.n_huge + kSscWarps * 4u - 1) / (kSscWarps * 4u);
        kern<<<blocks, kSscWarps * 32, mid_smem, s>>>(a);
    }
    if (a.n_huge > 0) {  // documents longer than kSscMidCap: one CTA histogram each
        const size_t smem = sizeof(uint32_t) * a.K_pad;
        const uint32_t blocks = a.n_huge < 148u * 2u ? a.n_huge : 148u * 2u;
        if (smem <= 200 * 1024) {
            if (const cudaError_t e = cudaFuncSetAttribute(ssc_long_kernel<true>,
                                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                           static_cast<int>(smem));
                e != cudaSuccess)
                return e;
            ssc_long_kernel<true><<<blocks, 256, smem, s>>>(a);
        } else {
            ssc_long_kernel<false><<<blocks, 256, 0, s>>>(a);
        }
    }
    return cudaGetLastError();
}

}  // namespace slda
