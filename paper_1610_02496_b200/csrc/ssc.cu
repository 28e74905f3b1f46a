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
// shuffle is fused into the sampler's store.  Warp per document: a two-level
// topic bitmap (below).  Long documents: CTA per document, K-bin histogram +
// ordered compaction.
// ============================================================================

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

template <int R>
__device__ __forceinline__ uint32_t ssc_doc_bitmap(const uint32_t* key, uint32_t lane, const SscBitmapSmem& w,
                                                   uint32_t n1, uint32_t* out_row, uint32_t tbits) {
#pragma unroll
    for (uint32_t r = 0; r < R; ++r) {
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
    {
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

// Warps per CTA (C3, SSC alone / whole iteration): 2 -> 6.22 / 99.85 ms, 4 -> 6.26 / 99.87,
// 8 -> 6.45 / 100.16, 16 -> 6.57 / 100.40; smaller CTAs hand SMs back to the M-step sooner.
constexpr uint32_t kSscBmWarps = 4;

__host__ __device__ inline size_t ssc_bitmap_warp_bytes(uint32_t K_pad) {
    const size_t n0 = (K_pad + 31u) / 32u, n1 = (n0 + 31u) / 32u;
    const size_t b = 4 * n0 + 4 * n1 + 4 * kSscWarpCap + 2 * n0 + 2 * kSscWarpCap;
    return (b + 15u) & ~static_cast<size_t>(15u);
}

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
    // Software pipeline over the warp's documents: the next document's extent, row offset and
    // (up to 128) topics are loaded while this one is counted.
    auto meta = [&](uint32_t dd, uint32_t& s0, uint32_t& n, uint32_t& rq) {
        s0 = 0; n = 0; rq = 0;
        if (dd < a.D) {
            s0 = __ldg(a.doc_start + dd);
            n = __ldg(a.doc_start + dd + 1) - s0;
            rq = __ldg(a.row4 + dd);
        }
    };
    uint32_t s0, n, rq, key[4];
    meta(gw, s0, n, rq);
    ssc_load_keys<4>(a.z + s0, n <= 128 ? n : 0u, lane, key);
    for (uint32_t d = gw; d < a.D; d += nw) {
        const uint32_t cs0 = s0, cn = n;
        uint32_t* row = a.A + rq * 4u;
        const uint32_t k0 = key[0], k1 = key[1], k2 = key[2], k3 = key[3];
        meta(d + nw, s0, n, rq);
        ssc_load_keys<4>(a.z + s0, n <= 128 ? n : 0u, lane, key);
        if (cn > kSscWarpCap || cn == 0) continue;  // ssc_long_kernel / empty document
        uint32_t nnz;
        const uint32_t ck[4] = {k0, k1, k2, k3};
        if (cn <= 32) nnz = ssc_doc_bitmap<1>(ck, lane, w, n1, row, a.tbits);
        else if (cn <= 64) nnz = ssc_doc_bitmap<2>(ck, lane, w, n1, row, a.tbits);
        else if (cn <= 128) nnz = ssc_doc_bitmap<4>(ck, lane, w, n1, row, a.tbits);
        else if (cn <= 256) {
            uint32_t k8[8];
            ssc_load_keys<8>(a.z + cs0, cn, lane, k8);
            nnz = ssc_doc_bitmap<8>(k8, lane, w, n1, row, a.tbits);
        } else {
            uint32_t k16[16];
            ssc_load_keys<16>(a.z + cs0, cn, lane, k16);
            nnz = ssc_doc_bitmap<16>(k16, lane, w, n1, row, a.tbits);
        }
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
        const size_t bm_smem = kSscBmWarps * ssc_bitmap_warp_bytes(a.K_pad);  // <= 67 KB for K <= 65536
        if (const cudaError_t e = cudaFuncSetAttribute(ssc_bitmap_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                       static_cast<int>(bm_smem));
            e != cudaSuccess)
            return e;
        // Short-lived CTAs (16 documents per warp) rather than a persistent grid: SSC runs
        // beside the M-step on a low-priority stream, and retiring CTAs let the scheduler
        // hand SMs to the higher-priority colsum/phi CTAs.
        const uint32_t blocks = static_cast<uint32_t>((a.D + kSscBmWarps * 16u - 1) / (kSscBmWarps * 16u));
        ssc_bitmap_kernel<<<blocks, kSscBmWarps * 32, bm_smem, s>>>(a);
    }
    if (a.n_long > 0) {
        const size_t smem = sizeof(uint32_t) * a.K_pad;
        const uint32_t blocks = a.n_long < 148u * 2u ? a.n_long : 148u * 2u;
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
