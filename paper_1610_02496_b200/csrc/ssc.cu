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

template <int R, bool kCompact>
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

// Warps per CTA (C3, SSC alone / whole iteration): 2 -> 6.22 / 99.85 ms, 4 -> 6.26 / 99.87,
// 8 -> 6.45 / 100.16, 16 -> 6.57 / 100.40; smaller CTAs hand SMs back to the M-step sooner.
constexpr uint32_t kSscBmWarps = 4;

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
        if (cn <= 32) nnz = ssc_doc_bitmap<1, kCompact>(ck, lane, w, n1, row, a.tbits);
        else if (cn <= 64) nnz = ssc_doc_bitmap<2, kCompact>(ck, lane, w, n1, row, a.tbits);
        else if (cn <= 128) nnz = ssc_doc_bitmap<4, kCompact>(ck, lane, w, n1, row, a.tbits);
        else if (cn <= 256) {
            uint32_t k8[8];
            ssc_load_keys<8>(a.z + cs0, cn, lane, k8);
            nnz = ssc_doc_bitmap<8, kCompact>(k8, lane, w, n1, row, a.tbits);
        } else {
            uint32_t k16[16];
            ssc_load_keys<16>(a.z + cs0, cn, lane, k16);
            nnz = ssc_doc_bitmap<16, kCompact>(k16, lane, w, n1, row, a.tbits);
        }
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

}  // namespace slda
