// zmove.cu -- the sampler's topics from execution order (word-major) to slot order
// (document-grouped z, what SSC, the z histogram and the getters read) on sm_100a.
//
// Why: a 2-byte store per token at a random slot dirties a 32-byte sector that the C_dk row
// stream evicts before its other 15 slots are written, so the sector is written back -- and read
// back for the merge -- about once per token: at C3 22.5 GB of the sampler's 27.3 GB of DRAM
// writes and 31 GB of its reads, 16.4 ms of an 85 ms launch.  Scattering the
// topics afterwards in one pass is no better: one L2 write request per token caps any pass at
// ~5.7 ms for C3's 738M tokens, and sectors filled over a long window are still written back
// partially.  So the sampler stores topics in execution order (full sectors) and three passes
// whose global stores are runs move them to slots:
//   1. zc = zx permuted to slot-range buckets (<= 256, 4M slots each at C3), bucket entries in
//      execution order: each CTA stages 16384 entries in shared memory and writes them bucket by
//      bucket (runs of ~64 entries; a run's destinations are consecutive, so each position carries
//      its source index and run id in one word, and the chunk's table one base per run);
//   2. zf = zc permuted to 16384-slot tiles, entries of a tile in zc order: the same kernel;
//   3. z = zf with each tile scattered inside shared memory by the slot's low 14 bits and stored
//      whole (fully coalesced).
// All tables are static (the PDOW order and the slots never change; engine.cu build_zlayout).
// Bytes per token per iteration: (2 + 4 + 2) x 2 + (2 + 2 + 2) = 22, plus the run tables
// (4 bytes per run: ~0.06 byte per token at C3).
#include "common.cuh"
#include "kernels.hpp"

namespace slda {

constexpr uint32_t kZChunk = 1u << kZChunkLog2;
constexpr uint32_t kZTile = 1u << kZTileLog2;
constexpr uint32_t kZWarps = 16;
constexpr uint32_t kZMaxKeys = 1024;  // keys per chunk: <= 256 buckets (level 1), <= 1024 tiles (level 2)

// One CTA per chunk: the chunk of src staged in shared memory; sorted position k of the chunk
// carries its source index (14 bits) and its run (bits 14+); the run's destinations are
// consecutive, so the chunk's table holds one base per run (first destination - first position,
// mod 2^32) instead of one destination per token.
__global__ void __launch_bounds__(512) zpermute_kernel(const uint16_t* __restrict__ src,
                                                       const uint32_t* __restrict__ zsk,
                                                       const uint32_t* __restrict__ zbase, uint32_t R, uint64_t T,
                                                       uint16_t* __restrict__ out) {
    __shared__ __align__(16) uint16_t buf[kZChunk];
    __shared__ uint32_t s_base[kZMaxKeys];
    const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kZChunk;
    const uint32_t n = static_cast<uint32_t>(min(static_cast<uint64_t>(kZChunk), T - base));
    if (n == kZChunk) {
        const uint4* s4 = reinterpret_cast<const uint4*>(src + base);
        uint4* b4 = reinterpret_cast<uint4*>(buf);
        for (uint32_t t = threadIdx.x; t < kZChunk / 8; t += blockDim.x) b4[t] = __ldg(s4 + t);
    } else {
        for (uint32_t t = threadIdx.x; t < n; t += blockDim.x) buf[t] = src[base + t];
    }
    for (uint32_t i = threadIdx.x; i < R; i += blockDim.x) s_base[i] = __ldg(zbase + static_cast<size_t>(blockIdx.x) * R + i);
    __syncthreads();
    for (uint32_t k = threadIdx.x; k < n; k += blockDim.x) {
        const uint32_t v = __ldg(zsk + base + k);
        out[s_base[v >> kZChunkLog2] + k] = buf[v & (kZChunk - 1u)];
    }
}

__global__ void __launch_bounds__(512) ztile_kernel(const uint16_t* __restrict__ zf, const uint16_t* __restrict__ loc,
                                                    uint64_t T, uint16_t* __restrict__ z) {
    __shared__ __align__(16) uint16_t buf[kZTile];
    const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kZTile;
    const uint32_t n = static_cast<uint32_t>(min(static_cast<uint64_t>(kZTile), T - base));
    {  // eight entries per thread per step: 16-byte loads of zf and loc (tile bases are 16384-aligned)
        const uint4* z4 = reinterpret_cast<const uint4*>(zf + base);
        const uint4* l4 = reinterpret_cast<const uint4*>(loc + base);
        for (uint32_t t = threadIdx.x; t < n / 8; t += blockDim.x) {
            const uint4 zv = __ldg(z4 + t), lv = __ldg(l4 + t);
            const uint32_t zw[4] = {zv.x, zv.y, zv.z, zv.w}, lw[4] = {lv.x, lv.y, lv.z, lv.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                buf[lw[j] & 0xFFFFu] = static_cast<uint16_t>(zw[j]);
                buf[lw[j] >> 16] = static_cast<uint16_t>(zw[j] >> 16);
            }
        }
        for (uint32_t k = (n & ~7u) + threadIdx.x; k < n; k += blockDim.x) buf[__ldg(loc + base + k)] = __ldg(zf + base + k);
    }
    __syncthreads();
    if (n == kZTile) {
        const uint4* b4 = reinterpret_cast<const uint4*>(buf);
        uint4* z4 = reinterpret_cast<uint4*>(z + base);
        for (uint32_t t = threadIdx.x; t < kZTile / 8; t += blockDim.x) z4[t] = b4[t];
    } else {
        for (uint32_t t = threadIdx.x; t < n; t += blockDim.x) z[base + t] = buf[t];
    }
}

cudaError_t launch_zpermute(const uint16_t* src, const uint32_t* zsk, const uint32_t* zbase, uint32_t R, uint64_t T,
                            uint16_t* out, cudaStream_t s) {
    if (T) zpermute_kernel<<<static_cast<uint32_t>((T + kZChunk - 1) / kZChunk), 512, 0, s>>>(src, zsk, zbase, R, T, out);
    return cudaGetLastError();
}

cudaError_t launch_ztile(const uint16_t* zf, const uint16_t* loc, uint64_t T, uint16_t* z, cudaStream_t s) {
    if (T) ztile_kernel<<<static_cast<uint32_t>((T + kZTile - 1) / kZTile), 512, 0, s>>>(zf, loc, T, z);
    return cudaGetLastError();
}

// ---- setup: the static tables --------------------------------------------------------------
// Both permutes are per-chunk stable counting sorts by a small key, so the tables come from two
// counting passes per level instead of global radix sorts (C3: 38 ms instead of 146-179 ms):
//   level 1: chunk c of the execution order, key = slot bucket (slot >> shift, <= 256 keys);
//            destinations (zc) are bucket-major, execution order inside a bucket;
//   level 2: chunk c of zc (inside one bucket: buckets are 2^shift >= 2^14 positions), key = the
//            slot's tile relative to the bucket's first tile (< 2^(shift-14) <= 1024 keys);
//            destinations (zf) are tile-major, zc order inside a tile.
// zhist_count_kernel counts (key, chunk) into a flat array whose order is the destination order,
// so its exclusive scan is every (key, chunk) run's first destination; zemit_kernel ranks each
// chunk's positions stably by key (warp segments walked in order, __match_any_sync peers) and
// writes zsk (source index | run << 14) and the chunk's run bases, plus slot_of at zc (level 1)
// or the tile-local slot at zf (level 2).
struct ZKeys {
    const uint2* tok;        // level 1: execution-order token records (.y = slot)
    const uint32_t* slot_of; // level 2: slot of every zc position
    uint64_t T;
    uint32_t shift;          // bucket = slot >> shift
    uint32_t level;          // 1 or 2
    uint32_t R;              // keys per chunk
    uint32_t nchunks;
};
__device__ __forceinline__ uint32_t zkey(const ZKeys& k, uint64_t p) {
    if (k.level == 1) return __ldg(&k.tok[p].y) >> k.shift;
    return (__ldg(k.slot_of + p) >> kZTileLog2) - (static_cast<uint32_t>(p >> k.shift) << (k.shift - kZTileLog2));
}
// Flat (key, chunk) index in destination order.
__device__ __forceinline__ size_t zflat(const ZKeys& k, uint32_t key, uint32_t c) {
    if (k.level == 1) return static_cast<size_t>(key) * k.nchunks + c;
    const uint32_t cpb = k.R, b = c / cpb;  // chunks per bucket == tiles per bucket
    return (static_cast<size_t>(b) * cpb + key) * cpb + (c - b * cpb);
}

__global__ void __launch_bounds__(512) zhist_count_kernel(ZKeys k, uint32_t* __restrict__ cnt) {
    __shared__ uint32_t h[kZMaxKeys];
    const uint32_t c = blockIdx.x;
    for (uint32_t i = threadIdx.x; i < k.R; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const uint64_t base = static_cast<uint64_t>(c) * kZChunk;
    const uint32_t n = static_cast<uint32_t>(min(static_cast<uint64_t>(kZChunk), k.T - base));
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) atomicAdd(h + zkey(k, base + i), 1u);
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < k.R; i += blockDim.x) cnt[zflat(k, i, c)] = h[i];
}

__global__ void __launch_bounds__(512) zemit_kernel(ZKeys k, const uint32_t* __restrict__ off,
                                                    uint32_t* __restrict__ zsk, uint32_t* __restrict__ zbase,
                                                    uint32_t* __restrict__ slot_of_out,
                                                    uint16_t* __restrict__ loc_out) {
    __shared__ uint16_t h[kZWarps * kZMaxKeys];  // per warp segment and key: count, then next local index
    __shared__ uint16_t start[kZMaxKeys];        // first local index of each key in the chunk
    const uint32_t c = blockIdx.x, w = threadIdx.x >> 5, lane = threadIdx.x & 31u, R = k.R;
    const uint64_t base = static_cast<uint64_t>(c) * kZChunk;
    const uint32_t n = static_cast<uint32_t>(min(static_cast<uint64_t>(kZChunk), k.T - base));
    constexpr uint32_t kSeg = kZChunk / kZWarps;
    const uint32_t s0 = w * kSeg, s1 = min(n, s0 + kSeg);
    for (uint32_t i = threadIdx.x; i < kZWarps * R; i += blockDim.x) h[i] = 0;
    __syncthreads();
    uint16_t* hw = h + w * R;
    const uint32_t lt = (1u << lane) - 1u;
    for (uint32_t p0 = s0; p0 < s1; p0 += 32) {
        const uint32_t p = p0 + lane;
        const uint32_t key = p < s1 ? zkey(k, base + p) : 0xFFFFFFFFu;
        const uint32_t peers = __match_any_sync(0xffffffffu, key);
        if (key != 0xFFFFFFFFu && (peers & lt) == 0) hw[key] = static_cast<uint16_t>(hw[key] + __popc(peers));
        __syncwarp();
    }
    __syncthreads();
    // Per key: warps' counts -> exclusive offsets over the warps; key totals -> chunk starts.
    __shared__ uint32_t tot[kZMaxKeys];
    for (uint32_t key = threadIdx.x; key < R; key += blockDim.x) {
        uint32_t run = 0;
        for (uint32_t ww = 0; ww < kZWarps; ++ww) {
            const uint32_t t = h[ww * R + key];
            h[ww * R + key] = static_cast<uint16_t>(run);
            run += t;
        }
        tot[key] = run;
    }
    __syncthreads();
    if (w == 0) {  // exclusive scan of the R <= 1024 key totals by one warp (contiguous lane ranges)
        const uint32_t per = (R + 31u) / 32u, a = min(R, lane * per), b = min(R, a + per);
        uint32_t mine = 0;
        for (uint32_t i = a; i < b; ++i) mine += tot[i];
        uint32_t incl = mine;
        for (uint32_t o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        uint32_t run = incl - mine;
        for (uint32_t i = a; i < b; ++i) {
            start[i] = static_cast<uint16_t>(run);
            run += tot[i];
        }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < kZWarps * R; i += blockDim.x)
        h[i] = static_cast<uint16_t>(h[i] + start[i % R]);
    // The chunk's run table: first destination - first sorted position of every run (mod 2^32).
    for (uint32_t key = threadIdx.x; key < R; key += blockDim.x)
        zbase[static_cast<size_t>(c) * R + key] = __ldg(off + zflat(k, key, c)) - start[key];
    __syncthreads();
    for (uint32_t p0 = s0; p0 < s1; p0 += 32) {
        const uint32_t p = p0 + lane;
        const bool v = p < s1;
        const uint32_t key = v ? zkey(k, base + p) : 0xFFFFFFFFu;
        const uint32_t peers = __match_any_sync(0xffffffffu, key);
        uint32_t local = 0;
        if (v) local = hw[key] + __popc(peers & lt);
        __syncwarp();
        if (v && (peers & lt) == 0) hw[key] = static_cast<uint16_t>(hw[key] + __popc(peers));
        __syncwarp();
        if (v) {
            const uint64_t kk = base + local;
            const uint32_t d = __ldg(off + zflat(k, key, c)) + (local - start[key]);
            zsk[kk] = p | (key << kZChunkLog2);
            if (k.level == 1) slot_of_out[d] = __ldg(&k.tok[base + p].y);
            else loc_out[d] = static_cast<uint16_t>(__ldg(k.slot_of + base + p) & (kZTile - 1u));
        }
    }
}

size_t zlayout_flat_size(uint64_t T, uint32_t shift, uint32_t level) {
    const uint64_t nchunks = (T + kZChunk - 1) / kZChunk, nbuckets = ((T - 1) >> shift) + 1;
    const uint64_t cpb = 1ull << (shift - kZTileLog2);
    return level == 1 ? nbuckets * nchunks : nbuckets * cpb * cpb;
}

cudaError_t launch_zlayout_count(const uint2* tok, const uint32_t* slot_of, uint64_t T, uint32_t shift,
                                 uint32_t level, uint32_t* cnt, size_t flat, cudaStream_t s) {
    if (!T) return cudaSuccess;
    const uint32_t nchunks = static_cast<uint32_t>((T + kZChunk - 1) / kZChunk);
    const uint32_t R = level == 1 ? static_cast<uint32_t>(((T - 1) >> shift) + 1) : 1u << (shift - kZTileLog2);
    if (R > kZMaxKeys || shift < kZTileLog2) return cudaErrorInvalidValue;
    if (const cudaError_t e = cudaMemsetAsync(cnt, 0, flat * 4, s); e != cudaSuccess) return e;
    zhist_count_kernel<<<nchunks, 512, 0, s>>>(ZKeys{tok, slot_of, T, shift, level, R, nchunks}, cnt);
    return cudaGetLastError();
}

uint32_t zlayout_keys(uint64_t T, uint32_t shift, uint32_t level) {
    return level == 1 ? static_cast<uint32_t>(((T - 1) >> shift) + 1) : 1u << (shift - kZTileLog2);
}

cudaError_t launch_zlayout_emit(const uint2* tok, const uint32_t* slot_of, uint64_t T, uint32_t shift, uint32_t level,
                                const uint32_t* off, uint32_t* zsk, uint32_t* zbase, uint32_t* slot_of_out,
                                uint16_t* loc_out, cudaStream_t s) {
    if (!T) return cudaSuccess;
    const uint32_t nchunks = static_cast<uint32_t>((T + kZChunk - 1) / kZChunk);
    const uint32_t R = level == 1 ? static_cast<uint32_t>(((T - 1) >> shift) + 1) : 1u << (shift - kZTileLog2);
    if (R > kZMaxKeys || shift < kZTileLog2) return cudaErrorInvalidValue;
    zemit_kernel<<<nchunks, 512, 0, s>>>(ZKeys{tok, slot_of, T, shift, level, R, nchunks}, off, zsk, zbase,
                                         slot_of_out, loc_out);
    return cudaGetLastError();
}

}  // namespace slda
