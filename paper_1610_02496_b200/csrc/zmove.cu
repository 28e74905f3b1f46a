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
//      bucket (runs of ~64 entries);
//   2. zf = zc permuted to 16384-slot tiles, entries of a tile in zc order: the same kernel;
//   3. z = zf with each tile scattered inside shared memory by the slot's low 14 bits and stored
//      whole (fully coalesced).
// All tables are static (the PDOW order and the slots never change; engine.cu build_zlayout).
// Bytes per token per iteration: (2 + 2 + 4 + 2) x 2 + (2 + 2 + 2) = 26.
#include "common.cuh"
#include "kernels.hpp"

namespace slda {

constexpr uint32_t kZChunk = 1u << kZChunkLog2;
constexpr uint32_t kZTile = 1u << kZTileLog2;

__global__ void __launch_bounds__(512) zpermute_kernel(const uint16_t* __restrict__ src,
                                                       const uint16_t* __restrict__ srcl,
                                                       const uint32_t* __restrict__ dst, uint64_t T,
                                                       uint16_t* __restrict__ out) {
    __shared__ __align__(16) uint16_t buf[kZChunk];
    const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kZChunk;
    const uint32_t n = static_cast<uint32_t>(min(static_cast<uint64_t>(kZChunk), T - base));
    if (n == kZChunk) {
        const uint4* s4 = reinterpret_cast<const uint4*>(src + base);
        uint4* b4 = reinterpret_cast<uint4*>(buf);
        for (uint32_t t = threadIdx.x; t < kZChunk / 8; t += blockDim.x) b4[t] = __ldg(s4 + t);
    } else {
        for (uint32_t t = threadIdx.x; t < n; t += blockDim.x) buf[t] = src[base + t];
    }
    __syncthreads();
    for (uint32_t k = threadIdx.x; k < n; k += blockDim.x) out[__ldg(dst + base + k)] = buf[__ldg(srcl + base + k)];
}

__global__ void __launch_bounds__(512) ztile_kernel(const uint16_t* __restrict__ zf, const uint16_t* __restrict__ loc,
                                                    uint64_t T, uint16_t* __restrict__ z) {
    __shared__ __align__(16) uint16_t buf[kZTile];
    const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kZTile;
    const uint32_t n = static_cast<uint32_t>(min(static_cast<uint64_t>(kZTile), T - base));
    for (uint32_t k = threadIdx.x; k < n; k += blockDim.x) buf[__ldg(loc + base + k)] = __ldg(zf + base + k);
    __syncthreads();
    if (n == kZTile) {
        const uint4* b4 = reinterpret_cast<const uint4*>(buf);
        uint4* z4 = reinterpret_cast<uint4*>(z + base);
        for (uint32_t t = threadIdx.x; t < kZTile / 8; t += blockDim.x) z4[t] = b4[t];
    } else {
        for (uint32_t t = threadIdx.x; t < n; t += blockDim.x) z[base + t] = buf[t];
    }
}

cudaError_t launch_zpermute(const uint16_t* src, const uint16_t* srcl, const uint32_t* dst, uint64_t T,
                            uint16_t* out, cudaStream_t s) {
    if (T) zpermute_kernel<<<static_cast<uint32_t>((T + kZChunk - 1) / kZChunk), 512, 0, s>>>(src, srcl, dst, T, out);
    return cudaGetLastError();
}

cudaError_t launch_ztile(const uint16_t* zf, const uint16_t* loc, uint64_t T, uint16_t* z, cudaStream_t s) {
    if (T) ztile_kernel<<<static_cast<uint32_t>((T + kZTile - 1) / kZTile), 512, 0, s>>>(zf, loc, T, z);
    return cudaGetLastError();
}

// ---- setup: the static tables --------------------------------------------------------------
#define ZFOR(i) for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < T; \
                     i += static_cast<uint64_t>(gridDim.x) * blockDim.x)

// mode 0: key = chunk(i) << 8 | (slot(i) >> shift)   (level-1 permute order)
// mode 1: key = slot(i) >> shift                    (level-1 destination order)
// mode 2: key = ord[i] >> shift (ord = the slots of the zc positions: level-2 destination order)
__global__ void zkey_u32_kernel(const uint2* __restrict__ tok, const uint32_t* __restrict__ ord, uint64_t T,
                                uint32_t mode, uint32_t shift, uint32_t* __restrict__ key) {
    ZFOR(i) {
        const uint32_t b = (mode == 2 ? ord[i] : tok[i].y) >> shift;
        key[i] = mode == 0 ? static_cast<uint32_t>((i >> kZChunkLog2) << 8) | b : b;
    }
}
// level 2 permute order: chunk(j) << 32 | tile(slot_of[j])
__global__ void zkey_u64_kernel(const uint32_t* __restrict__ slot_of, uint64_t T, uint32_t tile_shift,
                                unsigned long long* __restrict__ key) {
    ZFOR(j) key[j] = (static_cast<unsigned long long>(j >> kZChunkLog2) << 32) | (slot_of[j] >> tile_shift);
}
__global__ void zscatter_inv_kernel(const uint32_t* __restrict__ ord, uint64_t T, uint32_t* __restrict__ inv) {
    ZFOR(j) inv[ord[j]] = static_cast<uint32_t>(j);
}
// permute position k (chunk-major, sorted inside its chunk): its source inside the chunk and its
// destination (inv = position of the source in the destination order)
__global__ void ztables_kernel(const uint32_t* __restrict__ sorted, const uint32_t* __restrict__ inv, uint64_t T,
                               uint16_t* __restrict__ srcl, uint32_t* __restrict__ dst) {
    ZFOR(k) {
        const uint32_t from = sorted[k];
        srcl[k] = static_cast<uint16_t>(from & (kZChunk - 1u));
        dst[k] = inv[from];
    }
}
__global__ void zslot_of_kernel(const uint2* __restrict__ tok, const uint32_t* __restrict__ ord, uint64_t T,
                                uint32_t* __restrict__ slot_of) {
    ZFOR(j) slot_of[j] = tok[ord[j]].y;
}
__global__ void zloc_kernel(const uint32_t* __restrict__ slot_of, const uint32_t* __restrict__ ord, uint64_t T,
                            uint16_t* __restrict__ loc) {
    ZFOR(m) loc[m] = static_cast<uint16_t>(slot_of[ord[m]] & (kZTile - 1u));
}
#undef ZFOR

cudaError_t launch_zkey_u32(const uint2* tok, const uint32_t* ord, uint64_t T, uint32_t mode, uint32_t shift,
                            uint32_t* key, cudaStream_t s) {
    if (T) zkey_u32_kernel<<<148 * 8, 256, 0, s>>>(tok, ord, T, mode, shift, key);
    return cudaGetLastError();
}
cudaError_t launch_zkey_u64(const uint32_t* slot_of, uint64_t T, uint32_t tile_shift, unsigned long long* key,
                            cudaStream_t s) {
    if (T) zkey_u64_kernel<<<148 * 8, 256, 0, s>>>(slot_of, T, tile_shift, key);
    return cudaGetLastError();
}
cudaError_t launch_zscatter_inv(const uint32_t* ord, uint64_t T, uint32_t* inv, cudaStream_t s) {
    if (T) zscatter_inv_kernel<<<148 * 8, 256, 0, s>>>(ord, T, inv);
    return cudaGetLastError();
}
cudaError_t launch_ztables(const uint32_t* sorted, const uint32_t* inv, uint64_t T, uint16_t* srcl, uint32_t* dst,
                           cudaStream_t s) {
    if (T) ztables_kernel<<<148 * 8, 256, 0, s>>>(sorted, inv, T, srcl, dst);
    return cudaGetLastError();
}
cudaError_t launch_zslot_of(const uint2* tok, const uint32_t* ord, uint64_t T, uint32_t* slot_of, cudaStream_t s) {
    if (T) zslot_of_kernel<<<148 * 8, 256, 0, s>>>(tok, ord, T, slot_of);
    return cudaGetLastError();
}
cudaError_t launch_zloc(const uint32_t* slot_of, const uint32_t* ord, uint64_t T, uint16_t* loc, cudaStream_t s) {
    if (T) zloc_kernel<<<148 * 8, 256, 0, s>>>(slot_of, ord, T, loc);
    return cudaGetLastError();
}

}  // namespace slda
