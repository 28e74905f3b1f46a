// Microbenchmark (not product code): global-load patterns for reading the sampler's short
// random C_dk rows cooperatively, and the cost of staging them through shared memory.
// A warp owns 32 rows; step g loads sectors [G*g, G*g+G) of all 32 rows (32/G rows per
// instruction, G sectors of one row per G adjacent lanes).  Rows start ALIGN-byte aligned.
//   mode 0: registers only (xor-sum of the loaded data)          -> the global-load path
//   mode 1: + STS into an (G*32+16)-byte-stride stage + LDS.128 by the owning lane
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o scripts/mb_pattern scripts/mb_pattern.cu
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

struct Sector { uint4 lo, hi; };
__device__ __forceinline__ Sector ld256(const void* p) {
    Sector s;
    asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=r"(s.lo.x), "=r"(s.lo.y), "=r"(s.lo.z), "=r"(s.lo.w), "=r"(s.hi.x), "=r"(s.hi.y), "=r"(s.hi.z), "=r"(s.hi.w)
        : "l"(p));
    return s;
}
__device__ __forceinline__ uint32_t xs(const uint4& v) { return v.x ^ v.y ^ v.z ^ v.w; }

// rows: sector offset + nsect per token (precomputed), G sectors per row per step.
template <int G, int MODE>
__global__ void __launch_bounds__(256) pat(const uint4* __restrict__ A, const uint2* __restrict__ tok, uint32_t ntok,
                                           uint32_t* out) {
    constexpr int RPI = 32 / G;                 // rows per instruction
    constexpr int STRIDE = G * 32 + 16;         // stage row stride
    extern __shared__ __align__(16) unsigned char sm[];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, sub = lane % G, grp = lane / G;
    unsigned char* stage = sm + warp * 32 * STRIDE;
    uint32_t acc = 0;
    const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
    for (uint32_t base = (blockIdx.x * (blockDim.x >> 5) + warp) * 32; base < ntok; base += nwarps * 32) {
        const uint2 t = tok[base + lane];  // {sector offset, nsect}
        uint32_t ro[G], ns[G];
#pragma unroll
        for (int j = 0; j < G; ++j) { ro[j] = __shfl_sync(~0u, t.x, RPI * j + grp); ns[j] = __shfl_sync(~0u, t.y, RPI * j + grp); }
        const uint32_t maxg = __reduce_max_sync(~0u, (t.y + G - 1) / G);
        Sector q[G];
#pragma unroll
        for (int j = 0; j < G; ++j) q[j] = sub < ns[j] ? ld256(A + 2 * (ro[j] + sub)) : Sector{};
        for (uint32_t g = 0; g < maxg; ++g) {
            const bool more = g + 1 < maxg;
            Sector nx[G];
            if (more) {
#pragma unroll
                for (int j = 0; j < G; ++j) {
                    const uint32_t sec = G * (g + 1) + sub;
                    nx[j] = sec < ns[j] ? ld256(A + 2 * (ro[j] + sec)) : Sector{};
                }
            }
            if (MODE == 0) {
#pragma unroll
                for (int j = 0; j < G; ++j) acc += xs(q[j].lo) + xs(q[j].hi);
            } else {
                __syncwarp();
#pragma unroll
                for (int j = 0; j < G; ++j) {
                    unsigned char* p = stage + (RPI * j + grp) * STRIDE + sub * 32;
                    *reinterpret_cast<uint4*>(p) = q[j].lo;
                    *reinterpret_cast<uint4*>(p + 16) = q[j].hi;
                }
                __syncwarp();
                const unsigned char* mine = stage + lane * STRIDE;
#pragma unroll
                for (int u = 0; u < G; ++u)
                    if (G * g + u < t.y) {
                        acc += xs(*reinterpret_cast<const uint4*>(mine + 32 * u));
                        acc += xs(*reinterpret_cast<const uint4*>(mine + 32 * u + 16));
                    }
            }
            if (more) {
#pragma unroll
                for (int j = 0; j < G; ++j) q[j] = nx[j];
            }
        }
    }
    if (acc == 0x9e3779b9u) out[0] = acc;
}


// lane-private: each lane streams its own row, P sectors per step (next step prefetched).
template <int P>
__global__ void __launch_bounds__(256) lanepriv(const uint4* __restrict__ A, const uint2* __restrict__ tok, uint32_t ntok,
                                                uint32_t* out) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t acc = 0;
    const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
    for (uint32_t base = (blockIdx.x * (blockDim.x >> 5) + warp) * 32; base < ntok; base += nwarps * 32) {
        const uint2 t = tok[base + lane];
        const uint32_t steps = (t.y + P - 1) / P;
        Sector q[P];
#pragma unroll
        for (int u = 0; u < P; ++u) q[u] = u < (int)t.y ? ld256(A + 2 * (t.x + u)) : Sector{};
        for (uint32_t g = 0; g < steps; ++g) {
            Sector nx[P];
#pragma unroll
            for (int u = 0; u < P; ++u) {
                const uint32_t sec = P * (g + 1) + u;
                nx[u] = sec < t.y ? ld256(A + 2 * (t.x + sec)) : Sector{};
            }
#pragma unroll
            for (int u = 0; u < P; ++u) acc += xs(q[u].lo) + xs(q[u].hi);
#pragma unroll
            for (int u = 0; u < P; ++u) q[u] = nx[u];
        }
    }
    if (acc == 0x9e3779b9u) out[0] = acc;
}

int main(int argc, char** argv) {
    const double mean_sect = argc > 1 ? atof(argv[1]) : 10.0;
    const uint32_t D = 8'000'000;
    std::mt19937_64 rng(7);
    std::lognormal_distribution<double> ln(0.0, 0.6);
    std::vector<uint32_t> nsv(D);
    for (uint32_t d = 0; d < D; ++d) {
        uint32_t n = (uint32_t)std::max(1.0, std::round(mean_sect * ln(rng) / 1.197));
        nsv[d] = std::min(n, 400u);
    }
    std::vector<uint32_t> order;
    for (uint32_t d = 0; d < D; ++d) { uint32_t len = nsv[d] * 7; for (uint32_t i = 0; i < len && order.size() < 500'000'000; ++i) order.push_back(d); }
    std::shuffle(order.begin(), order.end(), rng);
    const uint32_t ntok = (uint32_t)(order.size() / 32 * 32);
    double row_bytes = 0;
    for (uint32_t i = 0; i < ntok; ++i) row_bytes += 32.0 * nsv[order[i]];
    uint4* dA; uint2* dT; uint32_t* dO;
    CK(cudaMalloc(&dA, 6ull << 30)); CK(cudaMemset(dA, 1, 6ull << 30));
    CK(cudaMalloc(&dT, (size_t)ntok * 8)); CK(cudaMalloc(&dO, 4));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    printf("tokens %u, mean row %.1f B, row bytes %.1f GB\n", ntok, row_bytes / ntok, row_bytes / 1e9);
    for (int align : {32}) {
        std::vector<uint32_t> off(D);
        uint64_t tot = 0;
        const uint32_t asec = align / 32;
        for (uint32_t d = 0; d < D; ++d) { tot = (tot + asec - 1) / asec * asec; off[d] = (uint32_t)tot; tot += nsv[d]; }
        std::vector<uint2> tk(ntok);
        for (uint32_t i = 0; i < ntok; ++i) tk[i] = make_uint2(off[order[i]], nsv[order[i]]);
        CK(cudaMemcpy(dT, tk.data(), (size_t)ntok * 8, cudaMemcpyHostToDevice));
        auto timeit = [&](const char* name, auto kern, int G) {
            const int smem = 8 * 32 * (G * 32 + 16);
            CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            int occ = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, smem);
            auto launch = [&] { kern<<<148 * occ * 4, 256, smem>>>(dA, dT, ntok, dO); };
            launch(); CK(cudaDeviceSynchronize());
            cudaEventRecord(e0); launch(); launch(); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
            float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 2;
            CK(cudaGetLastError());
            printf("align %3d %-12s occ %d  %8.2f ms  %7.1f GB/s\n", align, name, occ, ms, row_bytes / ms / 1e6);
        };
        timeit("G2 regs", pat<2, 0>, 2);
        timeit("G4 regs", pat<4, 0>, 4);
        timeit("G8 regs", pat<8, 0>, 8);
        timeit("G2 stage", pat<2, 1>, 2);
        timeit("lane P2", lanepriv<2>, 0);
        timeit("lane P4", lanepriv<4>, 0);
        timeit("G4 stage", pat<4, 1>, 4);
    }
    return 0;
}
