// mstep.cu -- K5/K6: column sums, phi and the tree prefix (the M-step) on sm_100a.
//
// Reference paths are relative to /root/reference/proj.  See DESIGN.md §4.
#include "common.cuh"
#include "kernels.hpp"

#include <cuda.h>  // CUtensorMap (the encoder is fetched through the runtime: no -lcuda)
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdlib>
#include <string>

namespace slda {

// ============================================================================
// K5/K6 -- preprocess (counts.cpp:37-63) + rebuild_trees (trainer.cpp:237-248,
// sampler.hpp:58-90, :142-149).  colsum: integer column sums (order-free).
// phi: thread per word row, 32-column tiles staged in shared memory by cp.async
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

// C_k from the topics themselves (one engine holding every token of C_wk): C_k is the number of
// tokens assigned topic k, so a histogram of z (2 B/token, 1.48 GB at C3) gives exactly the
// column sums of C_wk (4 B/cell, 5.64 GB).  Per-CTA shared-memory bins, flushed once.
__global__ void __launch_bounds__(512) zhist_kernel(const uint16_t* __restrict__ z, uint64_t T, uint32_t K_pad,
                                                    unsigned long long* __restrict__ colsum) {
    extern __shared__ uint32_t s_bin[];
    for (uint32_t i = threadIdx.x; i < K_pad; i += blockDim.x) s_bin[i] = 0u;
    __syncthreads();
    const uint64_t n8 = T / 8, stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    const uint4* z8 = reinterpret_cast<const uint4*>(z);
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n8; i += stride) {
        const uint4 v = __ldg(z8 + i);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            atomicAdd(s_bin + (w[j] & 0xFFFFu), 1u);
            atomicAdd(s_bin + (w[j] >> 16), 1u);
        }
    }
    for (uint64_t i = n8 * 8 + blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < T; i += stride)
        atomicAdd(s_bin + z[i], 1u);
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < K_pad; i += blockDim.x)
        if (s_bin[i]) atomicAdd(colsum + i, static_cast<unsigned long long>(s_bin[i]));
}

bool zhist_fits(uint32_t K_pad) { return static_cast<size_t>(K_pad) * 4 <= 200 * 1024; }

cudaError_t launch_zhist(const uint16_t* z, uint64_t T, uint32_t K_pad, unsigned long long* colsum, cudaStream_t s) {
    const size_t smem = static_cast<size_t>(K_pad) * 4;
    if (!zhist_fits(K_pad)) return cudaErrorInvalidValue;
    if (const cudaError_t e = cudaFuncSetAttribute(zhist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   static_cast<int>(smem));
        e != cudaSuccess)
        return e;
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, zhist_kernel, 512, smem);
    const uint64_t want = (T / 8 + 511) / 512;
    uint64_t grid = static_cast<uint64_t>(sms) * (per_sm > 0 ? per_sm : 1);
    if (want < grid) grid = want ? want : 1;
    zhist_kernel<<<static_cast<uint32_t>(grid), 512, smem, s>>>(z, T, K_pad, colsum);
    return cudaGetLastError();
}

// bhat = f32((cnt + beta) / denom_k) with the double quotient correctly rounded
// (counts.cpp:58-60), without a per-cell double division.  y = RN(x * RN(1/denom)) is within
// 2.5 double ulps of RN(x / denom), so both round to the same f32 unless an f32 rounding
// boundary (a midpoint between adjacent floats: low 29 mantissa bits == 2^28) lies within a
// few ulps of y, or y leaves the f32 normal range; those cells (~2^-22 of them) take the
// exact division.  rcp is NaN when RN(1/denom) is not a normal double, forcing the exact path.
__device__ __forceinline__ float phi_quotient(double x, double den, double rcp) {
    const double y = __dmul_rn(x, rcp);
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(y));
    const uint32_t lo = static_cast<uint32_t>(b) & 0x1FFFFFFFu;
    const uint32_t ex = static_cast<uint32_t>(b >> 52) & 0x7FFu;
    const bool near_mid = lo - (0x10000000u - 64u) <= 128u;
    const bool out_of_range = ex - 898u > 1149u - 898u;  // y in [2^-125, 2^127): f32 normal
    if (__builtin_expect(near_mid || out_of_range, 0)) return __double2float_rn(__ddiv_rn(x, den));
    return __double2float_rn(y);
}

__device__ __forceinline__ double phi_reciprocal(double den) {
    const double r = __ddiv_rn(1.0, den);
    const uint32_t ex = static_cast<uint32_t>(static_cast<unsigned long long>(__double_as_longlong(r)) >> 52) & 0x7FFu;
    return ex == 0u || ex == 0x7FFu ? __longlong_as_double(0x7FF8000000000000ll) : r;
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
        denom[K_pad + k] = phi_reciprocal(d);
        zv[k] = __double2float_rn(__ddiv_rn(__dadd_rn(0.0, beta), d));
    } else {
        denom[k] = 1.0;
        denom[K_pad + k] = 1.0;
        zv[k] = 0.0f;
    }
}

cudaError_t launch_denom(const unsigned long long* colsum, uint32_t K, uint32_t K_pad, uint32_t V,
                         double beta, double* denom, float* zv, cudaStream_t s) {
    denom_kernel<<<(K_pad + 255) / 256, 256, 0, s>>>(colsum, K, K_pad, V, beta, denom, zv);
    return cudaGetLastError();
}

// One thread per word row (the L4 prefix is a sequential f32 chain), 64 rows per CTA and
// C-column tiles (default C = 32).  A tile of C_wk lands in shared memory by cp.async (C/4
// threads per row segment, coalesced) in an S-stage pipeline, together with its columns'
// denom, 1/denom and zero-count bhat; each thread then reads its own row, writes bhat in place
// and the L4 prefix beside it, and the CTA stores both tiles back with the copy mapping.
// 16-byte quads are XOR-swizzled by row so the per-row and the per-segment accesses are both
// bank-conflict free.  32 x 4: 44 KB of shared memory, 5 CTAs = 320 rows per SM, 3 tiles
// (24 KB per CTA) in flight.  Padded columns (>= K) hold zero counts and zv = 0, so they add
// +0.0f to the chain (unchanged) and store bhat = 0, as the reference's padding.
constexpr int kPhiRows = 64;

// Word offset of 16-byte quad `quad` of tile row `row` (C columns, C/4 quads per row): quads are
// XOR-swizzled so eight consecutive rows reading the same quad, and one row-segment's quads
// read by consecutive threads, both fall in distinct banks.
template <int C>
__device__ __forceinline__ uint32_t phi_swz(uint32_t row, uint32_t quad) {
    constexpr uint32_t Q = C / 4, sh = Q == 4 ? 1u : 0u;
    return row * C + ((quad ^ ((row >> sh) & (Q - 1u))) << 2);
}

__device__ __forceinline__ void phi_cp16(void* smem, const void* gmem, bool valid) {
    const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(valid ? 16 : 0)
                 : "memory");
}

template <int C, int S>
constexpr size_t phi_smem_bytes() {
    return static_cast<size_t>(S) * (2 * C * 8 + kPhiRows * C * 4 + C * 4);
}

template <int C, int S>
__global__ void __launch_bounds__(kPhiRows, 4) phi_kernel(const uint32_t* __restrict__ B,
                                                         const double* __restrict__ denom,
                                                         const float* __restrict__ zv,
                                                         float* __restrict__ bhat,
                                                         float* __restrict__ l8, float* __restrict__ q,
                                                         uint32_t row_begin, uint32_t row_end,
                                                         uint32_t K_pad, uint32_t l8_stride, double beta,
                                                         float falpha) {
    static_assert(C == 16 || C == 32 || C == 64, "tile width");
    constexpr uint32_t Q = C / 4;              // quads per tile row
    constexpr uint32_t RP = kPhiRows / Q;      // rows per copy pass
    extern __shared__ __align__(16) unsigned char phi_smem[];
    // [stage][2][C] denom, 1/denom | [stage][rows*C] counts, then bhat | [stage][C] zv
    auto s_den = reinterpret_cast<double(*)[2][C]>(phi_smem);
    auto t_in = reinterpret_cast<uint32_t(*)[kPhiRows * C]>(phi_smem + S * 2 * C * 8);
    auto s_zv = reinterpret_cast<float(*)[C]>(phi_smem + S * (2 * C * 8 + kPhiRows * C * 4));
    const double* __restrict__ rcp = denom + K_pad;
    const uint32_t tid = threadIdx.x;
    const uint32_t v0 = row_begin + blockIdx.x * kPhiRows;
    const uint32_t v = v0 + tid;
    // Copy / store role: quad cq of rows crow + RP*p, p = 0..Q-1.
    const uint32_t cq = tid % Q, crow = tid / Q;
    const size_t stride = static_cast<size_t>(RP) * K_pad;
    const size_t g0 = static_cast<size_t>(v0 + crow) * K_pad + cq * 4u;
    const uint32_t ntiles = (K_pad + C - 1) / C;  // K_pad is a multiple of 32: a 64-column tile may be half
    auto issue = [&](uint32_t c0, int st) {
#pragma unroll
        for (uint32_t p = 0; p < Q; ++p) {
            const bool ok = v0 + crow + RP * p < row_end && (C <= 32 || c0 + cq * 4u < K_pad);
            phi_cp16(&t_in[st][phi_swz<C>(crow + RP * p, cq)], ok ? B + g0 + p * stride + c0 : B, ok);
        }
#pragma unroll
        for (uint32_t i = tid; i < C + C / 4; i += kPhiRows) {
            // past K_pad (half tile): zero-filled, so the padding cells read zv = 0
            const uint32_t col = i < C / 2 ? i * 2 : i < C ? (i - C / 2) * 2 : (i - C) * 4;
            const bool in = c0 + col < K_pad;
            if (i < C / 2) phi_cp16(&s_den[st][0][col], in ? denom + c0 + col : denom, in);
            else if (i < C) phi_cp16(&s_den[st][1][col], in ? rcp + c0 + col : rcp, in);
            else phi_cp16(&s_zv[st][col], in ? zv + c0 + col : zv, in);
        }
    };
    float run = 0.0f;
#pragma unroll
    for (uint32_t t = 0; t + 1 < S; ++t) {
        if (t < ntiles) issue(t * C, t);
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
    for (uint32_t t = 0; t < ntiles; ++t) {
        const int st = t % S;
        const uint32_t c0 = t * C;
        asm volatile("cp.async.wait_group %0;\n" ::"n"(S - 2) : "memory");
        __syncthreads();  // tile t visible; tile t-1's stores have read its stage
        if (t + S - 1 < ntiles) issue(c0 + (S - 1) * C, (t + S - 1) % S);
        asm volatile("cp.async.commit_group;\n" ::: "memory");
        float l8v[Q / 2];
#pragma unroll
        for (uint32_t j = 0; j < Q; ++j) {
            const uint32_t o = phi_swz<C>(tid, j);
            const uint4 cnt = *reinterpret_cast<const uint4*>(&t_in[st][o]);
            float4 bh = *reinterpret_cast<const float4*>(&s_zv[st][j * 4]);
            if ((cnt.x | cnt.y | cnt.z | cnt.w) != 0u) {
                const double* d = &s_den[st][0][j * 4];
                const double* r = &s_den[st][1][j * 4];
                if (cnt.x) bh.x = phi_quotient(__dadd_rn(static_cast<double>(cnt.x), beta), d[0], r[0]);
                if (cnt.y) bh.y = phi_quotient(__dadd_rn(static_cast<double>(cnt.y), beta), d[1], r[1]);
                if (cnt.z) bh.z = phi_quotient(__dadd_rn(static_cast<double>(cnt.z), beta), d[2], r[2]);
                if (cnt.w) bh.w = phi_quotient(__dadd_rn(static_cast<double>(cnt.w), beta), d[3], r[3]);
            }
            // The L4 prefix (sequential f32 chain, WaryTree::build) is not stored: only its value
            // at every 8th column (L8) and the total.  The sampler re-derives a block's 8 prefixes
            // from L8 and the phi row when it needs them (row_format.cuh tree_search).
            run = __fadd_rn(run, bh.x);
            run = __fadd_rn(run, bh.y);
            run = __fadd_rn(run, bh.z);
            run = __fadd_rn(run, bh.w);
            *reinterpret_cast<float4*>(&t_in[st][o]) = bh;
            if (j & 1u) l8v[j >> 1] = run;  // L8: the prefix at every 8th column
        }
        if (v < row_end) {
            const size_t o8 = static_cast<size_t>(v) * l8_stride + c0 / kLeaf;
            if (C >= 32) {
#pragma unroll
                for (uint32_t h = 0; h < Q / 8; ++h) {
                    if (c0 + 32 * h >= K_pad) break;
                    const float4 x = make_float4(l8v[4 * h], l8v[(4 * h + 1) % (Q / 2)], l8v[(4 * h + 2) % (Q / 2)],
                                                 l8v[(4 * h + 3) % (Q / 2)]);
                    *reinterpret_cast<float4*>(l8 + o8 + 4 * h) = x;
                }
            } else {
                const float2 x = make_float2(l8v[0], l8v[1 % (Q / 2)]);
                *reinterpret_cast<float2*>(l8 + o8) = x;
            }
        }
        __syncthreads();
#pragma unroll
        for (uint32_t p = 0; p < Q; ++p) {
            if (v0 + crow + RP * p < row_end && (C <= 32 || c0 + cq * 4u < K_pad)) {
                const uint32_t o = phi_swz<C>(crow + RP * p, cq);
                const float4 b = *reinterpret_cast<const float4*>(&t_in[st][o]);
                *reinterpret_cast<float4*>(bhat + g0 + p * stride + c0) = b;
            }
        }
    }
    if (v < row_end) {
        for (uint32_t j = K_pad / kLeaf; j < l8_stride; ++j) l8[static_cast<size_t>(v) * l8_stride + j] = run;
        q[v] = __fmul_rn(falpha, run);  // trainer.cpp:245
    }
}

// ---- phi by TMA tiles: warp per 32 word rows ---------------------------------------------------
// The same per-row computation as phi_kernel (thread = row, the sequential f32 chain over the
// row), but each warp owns its 32 rows and moves 32 x 32 tiles with the TMA engine: a 2-D tensor
// load of C_wk (128-byte swizzle: lane r reads 16-byte chunk j of its row at j ^ (r & 7), so
// every quarter-warp covers all 32 banks) plus 1-D bulk copies of the tile's denom / 1/denom /
// zero-count phi, all completing on one mbarrier per stage; phi is written back into the tile
// in place and a 2-D tensor store returns it.  No CTA barriers, no per-thread copy or store
// loops: one lane issues three TMA operations per tile.  The tensor maps start at row_begin with
// row_end - row_begin rows, so the last group's rows past the slice are zero-filled on load and
// clipped on store.
constexpr uint32_t kPhiTileBytes = 32u * 32u * 4u;          // 32 rows x 32 columns, u32 / f32
constexpr uint32_t kPhiAuxBytes = 32u * 8u * 2u + 32u * 4u;  // denom, 1/denom (f64), zero-count phi

template <int S, int W>
constexpr size_t phi_tma_smem_bytes() {
    return 1024 + static_cast<size_t>(W) * S * (kPhiTileBytes + kPhiAuxBytes + 8);
}

__device__ __forceinline__ void mbar_wait_parity(uint32_t bar, uint32_t parity) {
    asm volatile("{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
                 "@!P1 bra WAIT_%=;\n\t}" ::"r"(bar), "r"(parity)
                 : "memory");
}

template <int S, int W>
__global__ void __launch_bounds__(W * 32) phi_tma_kernel(const __grid_constant__ CUtensorMap t_cnt,
                                                         const __grid_constant__ CUtensorMap t_phi,
                                                         const double* __restrict__ denom,
                                                         const float* __restrict__ zv, float* __restrict__ l8,
                                                         float* __restrict__ q, uint32_t row_begin, uint32_t rows,
                                                         uint32_t K_pad, uint32_t l8_stride, double beta,
                                                         float falpha) {
    static_assert(S >= 3, "one stage computing, one being stored, at least one loading");
    extern __shared__ unsigned char phi_tma_raw[];
    // 128-byte swizzled TMA tiles need 1024-byte aligned destinations.
    unsigned char* base = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(phi_tma_raw) + 1023u) & ~static_cast<uintptr_t>(1023u));
    const uint32_t wid = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const uint32_t r0 = (blockIdx.x * W + wid) * 32u;  // first row of this warp (slice-relative)
    if (r0 >= rows) return;                             // warp-uniform; no CTA barriers below
    unsigned char* tiles = base + wid * S * kPhiTileBytes;
    unsigned char* aux = base + W * S * kPhiTileBytes + wid * S * kPhiAuxBytes;
    const uint32_t bars = static_cast<uint32_t>(__cvta_generic_to_shared(
        base + W * S * (kPhiTileBytes + kPhiAuxBytes) + wid * S * 8u));
    const uint32_t ntiles = K_pad / 32u;
    if (lane == 0) {
#pragma unroll
        for (int st = 0; st < S; ++st)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bars + st * 8u) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    auto load = [&](uint32_t t) {  // lane 0: tile t of C_wk + its columns' denom, 1/denom, zv
        const uint32_t st = t % S, bar = bars + st * 8u, c0 = t * 32u;
        const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(tiles + st * kPhiTileBytes));
        const uint32_t adst = static_cast<uint32_t>(__cvta_generic_to_shared(aux + st * kPhiAuxBytes));
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                     "r"(kPhiTileBytes + kPhiAuxBytes)
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
            ::"r"(dst), "l"(reinterpret_cast<uint64_t>(&t_cnt)), "r"(c0), "r"(r0), "r"(bar)
            : "memory");
        asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], 256, [%2];"
                     ::"r"(adst), "l"(denom + c0), "r"(bar)
                     : "memory");
        asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], 256, [%2];"
                     ::"r"(adst + 256u), "l"(denom + K_pad + c0), "r"(bar)
                     : "memory");
        asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], 128, [%2];"
                     ::"r"(adst + 512u), "l"(zv + c0), "r"(bar)
                     : "memory");
    };
    if (lane == 0)
        for (uint32_t t = 0; t + 2 < S && t < ntiles; ++t) load(t);
    const uint32_t v = row_begin + r0 + lane;
    const bool live = r0 + lane < rows;
    float* l8row = l8 + static_cast<size_t>(v) * l8_stride;
    float run = 0.0f;
    for (uint32_t t = 0; t < ntiles; ++t) {
        const uint32_t st = t % S, c0 = t * 32u;
        if (lane == 0 && t + S - 2 < ntiles) {
            // stage of tile t - 2: its tensor store must have finished reading shared memory
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            load(t + S - 2);
        }
        mbar_wait_parity(bars + st * 8u, (t / S) & 1u);
        uint32_t* tile = reinterpret_cast<uint32_t*>(tiles + st * kPhiTileBytes) + lane * 32u;
        const double* den = reinterpret_cast<const double*>(aux + st * kPhiAuxBytes);
        const double* rcp = den + 32;
        const float* zt = reinterpret_cast<const float*>(aux + st * kPhiAuxBytes + 512u);
        // All eight quads are loaded before any is written back, so their quotients are
        // independent work (the per-quad load -> divide -> store order serialises them).
        uint4 cnt[8];
        float4 bh[8];
#pragma unroll
        for (uint32_t j = 0; j < 8; ++j) {
            cnt[j] = *reinterpret_cast<const uint4*>(tile + ((j ^ (lane & 7u)) << 2));
            bh[j] = *reinterpret_cast<const float4*>(zt + j * 4);
        }
#pragma unroll
        for (uint32_t j = 0; j < 8; ++j) {
            const double* d = den + j * 4;
            const double* r = rcp + j * 4;
            if (cnt[j].x) bh[j].x = phi_quotient(__dadd_rn(static_cast<double>(cnt[j].x), beta), d[0], r[0]);
            if (cnt[j].y) bh[j].y = phi_quotient(__dadd_rn(static_cast<double>(cnt[j].y), beta), d[1], r[1]);
            if (cnt[j].z) bh[j].z = phi_quotient(__dadd_rn(static_cast<double>(cnt[j].z), beta), d[2], r[2]);
            if (cnt[j].w) bh[j].w = phi_quotient(__dadd_rn(static_cast<double>(cnt[j].w), beta), d[3], r[3]);
        }
        float l8v[4];
#pragma unroll
        for (uint32_t j = 0; j < 8; ++j) {
            run = __fadd_rn(run, bh[j].x);  // WaryTree::build's sequential chain (see phi_kernel)
            run = __fadd_rn(run, bh[j].y);
            run = __fadd_rn(run, bh[j].z);
            run = __fadd_rn(run, bh[j].w);
            *reinterpret_cast<float4*>(tile + ((j ^ (lane & 7u)) << 2)) = bh[j];
            if (j & 1u) l8v[j >> 1] = run;
        }
        if (live) *reinterpret_cast<float4*>(l8row + c0 / kLeaf) = make_float4(l8v[0], l8v[1], l8v[2], l8v[3]);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> TMA store
        __syncwarp();
        if (lane == 0) {
            asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
                         ::"l"(reinterpret_cast<uint64_t>(&t_phi)), "r"(c0), "r"(r0),
                         "r"(static_cast<uint32_t>(__cvta_generic_to_shared(tiles + st * kPhiTileBytes)))
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    if (live) {
        for (uint32_t j = K_pad / kLeaf; j < l8_stride; ++j) l8row[j] = run;
        q[v] = __fmul_rn(falpha, run);  // trainer.cpp:245
    }
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link dependency).
static cudaError_t encode_tile_map(CUtensorMap* m, CUtensorMapDataType type, void* base, uint32_t cols,
                                   uint32_t rows) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult qr{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr) != cudaSuccess ||
            qr != cudaDriverEntryPointSuccess || !fn)
            return cudaErrorNotSupported;
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    const cuuint64_t dims[2] = {cols, rows};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * 4u};
    const cuuint32_t box[2] = {32u, 32u};
    const cuuint32_t estr[2] = {1u, 1u};
    const CUresult r = encode(m, type, 2, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <int S, int W>
cudaError_t launch_phi_tma_t(const uint32_t* B, const double* denom, const float* zv, float* bhat, float* l8,
                             float* q, uint32_t row_begin, uint32_t row_end, uint32_t K_pad, uint32_t l8_stride,
                             double beta, float falpha, cudaStream_t s) {
    const uint32_t rows = row_end - row_begin;
    CUtensorMap tc, tp;
    const size_t off = static_cast<size_t>(row_begin) * K_pad;
    if (const cudaError_t e = encode_tile_map(&tc, CU_TENSOR_MAP_DATA_TYPE_UINT32, const_cast<uint32_t*>(B) + off,
                                              K_pad, rows);
        e != cudaSuccess)
        return e;
    if (const cudaError_t e = encode_tile_map(&tp, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, bhat + off, K_pad, rows);
        e != cudaSuccess)
        return e;
    constexpr size_t smem = phi_tma_smem_bytes<S, W>();
    if (const cudaError_t e = cudaFuncSetAttribute(phi_tma_kernel<S, W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   static_cast<int>(smem));
        e != cudaSuccess)
        return e;
    const uint32_t groups = (rows + 31u) / 32u;
    phi_tma_kernel<S, W><<<(groups + W - 1) / W, W * 32, smem, s>>>(tc, tp, denom, zv, l8, q, row_begin, rows, K_pad,
                                                                   l8_stride, beta, falpha);
    return cudaGetLastError();
}

template <int C, int S>
cudaError_t launch_phi_t(const uint32_t* B, const double* denom, const float* zv, float* bhat,
                         float* l8, float* q, uint32_t row_begin, uint32_t row_end, uint32_t K_pad,
                         uint32_t l8_stride, double beta, float falpha, cudaStream_t s) {
    constexpr size_t smem = phi_smem_bytes<C, S>();
    // Per launch: the opt-in is per device context (a process-wide flag would miss a second GPU).
    if (const cudaError_t e = cudaFuncSetAttribute(phi_kernel<C, S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   static_cast<int>(smem));
        e != cudaSuccess)
        return e;
    const uint32_t blocks = (row_end - row_begin + kPhiRows - 1) / kPhiRows;
    phi_kernel<C, S><<<blocks, kPhiRows, smem, s>>>(B, denom, zv, bhat, l8, q, row_begin, row_end, K_pad,
                                                    l8_stride, beta, falpha);
    return cudaGetLastError();
}

cudaError_t launch_phi(const uint32_t* B, const double* denom, const float* zv, float* bhat,
                       float* l8, float* q, uint32_t row_begin, uint32_t row_end,
                       uint32_t K, uint32_t K_pad, uint32_t l8_stride, double beta, float falpha,
                       cudaStream_t s) {
    (void)K;  // columns >= K are zero counts with zv = 0 (see above)
    if (row_end <= row_begin) return cudaSuccess;
    if (K_pad % 32) return cudaErrorInvalidValue;
    const char* e = std::getenv("SLDA_PHI_SHAPE");  // read per launch (tests switch it per engine)
    const std::string v = e ? e : "";
    // K_pad > 32768: the TMA warp-per-32-rows kernel (C5 K=50K phi alone 10.5 -> 9.4 ms; at K=10K
    // it is slower, 3.3 vs 2.9 ms: DESIGN.md §6).  SLDA_PHI_SHAPE=tma forces it (tests).
    if (v == "tma" || ((v.empty() || v == "default") && K_pad > 32768))
        return launch_phi_tma_t<3, 4>(B, denom, zv, bhat, l8, q, row_begin, row_end, K_pad, l8_stride, beta, falpha, s);
    int shape = v == "16x8" ? 1 : v == "32x3" ? 2 : v == "64x2" ? 3 : v == "64x3" ? 4 : v == "32x4" ? 5 : 0;
    // Tile columns x pipeline stages, phi alone (ms, C3 / C5 K=50K): 16x8 4.91 / 17.9,
    // 32x3 4.68 / 14.8, 32x4 4.10 / 15.7, 32x6 5.88 / 16.2.
    if (shape == 0) {
        // Uniform row blocks, so the last partial wave is pure tail: between 32 x 4 (fastest per
        // wave) and 32 x 3 (6 instead of 5 CTAs per SM) take the one whose last wave is fuller
        // (C3, 2204 blocks: 2.98 vs 2.48 waves -> 32 x 4, 4.10 vs 4.68 ms; C5 K=50K, 1563
        // blocks: 2.11 vs 1.76 waves -> 32 x 3, 14.8 vs 15.8 ms).
        static int slots4 = 0, slots3 = 0;
        if (!slots4) {
            int dev = 0, sms = 0, n4 = 0, n3 = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            cudaFuncSetAttribute(phi_kernel<32, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(phi_smem_bytes<32, 4>()));
            cudaFuncSetAttribute(phi_kernel<32, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(phi_smem_bytes<32, 3>()));
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n4, phi_kernel<32, 4>, kPhiRows, phi_smem_bytes<32, 4>());
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n3, phi_kernel<32, 3>, kPhiRows, phi_smem_bytes<32, 3>());
            slots4 = n4 * sms > 0 ? n4 * sms : 1;
            slots3 = n3 * sms > 0 ? n3 * sms : 1;
        }
        const double blocks = std::ceil((row_end - row_begin) / static_cast<double>(kPhiRows));
        const double w4 = blocks / slots4, w3 = blocks / slots3;
        const double fill4 = w4 / std::ceil(w4), fill3 = w3 / std::ceil(w3);
        shape = fill3 > fill4 + 0.05 ? 2 : 0;
    }
    switch (shape) {
        case 1: return launch_phi_t<16, 8>(B, denom, zv, bhat, l8, q, row_begin, row_end, K_pad, l8_stride, beta, falpha, s);
        case 2: return launch_phi_t<32, 3>(B, denom, zv, bhat, l8, q, row_begin, row_end, K_pad, l8_stride, beta, falpha, s);
        case 3: return launch_phi_t<64, 2>(B, denom, zv, bhat, l8, q, row_begin, row_end, K_pad, l8_stride, beta, falpha, s);
        case 4: return launch_phi_t<64, 3>(B, denom, zv, bhat, l8, q, row_begin, row_end, K_pad, l8_stride, beta, falpha, s);
        default: break;
    }
    return launch_phi_t<32, 4>(B, denom, zv, bhat, l8, q, row_begin, row_end, K_pad, l8_stride, beta, falpha, s);
}

// The L4 level on demand (slda_get_tree_prefix): thread per row, the same sequential f32 chain
// over the stored phi row as the phi kernel ran, so every value is the one WaryTree::build makes.
__global__ void l4_kernel(const float* __restrict__ bhat, uint32_t rows, uint32_t K_pad, float* __restrict__ l4) {
    const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= rows) return;
    const float4* src = reinterpret_cast<const float4*>(bhat + static_cast<size_t>(v) * K_pad);
    float4* dst = reinterpret_cast<float4*>(l4 + static_cast<size_t>(v) * K_pad);
    float run = 0.0f;
    for (uint32_t i = 0; i < K_pad / 4; ++i) {
        const float4 b = __ldg(src + i);
        float4 o;
        o.x = run = __fadd_rn(run, b.x);
        o.y = run = __fadd_rn(run, b.y);
        o.z = run = __fadd_rn(run, b.z);
        o.w = run = __fadd_rn(run, b.w);
        dst[i] = o;
    }
}

cudaError_t launch_l4(const float* bhat, uint32_t rows, uint32_t K_pad, float* l4, cudaStream_t s) {
    if (rows) l4_kernel<<<(rows + 127) / 128, 128, 0, s>>>(bhat, rows, K_pad, l4);
    return cudaGetLastError();
}

// ---- Peer-memory M-step exchange (world > 1; engine.cu m_step_peer) ---------------------------
// Every rank maps the other ranks' exchange buffers (CUDA IPC handles: NVLink peer memory on a
// multi-GPU node, the same HBM when ranks share one GPU).  C_wk is exchanged SPARSE: a rank's
// partial C_wk has at most T_rank non-zero cells, the reduced one at most min(V*K, T), against
// V*K dense cells (C3: 1.41G).  A row's non-zeros become u32 entries topic | count << 16 (counts
// above 65535 split into several entries, which the receivers add), indexed per row by
// {offset, n}.  Reduce-scatter: each rank adds the other ranks' entries of its word slice into
// its own B.  All-gather: each rank sparsifies its reduced slice and every rank adds the other
// slices' entries into its (zeroed) other rows -- after which every rank holds the full reduced
// C_wk and runs the ordinary colsum + phi over all rows locally.  Integer sums: bit-identical to
// one GPU at any rank count.

// All ranks increment rank 0's counter; each waits for the round's total.  System-scope fences
// publish this rank's prior writes (kernels earlier on the stream) before it arrives.
__global__ void peer_barrier_kernel(unsigned long long* counter, unsigned long long target) {
    __threadfence_system();
    atomicAdd_system(counter, 1ull);
    // A rank that died never arrives: give up after ~2 minutes (the kernel traps, the stream
    // reports an error) instead of spinning forever.
    const long long t0 = clock64();
    while (atomicAdd_system(counter, 0ull) < target) {
        __nanosleep(256);
        if (clock64() - t0 > 240'000'000'000LL) __trap();
    }
    __threadfence_system();
}

cudaError_t launch_peer_barrier(unsigned long long* counter, unsigned long long target, cudaStream_t s) {
    peer_barrier_kernel<<<1, 1, 0, s>>>(counter, target);
    return cudaGetLastError();
}

__device__ __forceinline__ uint32_t count_pieces(uint32_t c) { return (c + 65534u) / 65535u; }  // 0 for c == 0

// Warp per row of [row_lo, row_hi): pass 1 counts the row's entries, one atomic reserves them,
// pass 2 re-reads the row (L1/L2-hot) and writes them in topic order.  A reservation past
// `cap` (cannot happen with the engine's capacity bound) records an empty row and flags it.
__global__ void __launch_bounds__(256) sparsify_kernel(const uint32_t* __restrict__ B, uint32_t row_lo,
                                                       uint32_t row_hi, uint32_t K_pad, uint2* __restrict__ info,
                                                       uint32_t* __restrict__ entries, uint32_t* cursor, uint32_t cap,
                                                       uint32_t* overflow) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t nq = K_pad / 4u;
    for (uint32_t v = row_lo + (blockIdx.x * blockDim.x + threadIdx.x) / 32u; v < row_hi;
         v += gridDim.x * blockDim.x / 32u) {
        const uint4* row = reinterpret_cast<const uint4*>(B + static_cast<size_t>(v) * K_pad);
        uint32_t n = 0;
        for (uint32_t i = lane; i < nq; i += 32u) {
            const uint4 c = __ldg(row + i);
            n += count_pieces(c.x) + count_pieces(c.y) + count_pieces(c.z) + count_pieces(c.w);
        }
        n = __reduce_add_sync(0xffffffffu, n);
        uint32_t off = 0;
        if (lane == 0 && n) {
            off = atomicAdd(cursor, n);
            if (off + n > cap || off + n < off) {
                atomicOr(overflow, 1u);
                n = 0;
            }
        }
        off = __shfl_sync(0xffffffffu, off, 0);
        n = __shfl_sync(0xffffffffu, n, 0);
        if (lane == 0) info[v - row_lo] = make_uint2(off, n);
        if (n == 0) continue;
        for (uint32_t i0 = 0; i0 < nq; i0 += 32u) {
            const uint32_t i = i0 + lane;
            const uint4 c = i < nq ? __ldg(row + i) : make_uint4(0u, 0u, 0u, 0u);
            const uint32_t m = count_pieces(c.x) + count_pieces(c.y) + count_pieces(c.z) + count_pieces(c.w);
            uint32_t incl = m;
#pragma unroll
            for (uint32_t o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            uint32_t pos = off + incl - m;
            const uint32_t cs[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
            for (uint32_t j = 0; j < 4; ++j) {
                uint32_t left = cs[j];
                const uint32_t k = 4u * i + j;
                while (left) {
                    const uint32_t piece = left < 65535u ? left : 65535u;
                    entries[pos++] = k | (piece << 16);
                    left -= piece;
                }
            }
            off += __shfl_sync(0xffffffffu, incl, 31);
        }
    }
}

cudaError_t launch_sparsify(const uint32_t* B, uint32_t row_lo, uint32_t row_hi, uint32_t K_pad, uint2* info,
                            uint32_t* entries, uint32_t* cursor, uint32_t cap, uint32_t* overflow, cudaStream_t s) {
    if (row_hi <= row_lo) return cudaSuccess;
    const uint32_t rows = row_hi - row_lo;
    const uint32_t blocks = rows / 8u + 1u < 148u * 16u ? rows / 8u + 1u : 148u * 16u;
    sparsify_kernel<<<blocks, 256, 0, s>>>(B, row_lo, row_hi, K_pad, info, entries, cursor, cap, overflow);
    return cudaGetLastError();
}

// Warp per row of [row_lo, row_hi), skipping [skip_lo, skip_hi): adds the row's entries from
// its sources into B.  Reduce-scatter (per_slice == 0): every source, row index v - base.
// All-gather (per_slice > 0): the one source owning the row, src[v / per_slice], row index
// v - its base.  `bytes` tallies what was read from the sources (entries + row index).
__global__ void __launch_bounds__(256) gather_add_kernel(PeerSparse ps, uint32_t row_lo, uint32_t row_hi,
                                                         uint32_t skip_lo, uint32_t skip_hi, uint32_t per_slice,
                                                         uint32_t* __restrict__ B, uint32_t K_pad,
                                                         unsigned long long* bytes) {
    const uint32_t lane = threadIdx.x & 31u;
    unsigned long long got = 0;
    for (uint32_t v = row_lo + (blockIdx.x * blockDim.x + threadIdx.x) / 32u; v < row_hi;
         v += gridDim.x * blockDim.x / 32u) {
        if (v >= skip_lo && v < skip_hi) continue;
        uint32_t* brow = B + static_cast<size_t>(v) * K_pad;
        const uint32_t s0 = per_slice ? v / per_slice : 0u, s1 = per_slice ? s0 + 1u : ps.n;
        for (uint32_t si = s0; si < s1; ++si) {
            const SparseRows src = ps.src[si];
            if (!src.info) continue;
            const uint2 in = src.info[v - src.base];
            for (uint32_t e = lane; e < in.y; e += 32u) {
                const uint32_t x = src.entries[in.x + e];
                atomicAdd(brow + (x & 0xFFFFu), x >> 16);
            }
            if (lane == 0) got += 8ull + 4ull * in.y;
        }
    }
    if (lane == 0 && got) atomicAdd(bytes, got);
}

cudaError_t launch_gather_add(const PeerSparse& ps, uint32_t row_lo, uint32_t row_hi, uint32_t skip_lo,
                              uint32_t skip_hi, uint32_t per_slice, uint32_t* B, uint32_t K_pad,
                              unsigned long long* bytes, cudaStream_t s) {
    if (row_hi <= row_lo) return cudaSuccess;
    const uint32_t rows = row_hi - row_lo;
    const uint32_t blocks = rows / 8u + 1u < 148u * 16u ? rows / 8u + 1u : 148u * 16u;
    gather_add_kernel<<<blocks, 256, 0, s>>>(ps, row_lo, row_hi, skip_lo, skip_hi, per_slice, B, K_pad, bytes);
    return cudaGetLastError();
}

}  // namespace slda
