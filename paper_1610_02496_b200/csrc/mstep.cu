// mstep.cu -- K5/K6: column sums, phi and the tree prefix (the M-step) on sm_100a.
//
// Reference paths are relative to /root/reference/proj.  See DESIGN.md §4.
#include "common.cuh"
#include "kernels.hpp"

namespace slda {

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

template <bool kMirror>
__global__ void __launch_bounds__(kPhiRows, 4) phi_kernel(const uint32_t* __restrict__ B,
                                                        const double* __restrict__ denom,
                                                        const float* __restrict__ zv,
                                                        float* __restrict__ bhat, float* __restrict__ l4,
                                                        float* __restrict__ l8, float* __restrict__ q,
                                                        uint32_t row_begin, uint32_t row_end, uint32_t K,
                                                        uint32_t K_pad, uint32_t l8_stride, double beta,
                                                        float falpha, PeerMirror mirror) {
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
            if (kMirror)
                for (uint32_t p = 0; p < mirror.n; ++p)
                    *reinterpret_cast<float4*>(mirror.l8[p] + static_cast<size_t>(v) * l8_stride + c0 / kLeaf) = l8v;
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
                if (kMirror) {  // the all-gather, fused: the same values into every peer's replica
                    for (uint32_t p = 0; p < mirror.n; ++p) {
                        mirror.bhat[p][o] = t_bh[rr][cc];
                        mirror.l4[p][o] = t_l4[rr][cc];
                    }
                }
            }
        }
        __syncthreads();  // the next tile store overwrites t_in (== t_bh)
    }
    if (v < row_end) {
        for (uint32_t j = K_pad / kLeaf; j < l8_stride; ++j) l8[static_cast<size_t>(v) * l8_stride + j] = run;
        q[v] = __fmul_rn(falpha, run);  // trainer.cpp:245
        if (kMirror) {
            for (uint32_t p = 0; p < mirror.n; ++p) {
                for (uint32_t j = K_pad / kLeaf; j < l8_stride; ++j)
                    mirror.l8[p][static_cast<size_t>(v) * l8_stride + j] = run;
                mirror.q[p][v] = __fmul_rn(falpha, run);
            }
        }
    }
}

cudaError_t launch_phi(const uint32_t* B, const double* denom, const float* zv, float* bhat,
                       float* l4, float* l8, float* q, uint32_t row_begin, uint32_t row_end,
                       uint32_t K, uint32_t K_pad, uint32_t l8_stride, double beta, float falpha,
                       cudaStream_t s, const PeerMirror* mirror) {
    if (row_end <= row_begin) return cudaSuccess;
    const uint32_t blocks = (row_end - row_begin + kPhiRows - 1) / kPhiRows;
    if (mirror && mirror->n > 0)
        phi_kernel<true><<<blocks, kPhiRows, 0, s>>>(B, denom, zv, bhat, l4, l8, q, row_begin, row_end, K, K_pad,
                                                     l8_stride, beta, falpha, *mirror);
    else
        phi_kernel<false><<<blocks, kPhiRows, 0, s>>>(B, denom, zv, bhat, l4, l8, q, row_begin, row_end, K,
                                                      K_pad, l8_stride, beta, falpha, PeerMirror{});
    return cudaGetLastError();
}

// ---- Peer-memory M-step exchange (world > 1 without NCCL; engine.cu m_step_peer) -------------
// Every rank maps every other rank's buffers (CUDA IPC handles, NVLink peer memory on a multi-GPU
// node, the same HBM when the ranks share one GPU) and the collectives become parts of the
// kernels that need them: the reduce-scatter of C_wk is the colsum kernel reading its word
// slice from all ranks' partial C_wk; the all-reduce of C_k is the denominator kernel summing
// the ranks' column-sum partials; the all-gather of phi / L4 / L8 / Q is the phi kernel's
// epilogue storing its slice into every replica (above).  Ranks meet at device-side barriers.

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

// Reduce-scatter fused into colsum: own slice rows of every rank's partial C_wk are summed
// (integers: order-free, bit-identical to NCCL's), written back into this rank's B (its slice
// of the reduced C_wk) and column-summed into this rank's C_k partial.
__global__ void __launch_bounds__(256) peer_colsum_kernel(PeerCounts pc, uint32_t* __restrict__ B, uint32_t row_begin,
                                                          uint32_t row_end, uint32_t cols4, uint32_t rows_per_chunk,
                                                          unsigned long long* __restrict__ colsum) {
    __shared__ unsigned long long s_acc[256][4];
    const uint32_t c4 = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t r0 = row_begin + blockIdx.y * rows_per_chunk;
    const uint32_t r1 = min(row_end, r0 + rows_per_chunk);
    unsigned long long acc[4] = {0, 0, 0, 0};
    if (c4 < cols4) {
        for (uint32_t r = r0 + threadIdx.y; r < r1; r += blockDim.y) {
            const size_t o = static_cast<size_t>(r) * cols4 + c4;
            uint4 t = make_uint4(0u, 0u, 0u, 0u);
            for (uint32_t p = 0; p < pc.n; ++p) {
                const uint4 b = reinterpret_cast<const uint4*>(pc.B[p])[o];
                t.x += b.x; t.y += b.y; t.z += b.z; t.w += b.w;
            }
            reinterpret_cast<uint4*>(B)[o] = t;
            acc[0] += t.x; acc[1] += t.y; acc[2] += t.z; acc[3] += t.w;
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

cudaError_t launch_peer_colsum(const PeerCounts& pc, uint32_t* B, uint32_t row_begin, uint32_t row_end,
                               uint32_t K_pad, unsigned long long* colsum, cudaStream_t s) {
    if (row_end <= row_begin) return cudaSuccess;
    const uint32_t cols4 = K_pad / 4;
    const uint32_t bx = cols4 < 256 ? cols4 : 256;
    const uint32_t by = 256 / bx;
    const uint32_t gx = (cols4 + bx - 1) / bx;
    const uint32_t rows = row_end - row_begin;
    uint32_t gy = (148u * 8u + gx - 1) / gx;
    uint32_t per = (rows + gy - 1) / gy;
    if (per < by) per = by;
    gy = (rows + per - 1) / per;
    peer_colsum_kernel<<<dim3(gx, gy), dim3(bx, by), 0, s>>>(pc, B, row_begin, row_end, cols4, per, colsum);
    return cudaGetLastError();
}

// All-reduce of C_k fused into the denominator: sum of the ranks' partials (u64, order-free).
__global__ void peer_total_kernel(PeerColsums pc, uint32_t K_pad, unsigned long long* total) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= K_pad) return;
    unsigned long long t = 0;
    for (uint32_t p = 0; p < pc.n; ++p) t += pc.c[p][k];
    total[k] = t;
}

cudaError_t launch_peer_total(const PeerColsums& pc, uint32_t K_pad, unsigned long long* total, cudaStream_t s) {
    peer_total_kernel<<<(K_pad + 255) / 256, 256, 0, s>>>(pc, K_pad, total);
    return cudaGetLastError();
}

}  // namespace slda
