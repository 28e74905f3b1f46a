// heldout.cu -- heldout_ll (eval.cpp:49-133) on device.
//
// One CTA per held-out document: the estimation half's topics live in shared
// memory; each burn-in sweep recounts them (segmented_count, counts.cpp:65-94,
// as a shared-memory bitonic sort + run-length) and resamples every token with
// the training sampler's exact f32 arithmetic (sample_token, sampler.hpp:183-204)
// against the frozen phi / L4 / Q.  The log-mix of each evaluation token is
// written out and summed on the host in the reference's order.
#include "common.cuh"
#include "heldout.hpp"
#include "row_format.cuh"

namespace slda {

namespace {

__device__ void block_sort(uint32_t* keys, uint32_t N) {
    for (uint32_t k = 2; k <= N; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) {
                const uint32_t ixj = i ^ j;
                if (ixj > i) {
                    const uint32_t x = keys[i], y = keys[ixj];
                    const bool up = (i & k) == 0;
                    if ((x > y) == up) {
                        keys[i] = y;
                        keys[ixj] = x;
                    }
                }
            }
            __syncthreads();
        }
    }
}

// segmented_count of topics[0..n) into ascending (rt, rc); returns nnz.
__device__ uint32_t block_segmented_count(const uint32_t* topics, uint32_t n, uint32_t N, uint32_t* keys,
                                          uint32_t* starts, uint32_t* rt, uint32_t* rc, uint32_t* s_nnz) {
    for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) keys[i] = i < n ? topics[i] : 0xFFFFFFFFu;
    __syncthreads();
    block_sort(keys, N);
    if (threadIdx.x < 32) {
        const uint32_t lane = threadIdx.x;
        uint32_t nnz = 0;
        for (uint32_t base = 0; base < n; base += 32) {
            const uint32_t i = base + lane;
            const bool start = i < n && (i == 0 || keys[i] != keys[i - 1]);
            const uint32_t ballot = __ballot_sync(0xffffffffu, start);
            if (start) starts[nnz + __popc(ballot & ((1u << lane) - 1u))] = i;
            nnz += __popc(ballot);
        }
        if (lane == 0) *s_nnz = nnz;
    }
    __syncthreads();
    const uint32_t nnz = *s_nnz;
    for (uint32_t r = threadIdx.x; r < nnz; r += blockDim.x) {
        const uint32_t st = starts[r];
        const uint32_t en = r + 1 < nnz ? starts[r + 1] : n;
        rt[r] = keys[st];
        rc[r] = en - st;
    }
    __syncthreads();
    return nnz;
}

}  // namespace

__global__ void __launch_bounds__(256) heldout_kernel(HeldoutArgs a) {
    extern __shared__ __align__(16) uint32_t sm[];
    __shared__ uint32_t s_nnz;
    const uint32_t d = blockIdx.x;
    const uint64_t b0 = a.est_off[d], n64 = a.est_off[d + 1] - b0;
    const uint32_t n = static_cast<uint32_t>(n64);
    const uint64_t e0 = a.evl_off[d], ne = a.evl_off[d + 1] - e0;
    if (n == 0) {  // eval.cpp:85: no estimation tokens, doc contributes 0
        for (uint64_t j = threadIdx.x; j < ne; j += blockDim.x) a.ll_out[e0 + j] = 0.0;
        return;
    }
    uint32_t N = 1;
    while (N < n) N <<= 1;
    uint32_t* topics = sm;        // n
    uint32_t* keys = sm + a.cap;  // N
    uint32_t* starts = keys + a.cap;
    uint32_t* rt = starts + a.cap;  // nnz <= n
    uint32_t* rc = rt + a.cap;

    for (uint32_t j = threadIdx.x; j < n; j += blockDim.x)
        topics[j] = uniform_topic(a.seed, kHeldoutInitStream, b0 + j, a.K);
    __syncthreads();

    for (uint32_t sweep = 0; sweep < a.burn_in; ++sweep) {
        const uint32_t nnz = block_segmented_count(topics, n, N, keys, starts, rt, rc, &s_nnz);
        for (uint32_t j = threadIdx.x; j < n; j += blockDim.x) {
            const uint32_t v = a.est_word[b0 + j];
            const float* brow = a.bhat + static_cast<size_t>(v) * a.K_pad;
            float ub, up;
            draw2_f32(a.seed, kHeldoutSweepBase + sweep, b0 + j, ub, up);
            float s = 0.0f;
            for (uint32_t i = 0; i < nnz; ++i)
                s = __fadd_rn(s, __fmul_rn(__uint2float_rn(rc[i]), __ldg(brow + rt[i])));
            const float qv = __ldg(a.q + v);
            uint32_t topic;
            if (ub < __fdiv_rn(s, __fadd_rn(s, qv))) {
                const float x = __fmul_rn(up, s);
                float run = 0.0f;
                topic = rt[nnz - 1];
                for (uint32_t i = 0; i < nnz; ++i) {
                    run = __fadd_rn(run, __fmul_rn(__uint2float_rn(rc[i]), __ldg(brow + rt[i])));
                    if (run >= x) {
                        topic = rt[i];
                        break;
                    }
                }
            } else {
                const float* l8row = a.l8 + static_cast<size_t>(v) * a.l8_stride;
                const float total = __ldg(l8row + a.n_l8 - 1);  // L8's last entry is the row total
                float x = __fmul_rn(up, total);
                if (!(x <= total)) x = total;
                // lower_bound over L4 (== WaryTree::sample): the L8 level, then the block's 8
                // prefixes continued from L8 over the phi row (row_format.cuh tree_search).
                topic = tree_search<true>(x, l8row, a.n_l8, brow);
                if (topic >= a.K) topic = a.K - 1;
            }
            keys[j] = topic;  // keys is free once the counts are built
        }
        __syncthreads();
        for (uint32_t j = threadIdx.x; j < n; j += blockDim.x) topics[j] = keys[j];
        __syncthreads();
    }
    const uint32_t nnz = block_segmented_count(topics, n, N, keys, starts, rt, rc, &s_nnz);
    const double denom = __dadd_rn(static_cast<double>(n), __dmul_rn(static_cast<double>(a.K), a.alpha));
    for (uint64_t j = threadIdx.x; j < ne; j += blockDim.x) {
        const uint32_t v = a.evl_word[e0 + j];
        const float* brow = a.bhat + static_cast<size_t>(v) * a.K_pad;
        double mass = __dmul_rn(a.alpha, a.row_mass[v]);
        for (uint32_t i = 0; i < nnz; ++i)
            mass = __dadd_rn(mass, __dmul_rn(static_cast<double>(rc[i]), static_cast<double>(__ldg(brow + rt[i]))));
        a.ll_out[e0 + j] = log(__ddiv_rn(mass, denom));
    }
}

// eval.cpp:61-69: f64 sequential row sums of phi.
__global__ void row_mass_kernel(const float* bhat, uint32_t V, uint32_t K, uint32_t K_pad, double* out) {
    const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= V) return;
    const float* row = bhat + static_cast<size_t>(v) * K_pad;
    double s = 0.0;
    for (uint32_t k = 0; k < K; ++k) s = __dadd_rn(s, static_cast<double>(row[k]));
    out[v] = s;
}

cudaError_t launch_heldout(const HeldoutArgs& a, uint32_t num_docs, uint32_t V, uint32_t K,
                           uint32_t K_pad, double* row_mass, cudaStream_t s) {
    row_mass_kernel<<<(V + 127) / 128, 128, 0, s>>>(a.bhat, V, K, K_pad, row_mass);
    if (num_docs == 0) return cudaGetLastError();
    const size_t smem = sizeof(uint32_t) * 5 * static_cast<size_t>(a.cap);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(heldout_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
    }
    heldout_kernel<<<num_docs, 256, smem, s>>>(a);
    return cudaGetLastError();
}

}  // namespace slda
