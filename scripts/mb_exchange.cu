// mb_exchange.cu -- the sparse C_wk exchange kernels (mstep.cu sparsify_kernel /
// gather_add_kernel) on one GPU at C3's shape, for timing and ncu: a V x K_pad C_wk with a
// given number of non-zero cells, sparsified (all rows), then gathered back (add) into a
// zeroed matrix and checked.  Not product code.  Build: see scripts/gpu_mbx.sh.
//   ./mb_exchange V K nnz reps
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "kernels.hpp"

#define CK(x)                                                                      \
    do {                                                                           \
        cudaError_t e_ = (x);                                                      \
        if (e_ != cudaSuccess) {                                                   \
            std::fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));          \
            std::exit(1);                                                          \
        }                                                                          \
    } while (0)

int main(int argc, char** argv) {
    const uint32_t V = argc > 1 ? std::atoi(argv[1]) : 141000;
    const uint32_t K = argc > 2 ? std::atoi(argv[2]) : 10000;
    const uint64_t nnz = argc > 3 ? std::atoll(argv[3]) : 110000000ull;
    const int reps = argc > 4 ? std::atoi(argv[4]) : 5;
    const uint32_t K_pad = (K + 31) / 32 * 32;
    const size_t cells = static_cast<size_t>(V) * K_pad;
    std::vector<uint32_t> h(cells, 0);
    std::mt19937_64 rng(7);
    for (uint64_t i = 0; i < nnz; ++i) {
        const uint64_t r = rng();
        const size_t c = (r % V) * K_pad + (r >> 32) % K;
        h[c] += 1 + static_cast<uint32_t>((r >> 20) % 4);
    }
    uint64_t real_nnz = 0, total = 0;
    for (uint32_t x : h) {
        real_nnz += x != 0;
        total += x;
    }
    uint32_t *B, *B2, *ent, *cnt;
    uint2* info;
    unsigned long long* bytes;
    CK(cudaMalloc(&B, cells * 4));
    CK(cudaMalloc(&B2, cells * 4));
    CK(cudaMalloc(&info, static_cast<size_t>(V) * 8));
    const uint64_t cap = real_nnz + total / 65535 + 64;
    CK(cudaMalloc(&ent, cap * 4));
    CK(cudaMalloc(&cnt, 16));
    CK(cudaMalloc(&bytes, 8));
    CK(cudaMemcpy(B, h.data(), cells * 4, cudaMemcpyHostToDevice));
    cudaEvent_t a, b, c;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(cudaEventCreate(&c));
    slda::PeerSparse ps{};
    ps.src[0] = {info, ent, 0u};
    ps.n = 1;
    float t_sp = 0, t_ga = 0;
    for (int r = 0; r < reps; ++r) {
        CK(cudaMemset(cnt, 0, 16));
        CK(cudaMemset(B2, 0, cells * 4));
        CK(cudaMemset(bytes, 0, 8));
        CK(cudaEventRecord(a));
        CK(slda::launch_sparsify(B, 0, V, K_pad, info, ent, cnt, static_cast<uint32_t>(cap), cnt + 2, 0));
        CK(cudaEventRecord(b));
        CK(slda::launch_gather_add(ps, 0, V, V, V, 0, B2, K_pad, bytes, 0));
        CK(cudaEventRecord(c));
        CK(cudaEventSynchronize(c));
        float x, y;
        CK(cudaEventElapsedTime(&x, a, b));
        CK(cudaEventElapsedTime(&y, b, c));
        if (r) t_sp += x, t_ga += y;  // first repetition is warm-up
    }
    std::vector<uint32_t> back(cells);
    CK(cudaMemcpy(back.data(), B2, cells * 4, cudaMemcpyDeviceToHost));
    uint32_t cur[4];
    unsigned long long gb = 0;
    CK(cudaMemcpy(cur, cnt, 16, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&gb, bytes, 8, cudaMemcpyDeviceToHost));
    const bool ok = back == h && cur[2] == 0;
    const int n = reps > 1 ? reps - 1 : 1;
    t_sp /= n;
    t_ga /= n;
    // Algorithmic bytes: sparsify reads the dense matrix and writes the entries + row index;
    // gather reads the entries + index and read-modify-writes the touched cells (4 B each way).
    const double sp_bytes = cells * 4.0 + cur[0] * 4.0 + V * 8.0;
    const double ga_bytes = cur[0] * 4.0 + V * 8.0 + real_nnz * 8.0;
    std::printf("{\"V\": %u, \"K\": %u, \"nnz\": %llu, \"entries\": %u, \"ok\": %s, \"sparsify_ms\": %.3f, "
                "\"sparsify_gbs\": %.1f, \"gather_ms\": %.3f, \"gather_gbs\": %.1f, \"gather_bytes_read\": %llu}\n",
                V, K, static_cast<unsigned long long>(real_nnz), cur[0], ok ? "true" : "false", t_sp,
                sp_bytes / t_sp / 1e6, t_ga, ga_bytes / t_ga / 1e6, gb);
    return ok ? 0 : 1;
}
