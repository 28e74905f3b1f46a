// Microbenchmark (not product code): throughput of reading many short random rows,
// the sampler's dominant access pattern (C_dk rows, 32-byte aligned, `sect` sectors).
//   lane256 : each lane reads its own row, 256-bit loads, 4 in flight
//   coop    : the warp reads its 32 rows cooperatively (lane l -> sector l % sect of
//             row l / sect), i.e. coalesced 256-bit loads, then shuffles nothing (sum)
//   bulk    : each lane issues one cp.async.bulk of its row into shared memory
//             (TMA engine), the warp waits on an mbarrier, then reads it back
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/mb_rows scripts/microbench_rows.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

struct Sector { uint4 lo, hi; };

__device__ __forceinline__ Sector ld256(const void* p) {
    Sector s;
    asm("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=r"(s.lo.x), "=r"(s.lo.y), "=r"(s.lo.z), "=r"(s.lo.w), "=r"(s.hi.x), "=r"(s.hi.y), "=r"(s.hi.z), "=r"(s.hi.w)
        : "l"(p));
    return s;
}

__device__ __forceinline__ uint32_t hash(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

__device__ __forceinline__ uint64_t row_start(uint32_t tid, int r, uint64_t nsect, int sect) {
    return hash(tid * 977u + r * 131071u) % (uint32_t)(nsect - sect);
}

__global__ void lane256(const uint4* __restrict__ a, uint64_t nsect, int rpt, int sect, uint32_t* out) {
    uint32_t acc = 0;
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    for (int r = 0; r < rpt; ++r) {
        const uint4* row = a + 2 * row_start(tid, r, nsect, sect);
        for (int s = 0; s < sect; s += 4) {
            Sector q[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) q[u] = s + u < sect ? ld256(row + 2 * (s + u)) : Sector{};
#pragma unroll
            for (int u = 0; u < 4; ++u) acc += q[u].lo.x ^ q[u].hi.w ^ q[u].lo.z;
        }
    }
    if (acc == 0x12345678u) out[0] = acc;
}

__global__ void coop(const uint4* __restrict__ a, uint64_t nsect, int rpt, int sect, uint32_t* out) {
    uint32_t acc = 0;
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t lane = threadIdx.x & 31;
    for (int r = 0; r < rpt; ++r) {
        const uint64_t mine = row_start(tid, r, nsect, sect);
        // rows_per_inst rows per instruction, lanes cover their sectors
        const int rpi = 32 / sect;
        for (int base = 0; base < 32; base += rpi) {
            const int rr = base + (int)lane / sect;
            const int ss = lane % sect;
            const uint64_t st = __shfl_sync(0xffffffffu, mine, rr < 32 ? rr : 31);
            if (rr < 32 && (int)lane < rpi * sect) {
                const Sector q = ld256(a + 2 * (st + ss));
                acc += q.lo.x ^ q.hi.w ^ q.lo.z;
            }
        }
    }
    if (acc == 0x12345678u) out[0] = acc;
}

__global__ void bulk(const uint4* __restrict__ a, uint64_t nsect, int rpt, int sect, uint32_t* out) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) unsigned long long bar[8];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char* buf = smem + (size_t)threadIdx.x * sect * 32;
    const uint32_t bar_addr = (uint32_t)__cvta_generic_to_shared(&bar[warp]);
    if (lane == 0) asm volatile("mbarrier.init.shared.b64 [%0], %1;" :: "r"(bar_addr), "r"(32));
    __syncwarp();
    uint32_t acc = 0, phase = 0;
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t bytes = sect * 32;
    for (int r = 0; r < rpt; ++r) {
        const uint4* row = a + 2 * row_start(tid, r, nsect, sect);
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(buf);
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" :: "r"(bar_addr), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"(dst), "l"(row), "r"(bytes), "r"(bar_addr) : "memory");
        // wait for the phase
        asm volatile("{\n\t.reg .pred P1;\n\tWAIT:\n\t"
                     "mbarrier.try_wait.parity.shared.b64 P1, [%0], %1;\n\t"
                     "@!P1 bra WAIT;\n\t}" :: "r"(bar_addr), "r"(phase) : "memory");
        phase ^= 1;
        const uint4* s4 = reinterpret_cast<const uint4*>(buf);
        for (int q = 0; q < 2 * sect; ++q) { const uint4 v = s4[q]; acc += v.x ^ v.w; }
        __syncwarp();
    }
    if (acc == 0x12345678u) out[0] = acc;
}

typedef void (*Kern)(const uint4*, uint64_t, int, int, uint32_t*);

void run(const char* name, Kern k, const uint4* a, uint64_t nsect, int sect, uint32_t* out, int smem, int block = 256) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, block, smem);
    if (occ == 0) { printf("%s: occupancy 0\n", name); return; }
    const int grid = 148 * occ * 4;
    const int rpt = 32;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<<<grid, block, smem>>>(a, nsect, rpt, sect, out);
    cudaEventRecord(e0);
    k<<<grid, block, smem>>>(a, nsect, rpt, sect, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) { printf("%s: error %s\n", name, cudaGetErrorString(err)); return; }
    const double bytes = double(grid) * block * rpt * sect * 32.0;
    printf("%-8s sect/row=%2d smem=%3dKB occ=%d blk/SM : %7.1f GB/s\n", name, sect, smem / 1024, occ, bytes / ms / 1e6);
}

int main() {
    const uint64_t bytes = 3ull << 30;  // 3 GB, like C_dk at C3
    uint4* a; uint32_t* out;
    cudaMalloc(&a, bytes); cudaMalloc(&out, 4);
    cudaMemset(a, 1, bytes);
    const uint64_t nsect = bytes / 32;
    if (getenv("MB_CEILING")) {  // the sampler's pattern: ~10-sector random rows, coalesced reads
        for (int sect : {4, 8, 10, 12, 16, 32}) run("coop", coop, a, nsect, sect, out, 0);
        return 0;
    }
    for (int sect : {4, 8, 16}) {
        for (int smem : {0, 48 * 1024}) run("lane256", lane256, a, nsect, sect, out, smem);
        for (int smem : {0, 48 * 1024}) run("coop", coop, a, nsect, sect, out, smem);
        run("bulk", bulk, a, nsect, sect, out, 256 * sect * 32);
        run("bulk128", bulk, a, nsect, sect, out, 128 * sect * 32, 128);
    }
    return 0;
}
