// engine.cu -- the C-ABI (include/saberlda.h) over the sm_100a kernels.
//
// One engine = one GPU = one document shard (the reference's chunk,
// PAPER.md:403, with chunk -> GPU).  The whole ESCA state lives in HBM:
//   tok   uint2[T]      execution order (word, doc length desc, doc, token_id):
//                       {row4[doc], slot}
//   z     u16[T]        topic per slot; slots are doc-grouped (slot == corpus
//                       position for a doc-sorted corpus)
//   A     u32[4*Q]      C_dk rows: [nnz-1 | entries topic | count << tbits | zero
//                       padding to a multiple of 8], 32-byte aligned at row4[d]
//   B     u32[V_pad][K_pad], bhat/L4 f32[V_pad][K_pad], L8 f32[V_pad][l8s] (every 8th prefix), Q f32[V_pad]
// Reference paths are relative to /root/reference/proj.
#include <algorithm>
#include <chrono>
#include <thread>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include <cub/cub.cuh>

#include "../../include/saberlda.h"
#include "common.cuh"
#include "heldout.hpp"
#include "kernels.hpp"

namespace {

thread_local std::string g_error;

struct SldaError : std::runtime_error {
    int code;
    SldaError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] void validation(const std::string& m) { throw SldaError(SLDA_ERR_VALIDATION, m); }

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw SldaError(SLDA_ERR_DEVICE, std::string(what) + ": " + cudaGetErrorString(e));
}
#define CK(x) cuda_check((x), #x)

template <class F>
int guarded(F&& f) {
    try {
        f();
        return SLDA_OK;
    } catch (const SldaError& e) {
        g_error = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_error = "host allocation failed";
        return SLDA_ERR_DEVICE;
    } catch (const std::exception& e) {
        g_error = e.what();
        return SLDA_ERR_DEVICE;
    }
}

// --------------------------------------------------------------- buffers --
// Setup scratch arena: one cudaMalloc for all of init_state's temporaries (a stack: a block
// released while on top is popped, others wait for the arena's end), instead of ~25
// cudaMalloc/cudaFree pairs of GB-sized buffers whose mapping/unmapping made setup time vary
// 0.36-0.57 s at C3.  Temporaries are the DevMem allocations without a byte tally.
struct Arena {
    char* base = nullptr;
    size_t cap = 0, top = 0;
    Arena* prev = nullptr;
    static Arena*& current() {
        static thread_local Arena* a = nullptr;
        return a;
    }
    explicit Arena(size_t bytes) {
        if (cudaMalloc(&base, bytes) == cudaSuccess) cap = bytes;
        else { base = nullptr; cudaGetLastError(); }  // no arena: plain allocations
        prev = current();
        current() = this;
    }
    ~Arena() {
        current() = prev;
        if (base) {
            if (deferred) *deferred = base;  // released by the engine's scratch thread
            else cudaFree(base);
        }
    }
    void** deferred = nullptr;
    Arena(const Arena&) = delete;
    Arena& operator=(const Arena&) = delete;
    void* take(size_t n) {
        const size_t a = (n + 255) & ~static_cast<size_t>(255);
        if (!base || top + a > cap) return nullptr;
        void* p = base + top;
        top += a;
        return p;
    }
    void give_back(void* p, size_t n) {
        const size_t a = (n + 255) & ~static_cast<size_t>(255);
        if (static_cast<char*>(p) + a == base + top) top -= a;  // LIFO pop
    }
};

struct DevMem {
    void* p = nullptr;
    size_t bytes = 0;
    DevMem() = default;
    DevMem(const DevMem&) = delete;
    DevMem& operator=(const DevMem&) = delete;
    Arena* arena = nullptr;  // block of a setup scratch arena (not freed individually)
    ~DevMem() { release(); }
    void release() {
        if (p) {
            if (arena) arena->give_back(p, bytes);
            else cudaFree(p);
        }
        p = nullptr;
        bytes = 0;
        arena = nullptr;
    }
    void alloc(size_t n, size_t* tally) {
        release();
        if (n == 0) n = 16;
        if (!tally && Arena::current()) {
            if (void* q = Arena::current()->take(n)) {
                p = q;
                arena = Arena::current();
                bytes = n;
                return;
            }
        }
        cuda_check(cudaMalloc(&p, n), "cudaMalloc");
        bytes = n;
        if (tally) *tally += n;
    }
    template <class T> T* as() const { return static_cast<T*>(p); }
};

// Pinned host buffer: the chunk images of the streaming mode (slda_config.num_chunks).
struct HostBuf {
    void* p = nullptr;
    size_t bytes = 0;
    HostBuf() = default;
    HostBuf(const HostBuf&) = delete;
    HostBuf& operator=(const HostBuf&) = delete;
    HostBuf(HostBuf&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr, o.bytes = 0; }
    ~HostBuf() {
        if (p) cudaFreeHost(p);
    }
    void alloc(size_t n) {
        if (p) cudaFreeHost(p);
        p = nullptr;
        bytes = n;
        if (n) cuda_check(cudaMallocHost(&p, n), "cudaMallocHost");
    }
};

// One chunk of a streaming engine (the reference's file-backed ChunkStore slot,
// trainer.cpp:65-198, held in pinned host memory instead of a spill file): the device state
// build_state() produced for its document range, and the scalars that describe it.
struct ChunkImage {
    uint32_t doc_begin = 0, doc_end = 0, D = 0, nseg = 0, n_units = 0, n_long = 0, n_huge = 0, tbits = 1, wshift = 0;
    uint64_t T = 0, id_base = 0, out_offset = 0;
    bool doc_major = true, have_ids = false;
    std::vector<uint64_t> view_pos;  // gathered chunks: position in the engine's view per chunk token
    HostBuf tok, z, doc_start, row4, A, units, long_docs, ids, input_of_slot, seg_word, seg_off, seg_len, schedule;
};

uint32_t bits_for(uint64_t max_value) {
    uint32_t b = 1;
    while (b < 64 && (max_value >> b) != 0) ++b;
    return b;
}

}  // namespace

// =========================================================================
struct slda_engine {
    // Shape / config
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t side = nullptr;  // SSC, concurrent with the M-step (low priority)
    uint32_t D_all = 0, doc_begin = 0, doc_end = 0, D = 0;  // D = shard documents
    uint32_t V = 0, V_pad = 0, K = 0, K_pad = 0, l8_stride = 0, n_l8 = 0, tbits = 1;
    uint64_t T = 0;
    double alpha = 0, beta = 0;
    float falpha = 0;
    uint64_t seed = 0, id_base = 0;
    uint32_t iteration = 0;
    uint32_t rank = 0, world = 1;
    uint32_t nseg = 0, n_units = 0, n_long = 0, n_huge = 0;
    bool doc_major = true;
    bool have_ids = false;  // per-slot RNG element ids (non doc-major input or explicit ids)
    bool vanilla = false;  // SamplerKind::kVanilla (trainer.cpp:281-285)
    uint32_t tbits0 = 1;   // minimal C_dk topic field for K (configure)
    // One resident shard zeroes C_wk right after the phi kernel, inside the wait for the
    // side-stream SSC, instead of at the start of the next iteration (reset_word_topic off the
    // critical path); C_wk is then recounted from z when a caller asks for it.
    bool b_zeroed = false;
    bool early_reset() const { return !peer && !streaming && T > 0; }
    // Streaming mode (slda_config.num_chunks > 1 and the corpus state over device_budget): the
    // shard's documents in chunks whose state lives in pinned host memory and passes through
    // the device buffers above one chunk at a time.  T_view / D_view: the whole engine view.
    bool streaming = false;
    std::vector<ChunkImage> chunks;
    int resident = -1;      // chunk whose state is in the device buffers
    HostBuf chunk_nnz;      // per chunk: nnz of its C_dk after the last SSC (u64, pinned)
    DevMem chunk_cnt;       // per chunk: the SSC's nnz counter on the device
    unsigned long long* nnz_dst = nullptr;  // SSC nnz target (a chunk's counter while streaming)
    // The second device window: the next chunk is uploaded into it on `copy` while the current
    // one computes, then the windows swap (pointer swap) -- H2D, compute and D2H overlap.
    static constexpr int kStateBufs = 13;
    DevMem shadow[kStateBufs];
    cudaStream_t copy = nullptr;
    cudaEvent_t ev_in = nullptr, ev_done = nullptr, ev_copy_end = nullptr;
    DevMem* state_buf(int j) {
        DevMem* m[kStateBufs] = {&tok, &z, &doc_start, &row4, &A, &units, &long_docs, &ids, &input_of_slot,
                                 &seg_word, &seg_off, &seg_len, &schedule};
        return m[j];
    }
    static const HostBuf& image_buf(const ChunkImage& im, int j) {
        const HostBuf* m[kStateBufs] = {&im.tok, &im.z, &im.doc_start, &im.row4, &im.A, &im.units, &im.long_docs,
                                        &im.ids, &im.input_of_slot, &im.seg_word, &im.seg_off, &im.seg_len,
                                        &im.schedule};
        return *m[j];
    }
    void set_scalars(uint32_t ci);
    uint64_t T_view = 0;
    uint32_t D_view = 0, view_begin = 0, view_end = 0;
    uint32_t nseg_view = 0;  // streaming: distinct words over all chunks (the merged layout's segments)
    int sampler_shape = -1;  // SLDA_SAMPLER (sampler.cu launch_sampler); -1 = default by K
    bool serial = false;     // SLDA_SERIAL=1: SSC on the main stream (measurement of each kernel alone)
    uint32_t wshift = 0;  // word field shift of the execution-order key
    size_t device_bytes = 0;
    uint64_t nnz = 0;

    // Device state
    DevMem tok, z, doc_start, row4, A, units, long_docs, hist_scratch;
    DevMem seg_word, seg_off, seg_len, schedule;  // PDOW getters
    DevMem input_of_slot, ids;                    // only for non doc-major input / explicit ids
    DevMem assign_buf;                            // gather_assignments staging (allocated on first use)
    DevMem B, bhat, l8, q, colsum, denom, zv, counters;
    // z transpose (zmove.cu; resident engines): the sampler's execution-order topics (zx), the
    // two intermediate orders (zc: slot-range buckets, zf: 16384-slot tiles) and the static
    // tables of the three passes.
    DevMem zx, zc, zf, zsk1, zsk2, zloc;
    DevMem zbase1, zbase2;                  // per-chunk run tables of the two permutes
    uint32_t zruns1 = 0, zruns2 = 0;        // runs (keys) per chunk
    bool zmove = false;
    void build_zlayout(bool trace = false);

    // Per-iteration phase events, a ring so async iterations can be profiled afterwards.
    static constexpr uint32_t kRing = 64;
    // 0 start, 1 reset, 2 sampler, 3 m-step start, 4 colsum, 5 phi, 6 end, 7 SSC end (side stream),
    // 8 exchange end (world > 1: the sparse reduce-scatter + all-gather; == 3 on one GPU),
    // 9 z transposed to slots (zmove; == 2 without it)
    cudaEvent_t ring[kRing][10] = {};
    cudaEvent_t* ev = ring[0];
    uint32_t ring_launches[kRing] = {};
    uint32_t slot = 0;
    uint32_t enqueued = 0;  // iterations this engine has run (bounds the event ring reads)
    // Peer-memory exchange (world > 1): the other ranks' sparse C_wk lists mapped through CUDA
    // IPC handles (slda_peer_export / slda_peer_attach); mstep.cu describes the exchange.
    bool peer = false, attached = false;
    DevMem bar;                            // barrier counter (rank 0's is the shared one)
    DevMem info1, ent1;                    // this rank's partial C_wk, all rows: {offset, n} + entries
    DevMem info2, ent2;                    // this rank's reduced word slice
    DevMem xcnt;                           // [cursor1, cursor2, overflow] (u32)
    DevMem xbytes;                         // per ring slot: bytes read from the other ranks (u64)
    uint64_t cap1 = 0, cap2 = 0;           // entry capacities (pieces of counts, see alloc_exchange)
    void* pinfo1[slda::kMaxPeers] = {};
    void* pent1[slda::kMaxPeers] = {};
    void* pinfo2[slda::kMaxPeers] = {};
    void* pent2[slda::kMaxPeers] = {};
    unsigned long long* pbar = nullptr;
    uint64_t bar_seq = 0;
    std::vector<void*> opened;             // IPC mappings to close
    void peer_barrier() {
        ++bar_seq;
        CK(slda::launch_peer_barrier(pbar, static_cast<unsigned long long>(world) * bar_seq, stream));
    }
    // Capacities in u32 entries (a count c takes ceil(c / 65535) of them):
    //   partial : <= min(V*K_pad, T_rank) non-zero cells + T_rank/65535 extra pieces;
    //   slice   : <= slice cells + T_total/65535, T_total < 2^32 * kMaxPeers.
    void alloc_exchange() {
        const uint64_t cells = static_cast<uint64_t>(V) * K_pad;
        cap1 = std::min<uint64_t>(cells, T) + T / 65535 + 64;
        cap2 = static_cast<uint64_t>(slice_rows()) * K_pad + ((1ull << 32) * slda::kMaxPeers) / 65535 + 64;
        if (cap1 > 0xFFFFFFFFull || cap2 > 0xFFFFFFFFull)
            validation("peer-memory exchange: a rank's sparse C_wk list exceeds 2^32 entries");
        bar.alloc(8, &device_bytes);
        info1.alloc(static_cast<size_t>(V) * 8 + 8, &device_bytes);
        ent1.alloc(cap1 * 4, &device_bytes);
        info2.alloc(static_cast<size_t>(slice_rows()) * 8 + 8, &device_bytes);
        ent2.alloc(cap2 * 4, &device_bytes);
        xcnt.alloc(16, &device_bytes);
        xbytes.alloc(8 * kRing, &device_bytes);
        CK(cudaMemsetAsync(bar.p, 0, 8, stream));
        CK(cudaMemsetAsync(xbytes.p, 0, xbytes.bytes, stream));
    }
    void exchange();
    uint32_t launches = 0;

    unsigned long long* nnz_counter() const { return counters.as<unsigned long long>(); }
    unsigned long long* entries_counter(uint32_t s) const { return counters.as<unsigned long long>() + 1 + s; }
    unsigned long long* entries_counter() const { return entries_counter(slot); }

    // Word-row slice owned in the M-step: slda_word_slice (host.cpp), the rule the CPU
    // choreography test (tests/test_sharding_gloo.py) shares.
    uint32_t slice_rows() const { return V_pad / world; }
    uint32_t row_begin() const {
        uint32_t b = 0, e = 0;
        slda_word_slice(V, world, rank, &b, &e, nullptr);
        return b;
    }
    uint32_t row_end() const {
        uint32_t b = 0, e = 0;
        slda_word_slice(V, world, rank, &b, &e, nullptr);
        return e;
    }

    void* scratch_to_free = nullptr;
    void* scratch_kept = nullptr;
    std::thread scratch_thread;
    // cudaFree of the setup arena unmaps tens of GB (0.2-0.45 s at C3, a sixth to a third of
    // an end-to-end C3 run) and a concurrent unmap also slows the first iterations.  With room
    // on the device (a quarter of it still free) the arena is simply kept until the engine is
    // destroyed (C3, bench.py e2e leg: setup 0.23 s every run instead of 0.23-0.63 s, first
    // iteration 148 -> 128 ms); otherwise a helper thread frees it off the caller's path.
    void release_scratch_async() {
        if (!scratch_to_free) return;
        void* p = scratch_to_free;
        scratch_to_free = nullptr;
        size_t free_b = 0, total_b = 0;
        if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess && free_b > total_b / 4) {
            scratch_kept = p;
            return;
        }
        const int dev = device;
        scratch_thread = std::thread([p, dev] {
            cudaSetDevice(dev);
            cudaFree(p);
        });
    }
    ~slda_engine() {
        if (scratch_thread.joinable()) scratch_thread.join();
        if (device >= 0) cudaSetDevice(device);
        if (scratch_to_free) cudaFree(scratch_to_free);  // setup failed before the hand-off
        if (scratch_kept) cudaFree(scratch_kept);
        if (stream) cudaStreamSynchronize(stream);
        for (auto& set : ring)
            for (auto& e : set)
                if (e) cudaEventDestroy(e);
        for (void* p : opened) cudaIpcCloseMemHandle(p);
        if (copy) cudaStreamSynchronize(copy);
        if (ev_in) cudaEventDestroy(ev_in);
        if (ev_done) cudaEventDestroy(ev_done);
        if (ev_copy_end) cudaEventDestroy(ev_copy_end);
        if (copy) cudaStreamDestroy(copy);
        if (side) cudaStreamDestroy(side);
        if (stream) cudaStreamDestroy(stream);
    }

    void set_device() const { CK(cudaSetDevice(device)); }

    // ---- CUB helpers (setup only) ----
    template <class Fn>
    void cub_call(Fn&& fn) {
        size_t tmp = 0;
        CK(fn(nullptr, tmp));
        DevMem t;
        t.alloc(tmp, nullptr);
        CK(fn(t.p, tmp));
    }
    void exclusive_sum(const uint32_t* in, uint32_t* out, uint64_t n) {
        if (n == 0) return;
        cub_call([&](void* t, size_t& b) {
            return cub::DeviceScan::ExclusiveSum(t, b, in, out, static_cast<int64_t>(n), stream);
        });
    }
    template <class T> T d2h_scalar(const T* p) {
        T v;
        CK(cudaMemcpyAsync(&v, p, sizeof(T), cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        return v;
    }

    void configure(const slda_config& c, uint32_t vocab) {
        if (c.num_topics == 0) validation("number of topics must be >= 1");
        K = c.num_topics;
        alpha = c.alpha <= 0.0 ? 50.0 / K : c.alpha;  // trainer.cpp:18
        beta = c.beta;
        if (!(beta > 0.0)) validation("beta must be > 0");
        const uint32_t W = c.tree_branch ? c.tree_branch : 32u;
        if (W < 2) validation("tree branch must be >= 2");
        const uint64_t cap = static_cast<uint64_t>(W) * W * W;
        if (K > cap)
            validation("K=" + std::to_string(K) + " exceeds tree capacity W^3=" + std::to_string(cap));
        if (K > 65536) validation("device engine supports K <= 65536 (16-bit topics)");
        if (c.sampler > SLDA_SAMPLER_VANILLA) validation("unknown sampler kind");
        vanilla = c.sampler == SLDA_SAMPLER_VANILLA;
        if (vocab == 0) validation("preprocess requires V >= 1");
        world = c.world_size ? c.world_size : 1;
        rank = c.rank;
        if (rank >= world) validation("rank must be < world_size");
        seed = c.seed;
        falpha = static_cast<float>(alpha);
        V = vocab;
        {
            uint32_t b = 0, e = 0;
            slda_word_slice(V, world, rank, &b, &e, &V_pad);
        }
        K_pad = (K + slda::kBlock - 1) / slda::kBlock * slda::kBlock;
        n_l8 = K_pad / slda::kLeaf;
        l8_stride = (n_l8 + 3) / 4 * 4;
        tbits = tbits0 = bits_for(K - 1 ? K - 1 : 1);
        device = c.device;
        if (device < 0) CK(cudaGetDevice(&device));
        set_device();
        {
            // Main stream at the greatest priority, SSC's side stream at the least, so the
            // M-step's CTAs are dispatched first while both are pending.
            int least = 0, greatest = 0;
            CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
            const char* pr = std::getenv("SLDA_SSC_PRIORITY");  // "high": SSC's CTAs first (experiment)
            const bool ssc_high = pr && std::string(pr) == "high";
            CK(cudaStreamCreateWithPriority(&stream, cudaStreamNonBlocking, ssc_high ? least : greatest));
            CK(cudaStreamCreateWithPriority(&side, cudaStreamNonBlocking, ssc_high ? greatest : least));
        }
        for (auto& set : ring)
            for (auto& e : set) CK(cudaEventCreate(&e));
        if (world > 1) {
            // The ranks exchange through each other's memory (slda_peer_attach).
            if (world > slda::kMaxPeers)
                validation("peer-memory exchange supports world_size <= " + std::to_string(slda::kMaxPeers));
            peer = true;
        }
    }

    void alloc_model() {
        const size_t cells = static_cast<size_t>(V_pad) * K_pad;
        B.alloc(cells * 4, &device_bytes);
        bhat.alloc(cells * 4, &device_bytes);
        l8.alloc(static_cast<size_t>(V_pad) * l8_stride * 4, &device_bytes);
        q.alloc(static_cast<size_t>(V_pad) * 4, &device_bytes);
        colsum.alloc(static_cast<size_t>(K_pad) * 8, &device_bytes);
        denom.alloc(static_cast<size_t>(K_pad) * 16, &device_bytes);
        zv.alloc(static_cast<size_t>(K_pad) * 4, &device_bytes);
        counters.alloc(8 * (1 + kRing), &device_bytes);
        CK(cudaMemsetAsync(bhat.p, 0, bhat.bytes, stream));
        CK(cudaMemsetAsync(l8.p, 0, l8.bytes, stream));
        CK(cudaMemsetAsync(q.p, 0, q.bytes, stream));
    }

    // ---- init_state (trainer.cpp:354-417) ----
    void build(const slda_corpus_view& cv, const slda_config& c);
    // The device state of one document range (PDOW, C_dk, initial topics, its C_wk counts added
    // into B; B zeroed first when `first`).  `defer_scratch`: release the setup arena off the
    // caller's path (single-shard engines).
    void build_state(const slda_corpus_view& cv, const slda_config& c, bool first, bool defer_scratch);
    void build_streaming(const slda_corpus_view& cv, const slda_config& c);
    void save_image(ChunkImage& im);
    void swap_in(uint32_t ci);
    void swap_out(uint32_t ci);
    void enqueue_streaming_iteration();
    uint64_t doc_topic_nnz_total() const;
    // ---- run_iteration (trainer.cpp:419-449) ----
    void enqueue_iteration();
    // Sampler launch arguments of the next iteration.
    slda::SamplerArgs sampler_args() const {
        slda::SamplerArgs a{};
        a.tok = tok.as<uint2>();
        a.units = units.as<slda::Unit>();
        a.A = A.as<uint32_t>();
        a.bhat = bhat.as<float>();
        a.l8 = l8.as<float>();
        a.q = q.as<float>();
        a.ids = have_ids ? ids.as<uint64_t>() : nullptr;
        a.z = z.as<uint16_t>();
        a.zx = zmove ? zx.as<uint16_t>() : nullptr;
        a.zx_pos = nullptr;
        a.B = B.as<uint32_t>();
        a.seed = seed;
        a.id_base = id_base;
        a.stream_kind = iteration;  // trainer.cpp:423
        a.K = K;
        a.K_pad = K_pad;
        a.l8_stride = l8_stride;
        a.n_l8 = n_l8;
        a.tbits = tbits;
        a.row_entries = entries_counter();
        a.shape = sampler_shape;
        const char* an = std::getenv("SLDA_ASYNC_NEXT");  // default on; 0 = the register prefetch (A/B)
        a.async_next = an ? std::atoi(an) != 0 : 1u;
        a.vanilla = vanilla ? 1u : 0u;
        a.alpha = falpha;  // static_cast<float>(state.alpha), trainer.cpp:283
        return a;
    }

    void m_step();
    void ssc(cudaStream_t st);
};

// ----------------------------------------------------------------- build --
void slda_engine::build(const slda_corpus_view& cv, const slda_config& c) {
    D_all = cv.num_docs;
    if (cv.doc_begin > cv.doc_end || cv.doc_end > D_all) validation("invalid document shard range");
    if (cv.num_tokens > 0 && !cv.tokens) validation("tokens is null");
    configure(c, cv.vocab_size);
    alloc_model();
    // Streaming (the reference's file-backed chunks, trainer.cpp:406-415, with the GPU's memory
    // as the budget): the corpus state (~16 B/token resident, ~72 B/token more while building)
    // does not fit the device budget and more than one chunk was asked for.
    if (c.num_chunks > 1 && world == 1 && cv.num_tokens > 0) {
        uint64_t budget = c.device_budget;
        if (!budget) {
            size_t free_b = 0, total_b = 0;
            CK(cudaMemGetInfo(&free_b, &total_b));
            budget = static_cast<uint64_t>(free_b * 0.9);
        }
        const uint64_t need = cv.num_tokens * 88 + static_cast<uint64_t>(cv.doc_end - cv.doc_begin) * 144;
        streaming = need > budget;
    }
    if (streaming) {
        build_streaming(cv, c);
        return;
    }
    build_state(cv, c, true, true);
    T_view = T;
    D_view = D;
    view_begin = doc_begin;
    view_end = doc_end;
    if (peer) {  // the first M-step needs the other ranks: it runs in slda_peer_attach
        alloc_exchange();
    } else {
        m_step();
        if (early_reset()) {
            CK(cudaMemsetAsync(B.p, 0, B.bytes, stream));
            b_zeroed = true;
        }
    }
    CK(cudaStreamSynchronize(stream));
    nnz = d2h_scalar(nnz_counter());
}

void slda_engine::build_state(const slda_corpus_view& cv, const slda_config& c, bool first, bool defer_scratch) {
    // SLDA_TRACE=1: per-phase wall times of the setup on stderr (stream synchronised).
    const bool trace = std::getenv("SLDA_TRACE") != nullptr;
    auto t_last = std::chrono::steady_clock::now();
    auto phase = [&](const char* name) {
        if (!trace) return;
        if (stream) CK(cudaStreamSynchronize(stream));
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[slda setup] %-28s %8.1f ms\n", name,
                     std::chrono::duration<double, std::milli>(now - t_last).count());
        t_last = now;
    };
    doc_begin = cv.doc_begin;
    doc_end = cv.doc_end;
    D = doc_end - doc_begin;
    T = cv.num_tokens;
    if (T >= (1ull << 32)) validation("a single engine holds < 2^32 tokens; shard documents across GPUs");
    id_base = cv.token_id_base;
    tbits = tbits0;
    have_ids = false;
    // Scratch for every setup temporary below (~70 B/token at most); without room, plain
    // allocations.
    Arena arena(static_cast<size_t>(T) * 72 + static_cast<size_t>(D) * 64 + (256u << 20));
    if (defer_scratch) arena.deferred = &scratch_to_free;  // freed off the caller's path (release_scratch_async)
    phase("configure+alloc_model");

    // Copy the borrowed AoS tokens (sparselda::Token layout) and validate on device.
    DevMem aos, val;
    aos.alloc(T * 12, nullptr);
    val.alloc(sizeof(slda::ValidateOut), nullptr);
    if (T) CK(cudaMemcpyAsync(aos.p, cv.tokens, T * 12, cudaMemcpyHostToDevice, stream));
    {
        slda::ValidateOut init{~0ull, ~0ull, ~0ull, ~0ull, 0u};
        CK(cudaMemcpyAsync(val.p, &init, sizeof(init), cudaMemcpyHostToDevice, stream));
    }
    CK(slda::launch_validate(aos.as<uint32_t>(), T, doc_begin, doc_end, V, K,
                             val.as<slda::ValidateOut>(), stream));
    slda::ValidateOut vo;
    CK(cudaMemcpyAsync(&vo, val.p, sizeof(vo), cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    phase("h2d+validate");
    if (vo.bad_doc != ~0ull) validation("token " + std::to_string(vo.bad_doc) + ": doc outside the shard range");
    if (vo.bad_word != ~0ull) validation("token " + std::to_string(vo.bad_word) + ": word id out of range");
    bool draw = false;
    if (c.init_mode == SLDA_INIT_DRAW) {
        draw = true;
    } else if (c.init_mode == SLDA_INIT_GIVEN) {
        if (vo.first_invalid != ~0ull || vo.first_big != ~0ull)
            validation("token topic exceeds configured K");
    } else {
        // trainer.cpp:369-378: the first invalid topic ends the K check.
        if (vo.first_big < vo.first_invalid) validation("token topic exceeds configured K");
        draw = vo.first_invalid != ~0ull;
    }
    doc_major = vo.unsorted == 0 && cv.token_ids == nullptr;

    DevMem doc_local, word, topic_in;
    doc_local.alloc(T * 4, nullptr);
    word.alloc(T * 4, nullptr);
    if (!draw) topic_in.alloc(T * 4, nullptr);
    CK(slda::launch_deinterleave(aos.as<uint32_t>(), T, doc_begin, doc_local.as<uint32_t>(),
                                 word.as<uint32_t>(), draw ? nullptr : topic_in.as<uint32_t>(), stream));
    aos.release();
    phase("deinterleave");

    // Doc-grouped slot offsets (corpus.cpp:186-189).
    doc_start.alloc((static_cast<size_t>(D) + 1) * 4, &device_bytes);
    DevMem counts;  // document lengths, kept for the execution-order key
    uint32_t max_len = 0;
    {
        counts.alloc((static_cast<size_t>(D) + 1) * 4, nullptr);
        CK(cudaMemsetAsync(counts.p, 0, counts.bytes, stream));
        CK(slda::launch_doc_hist(doc_local.as<uint32_t>(), T, counts.as<uint32_t>(), stream));
        exclusive_sum(counts.as<uint32_t>(), doc_start.as<uint32_t>(), static_cast<uint64_t>(D) + 1);
        if (D) {
            DevMem mx;
            mx.alloc(4, nullptr);
            cub_call([&](void* t, size_t& b) {
                return cub::DeviceReduce::Max(t, b, counts.as<uint32_t>(), mx.as<uint32_t>(),
                                              static_cast<int64_t>(D), stream);
            });
            max_len = d2h_scalar(mx.as<uint32_t>());
        }
        // Counts in the high half-word whenever they fit (K <= 65536 is required anyway and no
        // document has more than 65535 tokens): the sampler's count decode is then one
        // I2F.U16.H1 (sampler.cu kC16).  Longer documents keep the minimal topic field.
        if (K <= 65536u && max_len <= 65535u) tbits = 16;
        if (tbits < 32 && (static_cast<uint64_t>(max_len) >> (32 - tbits)) != 0)
            validation("document of length " + std::to_string(max_len) +
                       " exceeds the packed C_dk count range at this K");
    }
    if (const char* f = std::getenv("SLDA_SAMPLER")) sampler_shape = slda::sampler_shape_from_name(f);
    if (const char* f = std::getenv("SLDA_SERIAL")) serial = std::string(f) == "1";

    phase("doc_start");
    // Slot permutation for corpora that are not doc-sorted: stable by doc keeps
    // corpus order within a document.
    if (!doc_major) {
        input_of_slot.alloc(T * 4, &device_bytes);
        DevMem iota, keys_out;
        iota.alloc(T * 4, nullptr);
        keys_out.alloc(T * 4, nullptr);
        CK(slda::launch_iota(iota.as<uint32_t>(), T, stream));
        const int dbits = static_cast<int>(bits_for(D ? D - 1 : 1));
        cub_call([&](void* t, size_t& b) {
            return cub::DeviceRadixSort::SortPairs(t, b, doc_local.as<uint32_t>(), keys_out.as<uint32_t>(),
                                                   iota.as<uint32_t>(), input_of_slot.as<uint32_t>(),
                                                   static_cast<int64_t>(T), 0, dbits, stream);
        });
        // RNG element id per slot (trainer.cpp:275 keys streams by corpus position).
        ids.alloc(T * 8, &device_bytes);
        have_ids = true;
        DevMem ids_in;
        if (cv.token_ids) {
            ids_in.alloc(T * 8, nullptr);
            CK(cudaMemcpyAsync(ids_in.p, cv.token_ids, T * 8, cudaMemcpyHostToDevice, stream));
        }
        CK(slda::launch_ids_by_slot(cv.token_ids ? ids_in.as<uint64_t>() : nullptr,
                                    input_of_slot.as<uint32_t>(), T, id_base, ids.as<uint64_t>(), stream));
        CK(cudaStreamSynchronize(stream));
    }

    // C_dk rows (header + entries, capacity len_d + 1 rounded to 8 entries, 32-byte
    // aligned); row offsets in uint4 units are static, so tok carries them.
    row4.alloc((static_cast<size_t>(D) + 1) * 4, &device_bytes);
    {
        DevMem quads;
        quads.alloc((static_cast<size_t>(D) + 1) * 4, nullptr);
        CK(cudaMemsetAsync(quads.p, 0, quads.bytes, stream));
        CK(slda::launch_row_quads(doc_start.as<uint32_t>(), D, quads.as<uint32_t>(), stream));
        exclusive_sum(quads.as<uint32_t>(), row4.as<uint32_t>(), static_cast<uint64_t>(D) + 1);
        const uint32_t total_quads = D ? d2h_scalar(row4.as<uint32_t>() + D) : 0;
        A.alloc(static_cast<size_t>(total_quads) * 16 + 512, &device_bytes);  // speculative group reads
        CK(cudaMemsetAsync(A.p, 0, A.bytes, stream));
    }

    phase("row offsets + A alloc");
    // PDOW: stable radix sort of keys laid out in slot order -> the reference's
    // (word, doc, token_id) order (corpus.cpp:157-175), refined by descending doc
    // length inside each word (execution order; getters re-derive the canonical one).
    tok.alloc(T * 8, &device_bytes);
    slda::KeyLayout kl{bits_for(D ? D - 1 : 1), bits_for(max_len ? max_len : 1), max_len};
    const uint32_t wbits = bits_for(V - 1 ? V - 1 : 1);
    if (kl.dbits + kl.lbits + wbits > 64) kl.lbits = 0;  // canonical order only
    wshift = kl.dbits + kl.lbits;
    {
        DevMem keys, keys_sorted, vals, slots_sorted, flags, seg_index;
        keys.alloc(T * 8, nullptr);
        keys_sorted.alloc(T * 8, nullptr);
        vals.alloc(T * 4, nullptr);
        slots_sorted.alloc(T * 4, nullptr);
        CK(slda::launch_make_keys(word.as<uint32_t>(), doc_local.as<uint32_t>(),
                                  doc_major ? nullptr : input_of_slot.as<uint32_t>(), counts.as<uint32_t>(), T,
                                  kl, keys.as<unsigned long long>(), vals.as<uint32_t>(), stream));
        if (T) {
            cub_call([&](void* t, size_t& b) {
                // Keys are laid out in slot order, which is doc-ascending (slots are doc-grouped),
                // and the radix sort is stable: sorting on the (word, length) bits alone already
                // yields (word, length, doc, slot) order -- 4 passes instead of 7 at C3.
                return cub::DeviceRadixSort::SortPairs(
                    t, b, keys.as<unsigned long long>(), keys_sorted.as<unsigned long long>(),
                    vals.as<uint32_t>(), slots_sorted.as<uint32_t>(), static_cast<int64_t>(T),
                    static_cast<int>(kl.dbits), static_cast<int>(wshift + wbits), stream);
            });
        }
        keys.release();
        vals.release();
        flags.alloc(T * 4, nullptr);
        seg_index.alloc(T * 4, nullptr);
        CK(slda::launch_make_tok(keys_sorted.as<unsigned long long>(), slots_sorted.as<uint32_t>(),
                                 row4.as<uint32_t>(), T, kl, tok.as<uint2>(), flags.as<uint32_t>(), stream));
        exclusive_sum(flags.as<uint32_t>(), seg_index.as<uint32_t>(), T);
        nseg = T ? d2h_scalar(seg_index.as<uint32_t>() + T - 1) + d2h_scalar(flags.as<uint32_t>() + T - 1) : 0;
        seg_word.alloc(static_cast<size_t>(nseg) * 4, &device_bytes);
        seg_off.alloc(static_cast<size_t>(nseg) * 4, &device_bytes);
        seg_len.alloc(static_cast<size_t>(nseg) * 4, &device_bytes);
        schedule.alloc(static_cast<size_t>(nseg) * 4, &device_bytes);
        CK(slda::launch_emit_segments(keys_sorted.as<unsigned long long>(), flags.as<uint32_t>(),
                                      seg_index.as<uint32_t>(), T, wshift, seg_word.as<uint32_t>(),
                                      seg_off.as<uint32_t>(), stream));
    }
    phase("PDOW sort + segments");
    // build_schedule (corpus.cpp:200-210): heavy first, ties by ascending word.
    if (nseg) {
        DevMem skeys, skeys_sorted, svals, counts, starts;
        skeys.alloc(static_cast<size_t>(nseg) * 8, nullptr);
        skeys_sorted.alloc(static_cast<size_t>(nseg) * 8, nullptr);
        svals.alloc(static_cast<size_t>(nseg) * 4, nullptr);
        CK(slda::launch_segment_lengths(seg_off.as<uint32_t>(), nseg, T, seg_len.as<uint32_t>(),
                                        skeys.as<unsigned long long>(), svals.as<uint32_t>(),
                                        seg_word.as<uint32_t>(), nullptr, stream));
        phase("  schedule keys");
        cub_call([&](void* t, size_t& b) {
            return cub::DeviceRadixSort::SortPairs(t, b, skeys.as<unsigned long long>(),
                                                   skeys_sorted.as<unsigned long long>(), svals.as<uint32_t>(),
                                                   schedule.as<uint32_t>(), static_cast<int64_t>(nseg), 0, 64,
                                                   stream);
        });
        phase("  schedule sort");
        counts.alloc(static_cast<size_t>(nseg) * 4, nullptr);
        starts.alloc(static_cast<size_t>(nseg) * 4, nullptr);
        CK(slda::launch_sched_counts(schedule.as<uint32_t>(), seg_len.as<uint32_t>(), nseg,
                                     counts.as<uint32_t>(), stream));
        exclusive_sum(counts.as<uint32_t>(), starts.as<uint32_t>(), nseg);
        n_units = d2h_scalar(starts.as<uint32_t>() + nseg - 1) + d2h_scalar(counts.as<uint32_t>() + nseg - 1);
        phase("  unit counts");
        units.alloc(static_cast<size_t>(n_units) * sizeof(slda::Unit), &device_bytes);
        CK(slda::launch_emit_units(schedule.as<uint32_t>(), seg_word.as<uint32_t>(), seg_off.as<uint32_t>(),
                                   seg_len.as<uint32_t>(), starts.as<uint32_t>(), nseg,
                                   units.as<slda::Unit>(), stream));
    } else {
        units.alloc(sizeof(slda::Unit), &device_bytes);
    }

    phase("schedule + units");
    // Documents longer than kSscWarpCap, for SSC's later passes: those longer than kSscMidCap
    // (the CTA histogram path) first, then the medium ones (the medium warp pass).
    {
        DevMem flags, iota, cnt;
        flags.alloc(static_cast<size_t>(D) * 4, nullptr);
        iota.alloc(static_cast<size_t>(D) * 4, nullptr);
        cnt.alloc(8, nullptr);
        long_docs.alloc(static_cast<size_t>(D) * 4, &device_bytes);
        if (D) {
            CK(slda::launch_iota(iota.as<uint32_t>(), D, stream));
            auto select = [&](uint32_t lo, uint32_t hi, uint32_t at) {
                CK(slda::launch_long_flags(doc_start.as<uint32_t>(), D, lo, hi, flags.as<uint32_t>(), stream));
                cub_call([&](void* t, size_t& b) {
                    return cub::DeviceSelect::Flagged(t, b, iota.as<uint32_t>(), flags.as<uint32_t>(),
                                                      long_docs.as<uint32_t>() + at, cnt.as<uint32_t>(),
                                                      static_cast<int64_t>(D), stream);
                });
                return d2h_scalar(cnt.as<uint32_t>());
            };
            n_huge = select(slda::kSscMidCap, 0xFFFFFFFFu, 0);
            n_long = n_huge + select(slda::kSscWarpCap, slda::kSscMidCap, n_huge);
        }
        if (n_huge && static_cast<size_t>(K_pad) * 4 > 200 * 1024)
            hist_scratch.alloc(static_cast<size_t>(std::min<uint32_t>(n_huge, 296)) * K_pad * 4, &device_bytes);
    }

    // Initial topics (trainer.cpp:383-388 / corpus.cpp:87-96), by slot.
    z.alloc(T * 2, &device_bytes);
    if (draw) {
        CK(slda::launch_init_topics(T, have_ids ? ids.as<uint64_t>() : nullptr, id_base, seed, K,
                                    z.as<uint16_t>(), stream));
    } else {
        CK(slda::launch_given_topics(topic_in.as<uint32_t>(), doc_major ? nullptr : input_of_slot.as<uint32_t>(),
                                     T, z.as<uint16_t>(), stream));
    }
    doc_local.release();
    word.release();
    topic_in.release();

    phase("long docs + init topics");
    // C_dk (rebuild_doc_topic), C_wk (count_chunk_into); phi + trees follow in build().
    ssc(stream);
    if (first) CK(cudaMemsetAsync(B.p, 0, B.bytes, stream));
    slda::RecountDraw rd{seed, id_base, have_ids ? ids.as<uint64_t>() : nullptr, draw ? K : 0u};
    CK(slda::launch_recount(tok.as<uint2>(), units.as<slda::Unit>(), n_units, z.as<uint16_t>(),
                            B.as<uint32_t>(), K_pad, rd, stream));
    phase("ssc + recount");
    if (!streaming) build_zlayout(trace);
    phase("z transpose layout");
}

// The static tables of the z transpose (zmove.cu): per level, (key, chunk) counts -> their
// exclusive scan (each run's first destination) -> the stable per-chunk ranking that writes the
// tables.  SLDA_ZMOVE=0 keeps the sampler's direct z[slot] stores (A/B).
void slda_engine::build_zlayout(bool trace) {
    const char* zm = std::getenv("SLDA_ZMOVE");
    zmove = T > 0 && !(zm && std::string(zm) == "0");
    if (!zmove) return;
    auto t_last = std::chrono::steady_clock::now();
    auto phase = [&](const char* name) {
        if (!trace) return;
        CK(cudaStreamSynchronize(stream));
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[slda setup]   z %-24s %8.1f ms\n", name,
                     std::chrono::duration<double, std::milli>(now - t_last).count());
        t_last = now;
    };
    uint32_t shift = slda::kZTileLog2;  // level-1 buckets: at most 256 slot ranges
    while (((T - 1) >> shift) >= 256) ++shift;
    const uint64_t nchunks = (T + (1u << slda::kZChunkLog2) - 1) >> slda::kZChunkLog2;
    zruns1 = slda::zlayout_keys(T, shift, 1);
    zruns2 = slda::zlayout_keys(T, shift, 2);
    zsk1.alloc(T * 4, &device_bytes);
    zsk2.alloc(T * 4, &device_bytes);
    zloc.alloc(T * 2, &device_bytes);
    zbase1.alloc(nchunks * zruns1 * 4, &device_bytes);
    zbase2.alloc(nchunks * zruns2 * 4, &device_bytes);
    DevMem slot_of, cnt, off;
    slot_of.alloc(T * 4, nullptr);  // slot of every zc position (level 1 writes, level 2 reads)
    for (uint32_t level = 1; level <= 2; ++level) {
        const size_t flat = slda::zlayout_flat_size(T, shift, level);
        cnt.alloc(flat * 4, nullptr);
        off.alloc(flat * 4, nullptr);
        CK(slda::launch_zlayout_count(tok.as<uint2>(), slot_of.as<uint32_t>(), T, shift, level, cnt.as<uint32_t>(),
                                      flat, stream));
        exclusive_sum(cnt.as<uint32_t>(), off.as<uint32_t>(), flat);
        CK(slda::launch_zlayout_emit(tok.as<uint2>(), slot_of.as<uint32_t>(), T, shift, level, off.as<uint32_t>(),
                                     level == 1 ? zsk1.as<uint32_t>() : zsk2.as<uint32_t>(),
                                     level == 1 ? zbase1.as<uint32_t>() : zbase2.as<uint32_t>(),
                                     slot_of.as<uint32_t>(), zloc.as<uint16_t>(), stream));
        off.release();
        cnt.release();
        phase(level == 1 ? "level 1 tables" : "level 2 tables");
    }
    CK(cudaStreamSynchronize(stream));
    zx.alloc(T * 2, &device_bytes);
    zc.alloc(T * 2, &device_bytes);
    zf.alloc(T * 2, &device_bytes);
    phase("zx/zc/zf alloc");
}

// ---- streaming mode (out-of-core chunks) ----
// The reference streams chunks through host RAM when their state exceeds memory_budget
// (trainer.cpp:406-415, ChunkStore :65-198: one chunk acquired at a time, spilled to a file
// on release).  Here the budget is the GPU's: each chunk's device state is built once, kept
// in pinned host memory, and passed through the engine's device buffers once per iteration
// (H2D of the chunk, sampler + SSC, D2H of its topics and C_dk rows), C_wk accumulating over
// the chunks before one M-step.  Token ids key the RNG and C_wk sums are integers, so the
// result is bit-identical to one resident shard (acceptance.cpp:426-445).
void slda_engine::build_streaming(const slda_corpus_view& cv, const slda_config& c) {
    const uint32_t b0 = cv.doc_begin, b1 = cv.doc_end;
    const uint64_t Tv = cv.num_tokens;
    const uint32_t* tk = cv.tokens;  // sparselda::Token AoS {doc, word, topic}
    // One host pass: validation (the device's messages), document lengths, doc-sortedness, and
    // the corpus-wide topic rule (trainer.cpp:369-378), decided once for every chunk.
    std::vector<uint32_t> lens(static_cast<size_t>(b1 - b0), 0u);
    bool sorted = cv.token_ids == nullptr;
    uint32_t mode = c.init_mode;
    bool decided = mode != SLDA_INIT_AUTO;
    for (uint64_t i = 0; i < Tv; ++i) {
        const uint32_t d = tk[3 * i], w = tk[3 * i + 1], t = tk[3 * i + 2];
        if (d < b0 || d >= b1) validation("token " + std::to_string(i) + ": doc outside the shard range");
        if (w >= V) validation("token " + std::to_string(i) + ": word id out of range");
        ++lens[d - b0];
        if (i && d < tk[3 * (i - 1)]) sorted = false;
        if (!decided) {
            if (t == 0xFFFFFFFFu) {
                mode = SLDA_INIT_DRAW;
                decided = true;
            } else if (t >= K) {
                validation("token topic exceeds configured K");
            }
        } else if (mode == SLDA_INIT_GIVEN && t >= K) {
            validation("token topic exceeds configured K");
        }
    }
    if (mode == SLDA_INIT_AUTO) mode = SLDA_INIT_GIVEN;
    const uint32_t Dv = b1 - b0;
    const uint32_t n = std::max<uint32_t>(1u, std::min<uint32_t>(c.num_chunks, std::max<uint32_t>(Dv, 1u)));
    std::vector<uint32_t> bnd(static_cast<size_t>(n) + 1, 0u);
    if (slda_shard_bounds(Dv, Tv, lens.data(), n, bnd.data()) != SLDA_OK) validation(g_error);
    std::vector<uint64_t> tok_first(static_cast<size_t>(n) + 1, 0);
    for (uint32_t ci = 0; ci < n; ++ci) {
        uint64_t t = 0;
        for (uint32_t d = bnd[ci]; d < bnd[ci + 1]; ++d) t += lens[d];
        tok_first[ci + 1] = tok_first[ci] + t;
    }
    chunks.clear();
    chunks.resize(n);
    std::vector<uint64_t> nnzs(n, 0);
    slda_config cc = c;
    cc.init_mode = mode;
    std::vector<uint32_t> gtok;
    std::vector<uint64_t> gids;
    for (uint32_t ci = 0; ci < n; ++ci) {
        ChunkImage& im = chunks[ci];
        slda_corpus_view sv = cv;
        sv.doc_begin = b0 + bnd[ci];
        sv.doc_end = b0 + bnd[ci + 1];
        if (sorted) {  // a contiguous token range
            const uint64_t f = tok_first[ci];
            sv.tokens = tk + 3 * f;
            sv.num_tokens = tok_first[ci + 1] - f;
            sv.token_id_base = cv.token_id_base + f;
            sv.token_ids = nullptr;
            im.out_offset = f;
        } else {  // gathered, in view order, with explicit ids
            gtok.clear();
            gids.clear();
            im.view_pos.clear();
            for (uint64_t i = 0; i < Tv; ++i) {
                const uint32_t d = tk[3 * i];
                if (d < sv.doc_begin || d >= sv.doc_end) continue;
                gtok.insert(gtok.end(), tk + 3 * i, tk + 3 * i + 3);
                gids.push_back(cv.token_ids ? cv.token_ids[i] : cv.token_id_base + i);
                im.view_pos.push_back(i);
            }
            sv.tokens = gtok.data();
            sv.num_tokens = gids.size();
            sv.token_id_base = 0;
            sv.token_ids = gids.data();
        }
        build_state(sv, cc, ci == 0, false);
        CK(cudaStreamSynchronize(stream));
        nnzs[ci] = d2h_scalar(nnz_counter());
        save_image(im);
    }
    chunk_nnz.alloc(8ull * n);
    std::memcpy(chunk_nnz.p, nnzs.data(), 8ull * n);
    resident = static_cast<int>(n) - 1;  // the last chunk built is still in the device buffers
    // Device buffers sized for the largest chunk, so iterations never allocate.
    auto grow = [&](DevMem& d, size_t need) {
        if (d.bytes < need) {
            DevMem t;
            t.alloc(need, &device_bytes);
            if (d.p && d.bytes) CK(cudaMemcpyAsync(t.p, d.p, d.bytes, cudaMemcpyDeviceToDevice, stream));
            CK(cudaStreamSynchronize(stream));
            std::swap(d.p, t.p);
            std::swap(d.bytes, t.bytes);
        }
    };
    size_t m[13] = {};
    for (const ChunkImage& im : chunks) {
        const HostBuf* hb[13] = {&im.tok, &im.z, &im.doc_start, &im.row4, &im.A, &im.units, &im.long_docs,
                                 &im.ids, &im.input_of_slot, &im.seg_word, &im.seg_off, &im.seg_len, &im.schedule};
        for (int j = 0; j < 13; ++j) m[j] = std::max(m[j], hb[j]->bytes);
    }
    DevMem* db[13] = {&tok, &z, &doc_start, &row4, &A, &units, &long_docs, &ids, &input_of_slot,
                      &seg_word, &seg_off, &seg_len, &schedule};
    for (int j = 0; j < 13; ++j) grow(*db[j], m[j]);
    for (int j = 0; j < kStateBufs; ++j)
        if (n > 1 && m[j]) shadow[j].alloc(m[j], &device_bytes);
    chunk_cnt.alloc(8ull * n, &device_bytes);
    CK(cudaMemcpyAsync(chunk_cnt.p, nnzs.data(), 8ull * n, cudaMemcpyHostToDevice, stream));
    CK(cudaStreamCreateWithFlags(&copy, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&ev_in, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ev_done, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ev_copy_end, cudaEventDisableTiming));
    uint64_t max_t = 0;
    uint32_t max_long = 0;
    for (const ChunkImage& im : chunks) {
        max_t = std::max(max_t, im.T);
        max_long = std::max(max_long, im.n_huge);
    }
    if (max_long && static_cast<size_t>(K_pad) * 4 > 200 * 1024)
        grow(hist_scratch, static_cast<size_t>(std::min<uint32_t>(max_long, 296)) * K_pad * 4);
    if (!assign_buf.p || assign_buf.bytes < max_t * 4) assign_buf.alloc(std::max<uint64_t>(max_t, 1) * 4, &device_bytes);
    T_view = Tv;
    D_view = Dv;
    view_begin = b0;
    view_end = b1;
    {
        std::vector<uint32_t> words;
        for (const ChunkImage& im : chunks) {
            const uint32_t* w = static_cast<const uint32_t*>(im.seg_word.p);
            words.insert(words.end(), w, w + im.nseg);
        }
        std::sort(words.begin(), words.end());
        nseg_view = static_cast<uint32_t>(std::unique(words.begin(), words.end()) - words.begin());
    }
    m_step();
    CK(cudaStreamSynchronize(stream));
    nnz = doc_topic_nnz_total();
}

void slda_engine::save_image(ChunkImage& im) {
    im.doc_begin = doc_begin;
    im.doc_end = doc_end;
    im.D = D;
    im.T = T;
    im.id_base = id_base;
    im.nseg = nseg;
    im.n_units = n_units;
    im.n_long = n_long;
    im.n_huge = n_huge;
    im.tbits = tbits;
    im.wshift = wshift;
    im.doc_major = doc_major;
    im.have_ids = have_ids;
    auto save = [&](HostBuf& h, const DevMem& d, size_t bytes) {
        h.alloc(bytes);
        if (bytes) CK(cudaMemcpyAsync(h.p, d.p, bytes, cudaMemcpyDeviceToHost, stream));
    };
    save(im.tok, tok, T * 8);
    save(im.z, z, T * 2);
    save(im.doc_start, doc_start, (static_cast<size_t>(D) + 1) * 4);
    save(im.row4, row4, (static_cast<size_t>(D) + 1) * 4);
    save(im.A, A, A.bytes);
    save(im.units, units, units.bytes);
    save(im.long_docs, long_docs, static_cast<size_t>(n_long) * 4);
    save(im.ids, ids, have_ids ? T * 8 : 0);
    save(im.input_of_slot, input_of_slot, doc_major ? 0 : T * 4);
    save(im.seg_word, seg_word, static_cast<size_t>(nseg) * 4);
    save(im.seg_off, seg_off, static_cast<size_t>(nseg) * 4);
    save(im.seg_len, seg_len, static_cast<size_t>(nseg) * 4);
    save(im.schedule, schedule, static_cast<size_t>(nseg) * 4);
    CK(cudaStreamSynchronize(stream));
}

// Chunk ci's state into the device buffers (stream-ordered, pinned -> HBM).
void slda_engine::swap_in(uint32_t ci) {
    if (resident == static_cast<int>(ci)) return;
    const ChunkImage& im = chunks[ci];
    for (int j = 0; j < kStateBufs; ++j) {
        const HostBuf& h = image_buf(im, j);
        if (!h.bytes) continue;
        DevMem& d = *state_buf(j);
        if (d.bytes < h.bytes) d.alloc(h.bytes, &device_bytes);  // only if build_streaming's sizing was short
        CK(cudaMemcpyAsync(d.p, h.p, h.bytes, cudaMemcpyHostToDevice, stream));
    }
    set_scalars(ci);
}

void slda_engine::set_scalars(uint32_t ci) {
    const ChunkImage& im = chunks[ci];
    doc_begin = im.doc_begin;
    doc_end = im.doc_end;
    D = im.D;
    T = im.T;
    id_base = im.id_base;
    nseg = im.nseg;
    n_units = im.n_units;
    n_long = im.n_long;
    n_huge = im.n_huge;
    tbits = im.tbits;
    wshift = im.wshift;
    doc_major = im.doc_major;
    have_ids = im.have_ids;
    resident = static_cast<int>(ci);
}

// The resident chunk's mutable state (topics, C_dk rows, its nnz) back to its image.
void slda_engine::swap_out(uint32_t ci) {
    ChunkImage& im = chunks[ci];
    if (im.z.bytes) CK(cudaMemcpyAsync(im.z.p, z.p, im.z.bytes, cudaMemcpyDeviceToHost, stream));
    if (im.A.bytes) CK(cudaMemcpyAsync(im.A.p, A.p, im.A.bytes, cudaMemcpyDeviceToHost, stream));
    CK(cudaMemcpyAsync(static_cast<uint64_t*>(chunk_nnz.p) + ci, chunk_cnt.as<unsigned long long>() + ci, 8,
                       cudaMemcpyDeviceToHost, stream));
}

uint64_t slda_engine::doc_topic_nnz_total() const {
    if (!streaming) return nnz;
    uint64_t t = 0;
    for (size_t ci = 0; ci < chunks.size(); ++ci) t += static_cast<const uint64_t*>(chunk_nnz.p)[ci];
    return t;
}

// run_iteration over the chunks (trainer.cpp:425-432 with a file-backed store): reset C_wk,
// then every chunk (the resident one first) through sampler + SSC, then one M-step.  Two device
// windows pipeline the chunks: while chunk k computes on the engine stream, the copy stream
// brings chunk k+1 into the other window (after writing chunk k-1's topics and C_dk rows back
// from it); then the windows swap.  Each transfer is ordered by events, so H2D, compute and D2H
// of neighbouring chunks overlap.
void slda_engine::enqueue_streaming_iteration() {
    launches = 0;
    slot = iteration % kRing;
    ev = ring[slot];
    CK(cudaEventRecord(ev[0], stream));
    CK(cudaMemsetAsync(B.p, 0, B.bytes, stream));  // reset_word_topic (counts.cpp:134-138)
    CK(cudaMemsetAsync(entries_counter(), 0, 8, stream));
    CK(cudaEventRecord(ev[1], stream));
    const uint32_t n = static_cast<uint32_t>(chunks.size());
    const uint32_t first = resident >= 0 ? static_cast<uint32_t>(resident) : 0u;
    swap_in(first);  // no-op unless a getter left another chunk resident
    auto order = [&](uint32_t k) { return (first + k) % n; };
    auto upload = [&](uint32_t ci) {  // into the shadow window, on the copy stream
        const ChunkImage& im = chunks[ci];
        for (int j = 0; j < kStateBufs; ++j) {
            const HostBuf& h = image_buf(im, j);
            if (h.bytes) CK(cudaMemcpyAsync(shadow[j].p, h.p, h.bytes, cudaMemcpyHostToDevice, copy));
        }
        CK(cudaEventRecord(ev_in, copy));
    };
    auto download = [&](uint32_t ci, DevMem* zb, DevMem* ab, cudaStream_t st) {  // topics + C_dk rows back
        ChunkImage& im = chunks[ci];
        if (im.z.bytes) CK(cudaMemcpyAsync(im.z.p, zb->p, im.z.bytes, cudaMemcpyDeviceToHost, st));
        if (im.A.bytes) CK(cudaMemcpyAsync(im.A.p, ab->p, im.A.bytes, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(static_cast<uint64_t*>(chunk_nnz.p) + ci, chunk_cnt.as<unsigned long long>() + ci, 8,
                           cudaMemcpyDeviceToHost, st));
    };
    CK(cudaStreamWaitEvent(copy, ev[1], 0));  // the previous iteration is done with both windows
    if (n > 1) upload(order(1));
    for (uint32_t k = 0; k < n; ++k) {
        const uint32_t ci = order(k);
        nnz_dst = chunk_cnt.as<unsigned long long>() + ci;
        CK(slda::launch_sampler(sampler_args(), n_units, stream));
        launches += n_units > 0;
        ssc(stream);
        nnz_dst = nullptr;
        if (k + 1 == n) {
            download(ci, &z, &A, stream);
            break;
        }
        CK(cudaEventRecord(ev_done, stream));
        CK(cudaStreamWaitEvent(stream, ev_in, 0));  // chunk k+1 has landed in the shadow window
        for (int j = 0; j < kStateBufs; ++j) {
            std::swap(state_buf(j)->p, shadow[j].p);
            std::swap(state_buf(j)->bytes, shadow[j].bytes);
        }
        set_scalars(order(k + 1));
        CK(cudaStreamWaitEvent(copy, ev_done, 0));  // chunk k's results are final
        download(ci, &shadow[1], &shadow[4], copy);  // shadow now holds chunk k (z = 1, A = 4)
        if (k + 2 < n) upload(order(k + 2));
    }
    CK(cudaEventRecord(ev_copy_end, copy));
    CK(cudaStreamWaitEvent(stream, ev_copy_end, 0));  // syncing the engine stream covers the copies
    CK(cudaEventRecord(ev[2], stream));
    CK(cudaEventRecord(ev[9], stream));
    CK(cudaEventRecord(ev[7], stream));
    m_step();
    CK(cudaEventRecord(ev[6], stream));
    ring_launches[slot] = launches;
    ++iteration;
    ++enqueued;
}

void slda_engine::ssc(cudaStream_t st) {
    CK(cudaMemsetAsync(nnz_dst ? nnz_dst : nnz_counter(), 0, 8, st));
    slda::SscArgs s{};
    s.z = z.as<uint16_t>();
    s.doc_start = doc_start.as<uint32_t>();
    s.D = D;
    s.row4 = row4.as<uint32_t>();
    s.A = A.as<uint32_t>();
    s.tbits = tbits;
    s.K_pad = K_pad;
    s.long_docs = long_docs.as<uint32_t>();
    s.n_long = n_long;
    s.n_huge = n_huge;
    s.hist_scratch = hist_scratch.as<uint32_t>();
    s.nnz_total = nnz_dst ? nnz_dst : nnz_counter();
    CK(slda::launch_ssc(s, st));
    launches += (D > 0) + (n_long > n_huge) + (n_huge > 0);
}

// M-step after the E-step's B: colsum -> denom -> phi/L4/L8/Q over every word row.  preprocess
// (counts.cpp:37-63) + rebuild_trees (trainer.cpp:237-248).  With world > 1 the sparse C_wk
// exchange first turns each rank's partial B into the full reduced C_wk (exchange()).
void slda_engine::m_step() {
    CK(cudaEventRecord(ev[3], stream));
    if (peer) exchange();
    CK(cudaEventRecord(ev[8], stream));
    CK(cudaMemsetAsync(colsum.p, 0, colsum.bytes, stream));
    // C_k: the topic histogram when this engine's z holds every token C_wk counts (one resident
    // shard: 2 B/token instead of 4 B/cell), else the column sums of the (exchanged) C_wk.
    if (!peer && !streaming && T > 0 && z.p && slda::zhist_fits(K_pad))
        CK(slda::launch_zhist(z.as<uint16_t>(), T, K_pad, colsum.as<unsigned long long>(), stream));
    else
        CK(slda::launch_colsum(B.as<uint32_t>(), 0, V_pad, K_pad, colsum.as<unsigned long long>(), stream));
    CK(slda::launch_denom(colsum.as<unsigned long long>(), K, K_pad, V, beta, denom.as<double>(),
                          zv.as<float>(), stream));
    CK(cudaEventRecord(ev[4], stream));
    CK(slda::launch_phi(B.as<uint32_t>(), denom.as<double>(), zv.as<float>(), bhat.as<float>(),
                        l8.as<float>(), q.as<float>(), 0, V_pad, K, K_pad, l8_stride, beta, falpha, stream));
    launches += 3;
    CK(cudaEventRecord(ev[5], stream));
    CK(cudaEventRecord(ev[6], stream));
}

// The C_wk reduce-scatter + all-gather over the other ranks' memory, sparse (mstep.cu):
// sparsify the partial B -> barrier -> add the other ranks' entries of the own word slice ->
// sparsify the reduced slice, clear the other rows -> barrier -> add every other slice's
// entries.  Afterwards B is the full reduced C_wk on every rank.  No trailing barrier: a
// rank's lists are next rewritten only after the next iteration's first barrier, which no rank
// passes before finishing this all-gather.  Integer sums: bit-identical to one GPU.
void slda_engine::exchange() {
    if (!attached) validation("peer-memory exchange: call slda_peer_attach on every rank first");
    const uint32_t r0 = row_begin(), r1 = row_end(), rows = slice_rows();
    uint32_t* cnt = xcnt.as<uint32_t>();
    unsigned long long* xb = xbytes.as<unsigned long long>() + slot;
    CK(cudaMemsetAsync(cnt, 0, 8, stream));  // cursors (the overflow flag stays sticky)
    CK(cudaMemsetAsync(xb, 0, 8, stream));
    CK(slda::launch_sparsify(B.as<uint32_t>(), 0, V, K_pad, info1.as<uint2>(), ent1.as<uint32_t>(), cnt,
                             static_cast<uint32_t>(cap1), cnt + 2, stream));
    peer_barrier();  // every rank's partial list is complete
    slda::PeerSparse rs{};
    for (uint32_t p = 0; p < world; ++p)
        if (p != rank)
            rs.src[rs.n++] = {static_cast<const uint2*>(pinfo1[p]), static_cast<const uint32_t*>(pent1[p]), 0u};
    CK(slda::launch_gather_add(rs, r0, r1, r1, r1, 0, B.as<uint32_t>(), K_pad, xb, stream));
    CK(slda::launch_sparsify(B.as<uint32_t>(), r0, r1, K_pad, info2.as<uint2>(), ent2.as<uint32_t>(), cnt + 1,
                             static_cast<uint32_t>(cap2), cnt + 2, stream));
    const size_t row_bytes = static_cast<size_t>(K_pad) * 4;
    if (r0 > 0) CK(cudaMemsetAsync(B.p, 0, r0 * row_bytes, stream));
    if (r1 < V_pad) CK(cudaMemsetAsync(B.as<uint32_t>() + static_cast<size_t>(r1) * K_pad, 0, (V_pad - r1) * row_bytes, stream));
    peer_barrier();  // every rank's reduced slice is listed
    slda::PeerSparse ag{};
    ag.n = world;
    for (uint32_t p = 0; p < world; ++p)
        if (p != rank)
            ag.src[p] = {static_cast<const uint2*>(pinfo2[p]), static_cast<const uint32_t*>(pent2[p]), p * rows};
    CK(slda::launch_gather_add(ag, 0, V, r0, r1, rows, B.as<uint32_t>(), K_pad, xb, stream));
    launches += 4;
}

// run_iteration (trainer.cpp:419-449) on the engine stream.
void slda_engine::enqueue_iteration() {
    if (streaming) {
        enqueue_streaming_iteration();
        return;
    }
    if (peer && !attached) validation("peer-memory exchange: call slda_peer_attach on every rank first");
    launches = 0;
    slot = iteration % kRing;
    ev = ring[slot];
    CK(cudaEventRecord(ev[0], stream));
    if (!b_zeroed) CK(cudaMemsetAsync(B.p, 0, B.bytes, stream));  // reset_word_topic (counts.cpp:134-138)
    b_zeroed = false;
    CK(cudaMemsetAsync(entries_counter(), 0, 8, stream));
    CK(cudaEventRecord(ev[1], stream));
    const slda::SamplerArgs a = sampler_args();
    CK(slda::launch_sampler(a, n_units, stream));
    launches += n_units > 0;
    CK(cudaEventRecord(ev[2], stream));
    if (zmove) {  // execution-order topics -> z by slot (zmove.cu)
        CK(slda::launch_zpermute(zx.as<uint16_t>(), zsk1.as<uint32_t>(), zbase1.as<uint32_t>(), zruns1, T,
                                 zc.as<uint16_t>(), stream));
        CK(slda::launch_zpermute(zc.as<uint16_t>(), zsk2.as<uint32_t>(), zbase2.as<uint32_t>(), zruns2, T,
                                 zf.as<uint16_t>(), stream));
        CK(slda::launch_ztile(zf.as<uint16_t>(), zloc.as<uint16_t>(), T, z.as<uint16_t>(), stream));
        launches += 3;
    }
    CK(cudaEventRecord(ev[9], stream));
    // The chunk's doc-topic rebuild (trainer.cpp:319-321) and the M-step both only read the
    // sampler's output (z / C_wk): SSC runs on the side stream, overlapped with colsum + phi,
    // and the iteration ends when both have.
    cudaStream_t ssc_stream = serial ? stream : side;
    CK(cudaStreamWaitEvent(ssc_stream, ev[9], 0));
    ssc(ssc_stream);
    CK(cudaEventRecord(ev[7], ssc_stream));
    m_step();
    if (early_reset()) {  // the next iteration's reset_word_topic, overlapped with SSC's tail
        CK(cudaMemsetAsync(B.p, 0, B.bytes, stream));
        b_zeroed = true;
    }
    CK(cudaStreamWaitEvent(stream, ev[7], 0));
    CK(cudaEventRecord(ev[6], stream));
    ring_launches[slot] = launches;
    ++iteration;
    ++enqueued;
}

void slda_set_error_internal(const std::string& msg) { g_error = msg; }

// =========================================================================
extern "C" {

const char* slda_last_error(void) { return g_error.c_str(); }
uint32_t slda_abi_version(void) { return SLDA_ABI_VERSION; }

int slda_create(const slda_corpus_view* corpus, const slda_config* config, slda_engine** out) {
    return guarded([&] {
        if (!corpus || !config || !out) validation("null argument");
        *out = nullptr;
        auto e = std::make_unique<slda_engine>();
        const auto t0 = std::chrono::steady_clock::now();
        e->build(*corpus, *config);
        e->release_scratch_async();
        if (std::getenv("SLDA_TRACE"))
            std::fprintf(stderr, "[slda setup] build total incl. scratch release %8.1f ms\n",
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
        *out = e.release();
    });
}

int slda_create_from_counts(uint32_t vocab_size, const uint32_t* word_topic, uint64_t num_tokens,
                            uint32_t iteration, const slda_config* config, slda_engine** out) {
    return guarded([&] {
        if (!config || !out || !word_topic) validation("null argument");
        *out = nullptr;
        auto e = std::make_unique<slda_engine>();
        e->configure(*config, vocab_size);
        e->alloc_model();
        e->iteration = iteration;
        e->T = 0;
        (void)num_tokens;
        e->units.alloc(sizeof(slda::Unit), &e->device_bytes);
        CK(cudaMemsetAsync(e->B.p, 0, e->B.bytes, e->stream));
        CK(cudaMemcpy2DAsync(e->B.p, static_cast<size_t>(e->K_pad) * 4, word_topic,
                             static_cast<size_t>(e->K) * 4, static_cast<size_t>(e->K) * 4, e->V,
                             cudaMemcpyHostToDevice, e->stream));
        if (e->world > 1) validation("create_from_counts is single-GPU");
        e->m_step();
        CK(cudaStreamSynchronize(e->stream));
        *out = e.release();
    });
}

void slda_destroy(slda_engine* e) { delete e; }

int slda_iterate_async(slda_engine* e) {
    return guarded([&] {
        if (!e) validation("null engine");
        e->set_device();
        e->enqueue_iteration();
    });
}

int slda_synchronize(slda_engine* e) {
    return guarded([&] {
        if (!e) validation("null engine");
        CK(cudaStreamSynchronize(e->stream));
    });
}

int slda_iterate(slda_engine* e, slda_iteration_stats* stats) {
    return guarded([&] {
        if (!e) validation("null engine");
        e->set_device();
        const auto start = std::chrono::steady_clock::now();
        e->enqueue_iteration();
        CK(cudaStreamSynchronize(e->stream));
        unsigned long long nnz_local = 0;
        if (e->streaming) nnz_local = e->doc_topic_nnz_total();
        else CK(cudaMemcpy(&nnz_local, e->nnz_counter(), 8, cudaMemcpyDeviceToHost));
        e->nnz = nnz_local;
        const double elapsed = std::chrono::duration<double>(std::chrono::steady_clock::now() - start).count();
        if (stats) {
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, e->ev[0], e->ev[6]));
            stats->iteration = e->iteration;
            stats->tokens = e->T_view;
            stats->elapsed_s = elapsed;
            stats->mtokens_per_s = elapsed > 0 ? static_cast<double>(e->T_view) / elapsed / 1e6 : 0.0;
            stats->mean_doc_topics = e->D_view ? static_cast<double>(nnz_local) / e->D_view : 0.0;
            stats->device_ms = ms;
        }
    });
}

int slda_set_iteration(slda_engine* e, uint32_t iteration) {
    return guarded([&] {
        if (!e) validation("null engine");
        e->iteration = iteration;
    });
}

int slda_get_info(const slda_engine* e, slda_info* info) {
    return guarded([&] {
        if (!e || !info) validation("null argument");
        info->num_docs = e->D_all;
        info->vocab_size = e->V;
        info->num_topics = e->K;
        info->iteration = e->iteration;
        info->num_tokens = e->T_view;
        info->doc_begin = e->view_begin;
        info->doc_end = e->view_end;
        info->rank = e->rank;
        info->world_size = e->world;
        info->alpha = e->alpha;
        info->beta = e->beta;
        info->seed = e->seed;
        info->num_segments = e->nseg;
        info->num_units = e->n_units;
        if (e->streaming) {
            info->num_segments = e->nseg_view;
            info->num_units = 0;
            for (const ChunkImage& im : e->chunks) info->num_units += im.n_units;
        }
        info->doc_topic_nnz = e->streaming ? e->doc_topic_nnz_total() : e->nnz;
        info->num_chunks = e->streaming ? static_cast<uint32_t>(e->chunks.size()) : 1u;
        info->streaming = e->streaming ? 1u : 0u;
        info->device_bytes = e->device_bytes;
        info->doc_major = e->doc_major ? 1u : 0u;
        info->padded_topics = e->K_pad;
        info->sampler_shape = static_cast<uint32_t>(slda::sampler_shape(e->sampler_args()));
    });
}

int slda_get_kernel_times_avg(const slda_engine* e, uint32_t last_n, slda_kernel_times* t) {
    return guarded([&] {
        if (!e || !t) validation("null argument");
        // Bounded by the iterations THIS engine enqueued (a resumed or checkpoint-loaded model
        // carries a larger iteration number but no recorded events).
        if (last_n == 0 || last_n > slda_engine::kRing || last_n > e->enqueued)
            validation("last_n must be in [1, min(64, iterations run by this engine)]");
        CK(cudaSetDevice(e->device));
        CK(cudaStreamSynchronize(e->stream));
        std::memset(t, 0, sizeof(*t));
        std::vector<unsigned long long> entries(slda_engine::kRing);
        CK(cudaMemcpy(entries.data(), e->entries_counter(0), 8 * slda_engine::kRing, cudaMemcpyDeviceToHost));
        for (uint32_t i = 0; i < last_n; ++i) {
            const uint32_t s = (e->iteration - 1 - i) % slda_engine::kRing;
            cudaEvent_t* ev = const_cast<cudaEvent_t*>(e->ring[s]);
            auto ms = [&](int a, int b) {
                float x = 0;
                CK(cudaEventElapsedTime(&x, ev[a], ev[b]));
                return static_cast<double>(x);
            };
            t->reset_ms += ms(0, 1);
            t->sampler_ms += ms(1, 2);
            t->zmove_ms += ms(2, 9);
            t->ssc_ms += ms(9, 7);  // side stream, concurrent with colsum + phi
            t->exchange_ms += ms(3, 8);
            t->colsum_ms += ms(8, 4);
            t->phi_ms += ms(4, 5);
            t->join_ms += ms(5, 6);  // phi end -> iteration end: the SSC join (+ the peer barrier)
            t->total_ms += ms(0, 6);
            t->sampler_row_entries += entries[s];
            t->launches += e->ring_launches[s];
        }
        const double n = last_n;
        t->reset_ms /= n;
        t->sampler_ms /= n;
        t->ssc_ms /= n;
        t->zmove_ms /= n;
        t->colsum_ms /= n;
        t->exchange_ms /= n;
        if (e->xbytes.p) {
            std::vector<unsigned long long> xb(slda_engine::kRing);
            CK(cudaMemcpy(xb.data(), e->xbytes.p, 8 * slda_engine::kRing, cudaMemcpyDeviceToHost));
            for (uint32_t i = 0; i < last_n; ++i) t->exchange_bytes += xb[(e->iteration - 1 - i) % slda_engine::kRing];
            t->exchange_bytes /= last_n;
        }
        t->phi_ms /= n;
        t->join_ms /= n;
        t->total_ms /= n;
        t->sampler_row_entries /= last_n;
        t->launches /= last_n;
    });
}

int slda_get_kernel_times(const slda_engine* e, slda_kernel_times* t) {
    return slda_get_kernel_times_avg(e, 1, t);
}

void* slda_stream(const slda_engine* e) { return e ? static_cast<void*>(e->stream) : nullptr; }

namespace {
void copy_matrix(slda_engine* e, const DevMem& m, void* out) {
    e->set_device();
    CK(cudaStreamSynchronize(e->stream));
    CK(cudaMemcpy2D(out, static_cast<size_t>(e->K) * 4, m.p, static_cast<size_t>(e->K_pad) * 4,
                    static_cast<size_t>(e->K) * 4, e->V, cudaMemcpyDeviceToHost));
}
}  // namespace

int slda_get_word_topic(slda_engine* e, uint32_t* out) {
    return guarded([&] {
        if (!e || !out) validation("null argument");
        e->set_device();
        // With world > 1 every rank's B holds the full reduced C_wk after the exchange.
        if (!e->b_zeroed) {
            copy_matrix(e, e->B, out);
            return;
        }
        // C_wk was zeroed for the next iteration: count_chunk_into (trainer.cpp:223-235) again
        // from the current topics, into a temporary.
        DevMem c;
        c.alloc(e->B.bytes, nullptr);
        CK(cudaMemsetAsync(c.p, 0, c.bytes, e->stream));
        slda::RecountDraw rd{e->seed, e->id_base, e->have_ids ? e->ids.as<uint64_t>() : nullptr, 0u};
        CK(slda::launch_recount(e->tok.as<uint2>(), e->units.as<slda::Unit>(), e->n_units, e->z.as<uint16_t>(),
                                c.as<uint32_t>(), e->K_pad, rd, e->stream));
        copy_matrix(e, c, out);
    });
}

int slda_get_word_topic_prob(slda_engine* e, float* out) {
    return guarded([&] {
        if (!e || !out) validation("null argument");
        copy_matrix(e, e->bhat, out);
    });
}

int slda_get_tree_prefix(slda_engine* e, float* out) {
    return guarded([&] {
        if (!e || !out) validation("null argument");
        // L4 is not kept (the sampler re-derives it from L8 and phi): materialise it here.
        DevMem l4;
        l4.alloc(e->bhat.bytes, nullptr);
        CK(slda::launch_l4(e->bhat.as<float>(), e->V_pad, e->K_pad, l4.as<float>(), e->stream));
        copy_matrix(e, l4, out);
    });
}

int slda_get_tree_mass(slda_engine* e, float* out) {
    return guarded([&] {
        if (!e || !out) validation("null argument");
        e->set_device();
        CK(cudaStreamSynchronize(e->stream));
        CK(cudaMemcpy(out, e->q.p, static_cast<size_t>(e->V) * 4, cudaMemcpyDeviceToHost));
    });
}

int slda_get_assignments(slda_engine* e, uint32_t* out) {
    return guarded([&] {
        if (!e || (!out && e->T_view)) validation("null argument");
        e->set_device();
        if (e->streaming) {  // chunk by chunk through the device buffers, into its positions
            std::vector<uint32_t> tmp;
            for (uint32_t ci = 0; ci < e->chunks.size(); ++ci) {
                const ChunkImage& im = e->chunks[ci];
                if (im.T == 0) continue;
                e->swap_in(ci);
                CK(slda::launch_assignments(e->z.as<uint16_t>(), e->doc_major ? nullptr : e->input_of_slot.as<uint32_t>(),
                                            e->T, e->assign_buf.as<uint32_t>(), e->stream));
                if (im.view_pos.empty()) {
                    CK(cudaMemcpyAsync(out + im.out_offset, e->assign_buf.p, im.T * 4, cudaMemcpyDeviceToHost, e->stream));
                } else {
                    tmp.resize(im.T);
                    CK(cudaMemcpyAsync(tmp.data(), e->assign_buf.p, im.T * 4, cudaMemcpyDeviceToHost, e->stream));
                    CK(cudaStreamSynchronize(e->stream));
                    for (uint64_t i = 0; i < im.T; ++i) out[im.view_pos[i]] = tmp[i];
                }
            }
            CK(cudaStreamSynchronize(e->stream));
            return;
        }
        if (e->T == 0) return;
        // Permute/widen on the device, then one D2H straight into the caller's buffer.
        if (!e->assign_buf.p) e->assign_buf.alloc(e->T * 4, &e->device_bytes);
        CK(slda::launch_assignments(e->z.as<uint16_t>(), e->doc_major ? nullptr : e->input_of_slot.as<uint32_t>(),
                                    e->T, e->assign_buf.as<uint32_t>(), e->stream));
        CK(cudaMemcpyAsync(out, e->assign_buf.p, e->T * 4, cudaMemcpyDeviceToHost, e->stream));
        CK(cudaStreamSynchronize(e->stream));
    });
}

int slda_peer_export(slda_engine* e, slda_peer_handles* out) {
    return guarded([&] {
        if (!e || !out) validation("null argument");
        if (!e->peer) validation("slda_peer_export: engine was not created for peer-memory exchange");
        e->set_device();
        auto h = [&](const DevMem& m, unsigned char* dst) {
            cudaIpcMemHandle_t ih;
            CK(cudaIpcGetMemHandle(&ih, m.p));
            static_assert(sizeof(ih) == SLDA_PEER_HANDLE_BYTES, "cudaIpcMemHandle_t size");
            std::memcpy(dst, &ih, sizeof(ih));
        };
        h(e->info1, out->partial_index);
        h(e->ent1, out->partial_entries);
        h(e->info2, out->slice_index);
        h(e->ent2, out->slice_entries);
        h(e->bar, out->barrier);
    });
}

int slda_peer_attach(slda_engine* e, const slda_peer_handles* all) {
    return guarded([&] {
        if (!e || !all) validation("null argument");
        if (!e->peer) validation("slda_peer_attach: engine was not created for peer-memory exchange");
        if (e->attached) validation("slda_peer_attach: already attached");
        e->set_device();
        auto open = [&](const unsigned char* src) -> void* {
            cudaIpcMemHandle_t ih;
            std::memcpy(&ih, src, sizeof(ih));
            void* p = nullptr;
            CK(cudaIpcOpenMemHandle(&p, ih, cudaIpcMemLazyEnablePeerAccess));
            e->opened.push_back(p);
            return p;
        };
        for (uint32_t r = 0; r < e->world; ++r) {
            if (r == e->rank) continue;
            e->pinfo1[r] = open(all[r].partial_index);
            e->pent1[r] = open(all[r].partial_entries);
            e->pinfo2[r] = open(all[r].slice_index);
            e->pent2[r] = open(all[r].slice_entries);
        }
        e->pbar = e->rank == 0 ? e->bar.as<unsigned long long>()
                               : static_cast<unsigned long long*>(open(all[0].barrier));
        e->attached = true;
        e->m_step();  // init_state's M-step (trainer.cpp:395-400), now that every rank is reachable
        CK(cudaStreamSynchronize(e->stream));
    });
}

}  // extern "C"

namespace {
// C_dk rows copied to the host; empty documents have none.
struct HostRows {
    std::vector<uint32_t> doc_start, row4, A;
    uint32_t mask = 0, tbits = 0;
    const uint32_t* row(uint32_t d) const { return A.data() + static_cast<size_t>(row4[d]) * 4; }
    uint32_t nnz(uint32_t d) const {
        if (doc_start[d + 1] == doc_start[d]) return 0u;
        return (row(d)[0] & mask) + 1u;
    }
    // Decoded (topic, count) pairs in ascending topic order.
    template <class F>
    void for_each(uint32_t d, F&& f) const {
        const uint32_t n = nnz(d);
        const uint32_t* r = row(d);
        for (uint32_t i = 0; i < n; ++i) f(r[1 + i] & mask, r[1 + i] >> tbits);
    }
};

HostRows fetch_rows(slda_engine* e) {
    HostRows h;
    h.mask = (1u << e->tbits) - 1u;
    h.tbits = e->tbits;
    h.doc_start.resize(static_cast<size_t>(e->D) + 1);
    h.row4.resize(static_cast<size_t>(e->D) + 1);
    h.A.resize(e->A.bytes / 4);
    CK(cudaMemcpy(h.doc_start.data(), e->doc_start.p, h.doc_start.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(h.row4.data(), e->row4.p, h.row4.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(h.A.data(), e->A.p, e->A.bytes, cudaMemcpyDeviceToHost));
    return h;
}

// A streaming engine's chunk rows, from the chunk's pinned image (current after every
// completed iteration: swap_out copies them back).
HostRows image_rows(const ChunkImage& im) {
    HostRows h;
    h.mask = (1u << im.tbits) - 1u;
    h.tbits = im.tbits;
    const uint32_t* ds = static_cast<const uint32_t*>(im.doc_start.p);
    const uint32_t* r4 = static_cast<const uint32_t*>(im.row4.p);
    const uint32_t* a = static_cast<const uint32_t*>(im.A.p);
    h.doc_start.assign(ds, ds + im.D + 1);
    h.row4.assign(r4, r4 + im.D + 1);
    h.A.assign(a, a + im.A.bytes / 4);
    return h;
}

// Every (rows, D) of the engine: its resident shard, or each streamed chunk in document order.
template <class F>
void for_each_rows(slda_engine* e, F&& f) {
    if (!e->streaming) {
        f(fetch_rows(e), e->D);
        return;
    }
    for (const ChunkImage& im : e->chunks) f(image_rows(im), im.D);
}
}  // namespace

extern "C" {

int slda_get_doc_topic_nnz(slda_engine* e, uint64_t* nnz) {
    return guarded([&] {
        if (!e || !nnz) validation("null argument");
        e->set_device();
        CK(cudaStreamSynchronize(e->stream));
        uint64_t n = 0;
        for_each_rows(e, [&](const HostRows& h, uint32_t D) {
            for (uint32_t d = 0; d < D; ++d) n += h.nnz(d);
        });
        *nnz = n;
    });
}

int slda_get_doc_topic(slda_engine* e, uint64_t* row_offsets, uint32_t* topics, uint32_t* counts) {
    return guarded([&] {
        if (!e || !row_offsets) validation("null argument");
        e->set_device();
        CK(cudaStreamSynchronize(e->stream));
        uint64_t pos = 0, row = 0;
        row_offsets[0] = 0;
        for_each_rows(e, [&](const HostRows& h, uint32_t D) {
            for (uint32_t d = 0; d < D; ++d) {
                h.for_each(d, [&](uint32_t topic, uint32_t count) {
                    topics[pos] = topic;
                    counts[pos] = count;
                    ++pos;
                });
                row_offsets[++row] = pos;
            }
        });
    });
}

}  // extern "C"

namespace {
// The reference's single-chunk PDOW layout of the engine's resident shard (corpus.cpp:125-198).
struct Layout {
    std::vector<uint32_t> sorted_doc, sorted_word, shuffle_ptrs, doc_offsets, seg_word, seg_off, seg_len, schedule;
    std::vector<uint64_t> token_ids;
};

Layout shard_layout(slda_engine* e) {
    CK(cudaStreamSynchronize(e->stream));
    const uint64_t T = e->T;
    std::vector<uint2> tok(T);
    std::vector<uint32_t> dst(static_cast<size_t>(e->D) + 1), sw(e->nseg), so(e->nseg), sl(e->nseg), sc(e->nseg);
    std::vector<uint64_t> ids;
    if (T) CK(cudaMemcpy(tok.data(), e->tok.p, T * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(dst.data(), e->doc_start.p, dst.size() * 4, cudaMemcpyDeviceToHost));
    if (e->nseg) {
        CK(cudaMemcpy(sw.data(), e->seg_word.p, e->nseg * 4ull, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(so.data(), e->seg_off.p, e->nseg * 4ull, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(sl.data(), e->seg_len.p, e->nseg * 4ull, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(sc.data(), e->schedule.p, e->nseg * 4ull, cudaMemcpyDeviceToHost));
    }
    if (e->have_ids) {
        ids.resize(T);
        CK(cudaMemcpy(ids.data(), e->ids.p, T * 8, cudaMemcpyDeviceToHost));
    }
    // Canonical chunk order (word, doc, token_id) from the execution order: within a word
    // segment, sort by doc; slots are doc-grouped in corpus order, so sorting by slot gives
    // (doc, token_id).
    std::vector<uint32_t> slot(T), doc(T);
    for (uint64_t i = 0; i < T; ++i) slot[i] = tok[i].y;
    for (uint32_t s = 0; s < e->nseg; ++s) std::sort(slot.begin() + so[s], slot.begin() + so[s] + sl[s]);
    for (uint64_t i = 0; i < T; ++i)
        doc[i] = static_cast<uint32_t>(std::upper_bound(dst.begin(), dst.end(), slot[i]) - dst.begin() - 1);
    Layout L;
    L.sorted_doc.resize(T);
    L.sorted_word.resize(T);
    L.token_ids.resize(T);
    L.shuffle_ptrs.resize(T);
    // shuffle_ptrs: doc-grouped slot in word-major order per doc (corpus.cpp:190-195).
    std::vector<uint32_t> cursor(dst.begin(), dst.end() - 1);
    uint32_t seg = 0;
    for (uint64_t i = 0; i < T; ++i) {
        while (seg + 1 < e->nseg && so[seg + 1] <= i) ++seg;
        L.sorted_doc[i] = doc[i] + e->doc_begin;
        L.sorted_word[i] = sw[seg];
        L.token_ids[i] = ids.empty() ? e->id_base + slot[i] : ids[slot[i]];
        L.shuffle_ptrs[i] = cursor[doc[i]]++;
    }
    L.doc_offsets = std::move(dst);
    L.seg_word = std::move(sw);
    L.seg_off = std::move(so);
    L.seg_len = std::move(sl);
    L.schedule = std::move(sc);
    return L;
}

// A streaming engine's layout as one chunk (what build_chunks(corpus, 1) gives): per word, the
// chunks' segments in chunk order (their documents ascend), doc-grouped slots offset by the
// tokens of the earlier chunks, and the schedule rebuilt over the merged segments
// (corpus.cpp:200-210).
Layout merged_layout(slda_engine* e) {
    std::vector<Layout> parts;
    for (uint32_t ci = 0; ci < e->chunks.size(); ++ci) {
        e->swap_in(ci);
        parts.push_back(shard_layout(e));
    }
    Layout L;
    L.doc_offsets.push_back(0);
    std::vector<uint64_t> base(parts.size() + 1, 0);
    for (size_t c = 0; c < parts.size(); ++c) {
        base[c + 1] = base[c] + parts[c].sorted_doc.size();
        for (size_t d = 1; d < parts[c].doc_offsets.size(); ++d)
            L.doc_offsets.push_back(static_cast<uint32_t>(base[c] + parts[c].doc_offsets[d]));
    }
    std::vector<size_t> next(parts.size(), 0);  // next segment of each chunk
    for (;;) {
        uint32_t w = 0xFFFFFFFFu;
        for (size_t c = 0; c < parts.size(); ++c)
            if (next[c] < parts[c].seg_word.size()) w = std::min(w, parts[c].seg_word[next[c]]);
        if (w == 0xFFFFFFFFu) break;
        L.seg_word.push_back(w);
        L.seg_off.push_back(static_cast<uint32_t>(L.sorted_doc.size()));
        for (size_t c = 0; c < parts.size(); ++c) {
            const Layout& P = parts[c];
            if (next[c] >= P.seg_word.size() || P.seg_word[next[c]] != w) continue;
            const uint32_t o = P.seg_off[next[c]], n = P.seg_len[next[c]];
            for (uint32_t i = o; i < o + n; ++i) {
                L.sorted_doc.push_back(P.sorted_doc[i]);
                L.sorted_word.push_back(P.sorted_word[i]);
                L.token_ids.push_back(P.token_ids[i]);
                L.shuffle_ptrs.push_back(static_cast<uint32_t>(base[c] + P.shuffle_ptrs[i]));
            }
            ++next[c];
        }
        L.seg_len.push_back(static_cast<uint32_t>(L.sorted_doc.size()) - L.seg_off.back());
    }
    L.schedule.resize(L.seg_word.size());
    for (uint32_t i = 0; i < L.schedule.size(); ++i) L.schedule[i] = i;
    std::stable_sort(L.schedule.begin(), L.schedule.end(), [&](uint32_t a, uint32_t b) {
        return L.seg_len[a] != L.seg_len[b] ? L.seg_len[a] > L.seg_len[b] : L.seg_word[a] < L.seg_word[b];
    });
    return L;
}
}  // namespace

extern "C" {

int slda_get_pdow(slda_engine* e, uint32_t* sorted_doc, uint32_t* sorted_word, uint64_t* token_ids,
                  uint32_t* shuffle_ptrs, uint32_t* doc_offsets, uint32_t* seg_word,
                  uint32_t* seg_offset, uint32_t* seg_length, uint32_t* schedule) {
    return guarded([&] {
        if (!e) validation("null engine");
        e->set_device();
        const Layout L = e->streaming ? merged_layout(e) : shard_layout(e);
        auto put = [](auto* dst, const auto& v) {
            if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(v[0]));
        };
        put(sorted_doc, L.sorted_doc);
        put(sorted_word, L.sorted_word);
        put(token_ids, L.token_ids);
        put(shuffle_ptrs, L.shuffle_ptrs);
        put(doc_offsets, L.doc_offsets);
        put(seg_word, L.seg_word);
        put(seg_offset, L.seg_off);
        put(seg_length, L.seg_len);
        put(schedule, L.schedule);
    });
}

int slda_heldout_ll(slda_engine* e, uint32_t num_docs, uint32_t vocab_size, uint64_t num_tokens,
                    const uint32_t* tokens, uint32_t burn_in, uint64_t seed, double* per_token_ll,
                    uint64_t* tokens_evaluated) {
    return guarded([&] {
        if (!e || !per_token_ll || !tokens_evaluated || (num_tokens && !tokens)) validation("null argument");
        // eval.cpp:53-59 validations, HeldoutSet::from_corpus split (eval.cpp:14-28).
        if (num_docs == 0) validation("held-out set is empty");
        if (vocab_size != e->V) validation("held-out vocabulary size does not match model");
        std::vector<uint64_t> est_off(static_cast<size_t>(num_docs) + 1, 0), evl_off(est_off);
        std::vector<uint32_t> seen(num_docs, 0);
        for (uint64_t t = 0; t < num_tokens; ++t) {
            const uint32_t d = tokens[3 * t], w = tokens[3 * t + 1];
            if (d >= num_docs || w >= vocab_size) validation("held-out token id out of range");
            (seen[d]++ % 2 == 0 ? est_off : evl_off)[d + 1]++;
        }
        for (uint32_t d = 0; d < num_docs; ++d) {
            est_off[d + 1] += est_off[d];
            evl_off[d + 1] += evl_off[d];
        }
        const uint64_t n_est = est_off[num_docs], n_evl = evl_off[num_docs];
        if (n_evl == 0) validation("held-out set has no evaluation tokens");
        std::vector<uint32_t> est_w(n_est ? n_est : 1), evl_w(n_evl);
        std::vector<uint64_t> ce(est_off.begin(), est_off.end() - 1), cv(evl_off.begin(), evl_off.end() - 1);
        std::fill(seen.begin(), seen.end(), 0u);
        uint64_t max_est = 0;
        for (uint64_t t = 0; t < num_tokens; ++t) {
            const uint32_t d = tokens[3 * t], w = tokens[3 * t + 1];
            if (seen[d]++ % 2 == 0) est_w[ce[d]++] = w; else evl_w[cv[d]++] = w;
        }
        for (uint32_t d = 0; d < num_docs; ++d) max_est = std::max(max_est, est_off[d + 1] - est_off[d]);
        uint32_t cap = 1;
        while (cap < max_est) cap <<= 1;
        if (static_cast<size_t>(cap) * 20 > 220 * 1024)
            validation("held-out document estimation half longer than the device limit (8192)");

        e->set_device();
        DevMem d_est_off, d_evl_off, d_est, d_evl, d_ll, d_mass;
        d_est_off.alloc(est_off.size() * 8, nullptr);
        d_evl_off.alloc(evl_off.size() * 8, nullptr);
        d_est.alloc(est_w.size() * 4, nullptr);
        d_evl.alloc(evl_w.size() * 4, nullptr);
        d_ll.alloc(n_evl * 8, nullptr);
        d_mass.alloc(static_cast<size_t>(e->V) * 8, nullptr);
        CK(cudaMemcpyAsync(d_est_off.p, est_off.data(), est_off.size() * 8, cudaMemcpyHostToDevice, e->stream));
        CK(cudaMemcpyAsync(d_evl_off.p, evl_off.data(), evl_off.size() * 8, cudaMemcpyHostToDevice, e->stream));
        CK(cudaMemcpyAsync(d_est.p, est_w.data(), est_w.size() * 4, cudaMemcpyHostToDevice, e->stream));
        CK(cudaMemcpyAsync(d_evl.p, evl_w.data(), evl_w.size() * 4, cudaMemcpyHostToDevice, e->stream));
        slda::HeldoutArgs a{};
        a.est_off = d_est_off.as<uint64_t>();
        a.est_word = d_est.as<uint32_t>();
        a.evl_off = d_evl_off.as<uint64_t>();
        a.evl_word = d_evl.as<uint32_t>();
        a.bhat = e->bhat.as<float>();
        a.l8 = e->l8.as<float>();
        a.q = e->q.as<float>();
        a.row_mass = d_mass.as<double>();
        a.ll_out = d_ll.as<double>();
        a.seed = seed;
        a.alpha = e->alpha;
        a.burn_in = burn_in;
        a.K = e->K;
        a.K_pad = e->K_pad;
        a.l8_stride = e->l8_stride;
        a.n_l8 = e->n_l8;
        a.cap = cap;
        CK(slda::launch_heldout(a, num_docs, e->V, e->K, e->K_pad, d_mass.as<double>(), e->stream));
        std::vector<double> ll(n_evl);
        CK(cudaMemcpyAsync(ll.data(), d_ll.p, n_evl * 8, cudaMemcpyDeviceToHost, e->stream));
        CK(cudaStreamSynchronize(e->stream));
        // eval.cpp:110-130: per-doc sequential sum, then the doc sums in doc order.
        double total = 0.0;
        for (uint32_t d = 0; d < num_docs; ++d) {
            double doc = 0.0;
            if (est_off[d + 1] > est_off[d])
                for (uint64_t j = evl_off[d]; j < evl_off[d + 1]; ++j) doc += ll[j];
            total += doc;
        }
        *per_token_ll = total / static_cast<double>(n_evl);
        *tokens_evaluated = n_evl;
    });
}

}  // extern "C"
