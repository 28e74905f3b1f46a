/*
 * saberlda.h -- C-ABI of the B200-native SaberLDA/ESCA engine.
 *
 * The drop-in boundary for the reference's hot path (arxiv/paper_1610_02496,
 * `proj/`): one ESCA training iteration plus its setup.  Plain pointers and
 * sizes only; no torch or C++ types.  Every entry point names the reference
 * interface it replaces (paths relative to /root/reference/proj).
 *
 * Threading: calls on one engine are serialised by the caller (the reference
 * ModelState is not re-entrant either, trainer.cpp:325-332); different
 * engines are independent.  Ownership: the engine owns every device buffer;
 * host arrays passed in are borrowed and copied during the call; getters fill
 * caller-allocated buffers.
 *
 * Errors: every int-returning call returns SLDA_OK or one of the codes below,
 * mirroring sparselda::ValidationError / IoError (types.hpp:28-35) plus a
 * device code; slda_last_error() returns the calling thread's message.
 */
#ifndef SABERLDA_H
#define SABERLDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SLDA_ABI_VERSION 5u

enum {
    SLDA_OK = 0,
    SLDA_ERR_VALIDATION = 1, /* sparselda::ValidationError, CLI exit 1, Python ValueError */
    SLDA_ERR_IO = 2,         /* sparselda::IoError, CLI exit 2, Python IOError */
    SLDA_ERR_DEVICE = 3      /* CUDA failure (no reference analogue) */
};

#define SLDA_INVALID_TOPIC 0xFFFFFFFFu /* kInvalidTopic, types.hpp:17 */

/* How initial topics are chosen (trainer.cpp:369-388). */
enum {
    SLDA_INIT_AUTO = 0,  /* reference rule over the tokens passed in: if any topic is
                            kInvalidTopic, draw all uniformly; else validate topic < K */
    SLDA_INIT_DRAW = 1,  /* draw all uniformly (sharded runs: the host decided globally) */
    SLDA_INIT_GIVEN = 2  /* keep the given topics (validated < K) */
};

typedef struct slda_engine slda_engine;

/* A borrowed view of (a document shard of) a sparselda::Corpus (corpus.hpp:12-20).
 * tokens is T x 3 uint32 (doc, word, topic), the exact layout of sparselda::Token
 * (types.hpp:21-25).  Every token's doc must lie in [doc_begin, doc_end). */
typedef struct slda_corpus_view {
    uint32_t num_docs;        /* D of the whole corpus */
    uint32_t vocab_size;      /* V */
    uint64_t num_tokens;      /* T of this view (< 2^32 unless streaming: then < 2^32 per chunk) */
    const uint32_t* tokens;   /* T x 3 AoS */
    uint32_t doc_begin;       /* shard document range; [0, D) for one GPU */
    uint32_t doc_end;
    uint64_t token_id_base;   /* corpus position of tokens[0] */
    const uint64_t* token_ids;/* optional: per-token corpus position (RNG element id,
                                 trainer.cpp:275); NULL -> token_id_base + i */
} slda_corpus_view;

/* sparselda::TrainConfig (trainer.hpp:20-36) plus device placement. */
typedef struct slda_config {
    uint32_t num_topics;      /* K >= 1 */
    double alpha;             /* <= 0 resolves to 50/K (trainer.cpp:18) */
    double beta;              /* > 0 */
    uint64_t seed;
    uint32_t tree_branch;     /* W: capacity check K <= W^3 as the reference (trainer.cpp:19-26);
                                 0 -> 32.  The device search is layout-free (acceptance.cpp:140-200). */
    uint32_t init_mode;       /* SLDA_INIT_* */
    int32_t device;           /* CUDA ordinal; -1 = current device */
    uint32_t rank;            /* document shard index (0 for one GPU) */
    uint32_t world_size;      /* number of shards/GPUs (1 = no exchange; > 1: peer-memory
                                 exchange, slda_peer_export / slda_peer_attach) */
    uint32_t sampler;         /* SLDA_SAMPLER_* -- TrainConfig::sampler (trainer.hpp:18, :30) */
    uint32_t num_chunks;      /* TrainConfig::num_chunks (trainer.hpp:25); 0/1 = one resident shard */
    uint64_t device_budget;   /* bytes of device memory the corpus state may use (0 = the free
                                 memory).  With num_chunks > 1 and a state (~16 B/token, ~88 B/token
                                 while building) above it, the engine STREAMS: each chunk's state
                                 lives in pinned host memory and passes through the GPU once per
                                 iteration -- the reference's file-backed ChunkStore
                                 (trainer.cpp:65-198, :406-415) with HBM as the budget.  Results
                                 are bit-identical either way. */
} slda_config;

/* sparselda::SamplerKind (trainer.hpp:18). */
#define SLDA_SAMPLER_SPARSE 0u   /* ESCA sparsity-aware sampler (sampler.hpp:183-204) */
#define SLDA_SAMPLER_VANILLA 1u  /* O(K) dense-row baseline (sampler.hpp:222-236) */

/* sparselda::IterationStats (trainer.hpp:38-44) + device timings. */
typedef struct slda_iteration_stats {
    uint32_t iteration;       /* 1-based count after the call */
    uint64_t tokens;          /* T of this engine's shard */
    double elapsed_s;         /* host wall time of the iteration (trainer.cpp:422-447 span) */
    double mtokens_per_s;
    double mean_doc_topics;   /* K_d over this engine's documents (trainer.cpp:335-350) */
    double device_ms;         /* CUDA-event time of the iteration on the engine stream */
} slda_iteration_stats;

typedef struct slda_info {
    uint32_t num_docs, vocab_size, num_topics, iteration;
    uint64_t num_tokens;      /* shard tokens */
    uint32_t doc_begin, doc_end, rank, world_size;
    double alpha, beta;
    uint64_t seed;
    uint32_t num_segments;    /* distinct words in the shard (PDOW word segments) */
    uint32_t num_units;       /* sampler work units after heavy-word splitting */
    uint64_t doc_topic_nnz;   /* nnz of the shard's C_dk (after the last rebuild) */
    uint64_t device_bytes;    /* bytes of device memory held by the engine */
    uint32_t doc_major;       /* 1 if tokens came doc-sorted (no slot permutation) */
    uint32_t padded_topics;   /* K rounded up to the L4 block width (32) */
    uint32_t sampler_shape;   /* SLDA_SHAPE_*: the sampler kernel the iterations launch */
    uint32_t num_chunks;      /* chunks the state is held in (1 unless streaming) */
    uint32_t streaming;       /* 1: chunks stream through the GPU each iteration (device_budget) */
} slda_info;

/* Sampler kernels (slda_info.sampler_shape). */
#define SLDA_SHAPE_ROUND 0u    /* round-based lane-per-token, 4-sector groups */
#define SLDA_SHAPE_QUAD512 1u  /* quad-lane, 512-thread CTAs, next-line prefetch */
#define SLDA_SHAPE_QUAD256 2u  /* quad-lane, 256-thread CTAs */
#define SLDA_SHAPE_GLOBAL 3u   /* quad-lane, phi gathered from global memory (large K) */
#define SLDA_SHAPE_VANILLA 4u  /* SamplerKind::kVanilla O(K) baseline */

/* Per-kernel device times (ms) of the last iteration, for roofline accounting. */
typedef struct slda_kernel_times {
    double reset_ms, sampler_ms, ssc_ms, colsum_ms, phi_ms;
    double join_ms;               /* phi end -> iteration end: the wait for the side-stream SSC */
    double total_ms;
    uint64_t sampler_row_entries; /* sum over tokens of nnz(A_d) read by the sampler */
    uint32_t launches;            /* kernels launched by the iteration */
    double exchange_ms;           /* world > 1: the sparse C_wk reduce-scatter + all-gather (0 on one GPU) */
    uint64_t exchange_bytes;      /* world > 1: bytes this rank read from the other ranks' memory */
    double zmove_ms;              /* the sampler's topics from execution order to slots (zmove.cu) */
} slda_kernel_times;

/* ------------------------------------------------------------------ engine -- */

/* init_state (trainer.cpp:354-417): copies the corpus, builds the PDOW layout on device
 * (build_chunks corpus.cpp:125-198, build_schedule :200-210), initial topics
 * (init_assignments corpus.cpp:87-96), C_dk (rebuild_doc_topic counts.cpp:103-125),
 * C_wk (count_chunk_into trainer.cpp:223-235), phi (preprocess counts.cpp:37-63)
 * and the sampling trees (rebuild_trees trainer.cpp:237-248).
 * Device limits the reference does not have (SLDA_ERR_VALIDATION, never silent): K <= 65536;
 * every document shorter than 2^(32 - ceil(log2 K)) tokens (its counts share a 32-bit C_dk
 * entry with the topic: 2^18 at K = 10K). */
int slda_create(const slda_corpus_view* corpus, const slda_config* config, slda_engine** out);

/* Eval-only model from checkpointed counts (model_from_checkpoint trainer.cpp:514-532):
 * word_topic is V x K; no tokens. */
int slda_create_from_counts(uint32_t vocab_size, const uint32_t* word_topic,
                            uint64_t num_tokens, uint32_t iteration, const slda_config* config,
                            slda_engine** out);

void slda_destroy(slda_engine* e);

/* run_iteration (trainer.cpp:419-449): synchronous; fills stats (may be NULL). */
int slda_iterate(slda_engine* e, slda_iteration_stats* stats);
/* Enqueue one iteration on the engine stream without waiting (bench / pipelining). */
int slda_iterate_async(slda_engine* e);
int slda_synchronize(slda_engine* e);
/* Sets the RNG stream of the next iteration (resume; trainer.cpp:423). */
int slda_set_iteration(slda_engine* e, uint32_t iteration);

int slda_get_info(const slda_engine* e, slda_info* info);
int slda_get_kernel_times(const slda_engine* e, slda_kernel_times* t);
/* Average over the last `last_n` iterations (1..64), e.g. a run of slda_iterate_async. */
int slda_get_kernel_times_avg(const slda_engine* e, uint32_t last_n, slda_kernel_times* t);
/* cudaStream_t the engine launches on (as void*). */
void* slda_stream(const slda_engine* e);

/* ------------------------------------------------------------------ getters -- */

/* ModelState::word_topic (trainer.hpp:158), V x K row-major.  Sharded: collective. */
int slda_get_word_topic(slda_engine* e, uint32_t* out);
/* ModelState::word_topic_prob (trainer.hpp:159), V x K f32. */
int slda_get_word_topic_prob(slda_engine* e, float* out);
/* ModelState::tree_mass (trainer.hpp:160), V f32. */
int slda_get_tree_mass(slda_engine* e, float* out);
/* WaryTree::prefix() of every word (sampler.hpp:119), V x K f32 (the L4 level). */
int slda_get_tree_prefix(slda_engine* e, float* out);
/* ModelState::gather_assignments (trainer.cpp:203-213): T topics in view order. */
int slda_get_assignments(slda_engine* e, uint32_t* out);
/* DocTopicMatrix rows of the shard's documents (counts.hpp:33-80):
 * row_offsets has (doc_end-doc_begin)+1 entries; topics/counts have nnz entries. */
int slda_get_doc_topic_nnz(slda_engine* e, uint64_t* nnz);
int slda_get_doc_topic(slda_engine* e, uint64_t* row_offsets, uint32_t* topics,
                       uint32_t* counts);
/* Chunk PDOW arrays of the shard as one chunk (corpus.hpp:33-43): tokens sorted by
 * (word, doc, token_id) -> sorted_doc/sorted_word/token_ids (corpus positions, u64),
 * shuffle_ptrs, doc_offsets (docs+1), word_segments ascending (seg_*, num_segments),
 * and the heavy-first schedule (build_schedule) as segment indices. */
int slda_get_pdow(slda_engine* e, uint32_t* sorted_doc, uint32_t* sorted_word,
                  uint64_t* token_ids, uint32_t* shuffle_ptrs, uint32_t* doc_offsets,
                  uint32_t* seg_word, uint32_t* seg_offset, uint32_t* seg_length,
                  uint32_t* schedule);

/* ------------------------------------------------------------------ eval -- */

/* heldout_ll (eval.cpp:49-133) over a held-out corpus (AoS tokens, all docs), split by
 * HeldoutSet::from_corpus (eval.cpp:14-28).  Device limit: a document's estimation half (its
 * even positions) holds at most 8192 tokens (SLDA_ERR_VALIDATION otherwise). */
int slda_heldout_ll(slda_engine* e, uint32_t num_docs, uint32_t vocab_size, uint64_t num_tokens,
                    const uint32_t* tokens, uint32_t burn_in, uint64_t seed,
                    double* per_token_ll, uint64_t* tokens_evaluated);

/* ------------------------------------------------------------------ misc -- */

const char* slda_last_error(void);
uint32_t slda_abi_version(void);
/* Document shard bounds by the chunk_boundaries rule (corpus.cpp:103-121):
 * bounds has num_shards+1 entries.  Host-only. */
int slda_shard_bounds(uint32_t num_docs, uint64_t num_tokens, const uint32_t* doc_lengths,
                      uint32_t num_shards, uint32_t* bounds);
/* Word-row slice [*row_begin, *row_end) that shard `rank` of `world` owns in the M-step
 * (reduce-scatter of C_wk, phi/L4 rows, all-gather): V is padded to a multiple of world
 * (*padded_rows) and split evenly.  Host-only. */
int slda_word_slice(uint32_t vocab_size, uint32_t world, uint32_t rank, uint32_t* row_begin,
                    uint32_t* row_end, uint32_t* padded_rows);

/* Synthetic corpora.  Host-only, multi-threaded, deterministic in
 * (params, seed) regardless of thread count.  family 0 = G (LDA-generative: Zipf(1)
 * topics over seeded vocabulary permutations, Dirichlet(0.1) docs, lognormal(0.6)
 * lengths rescaled to sum to T), family 1 = U (uniform words, Poisson lengths).
 * Doc-major output: tokens T x 3 (doc, word, kInvalidTopic). */
typedef struct slda_gen_params {
    uint32_t family;
    uint32_t num_docs, vocab_size;
    uint64_t num_tokens;      /* exact T for family G; family U: mean length = T/D */
    uint32_t latent_topics;   /* family G K_true (default 100) */
    double zipf_s;            /* family G (default 1.0) */
    double doc_dirichlet;     /* family G (default 0.1) */
    double length_sigma;      /* family G lognormal sigma (default 0.6) */
    uint64_t seed;            /* default 20161008 */
    uint32_t threads;         /* 0 = hardware concurrency */
} slda_gen_params;
/* Returns the exact T that will be generated (two-phase use: size, then fill). */
int slda_generate_corpus_size(const slda_gen_params* p, uint64_t* num_tokens);
int slda_generate_corpus(const slda_gen_params* p, uint32_t* tokens, uint64_t capacity);
/* Per-document lengths (num_docs entries) and the tokens of documents [doc_begin, doc_end)
 * only, identical to the corresponding slice of slda_generate_corpus (sharded ranks). */
int slda_generate_doc_lengths(const slda_gen_params* p, uint32_t* lengths);
int slda_generate_docs(const slda_gen_params* p, uint32_t doc_begin, uint32_t doc_end,
                       uint32_t* tokens, uint64_t capacity);

/* ---- Peer-memory exchange (multi-GPU) --------------------------------------------------------
 * Create every rank's engine with world_size > 1, export each engine's buffer handles (CUDA
 * IPC), exchange them over any host channel, and attach every engine to all ranks' handles
 * (indexed by rank).  Every M-step then exchanges C_wk SPARSE over peer memory inside its own
 * kernels -- each rank lists its partial C_wk's non-zeros, adds the other ranks' entries of its
 * word slice (the reduce-scatter), lists its reduced slice, and adds every other slice's entries
 * (the all-gather) -- after which every rank holds the full reduced C_wk and computes phi / L4 /
 * L8 / Q locally (trainer.cpp:395-400 / 436-440 semantics).  NVLink on a multi-GPU node; the
 * same HBM when ranks share one GPU.  slda_peer_attach runs init_state's first M-step and is
 * collective. */
#define SLDA_PEER_HANDLE_BYTES 64
typedef struct slda_peer_handles {
    unsigned char partial_index[SLDA_PEER_HANDLE_BYTES];   /* {offset, n} per word row of the partial C_wk list */
    unsigned char partial_entries[SLDA_PEER_HANDLE_BYTES]; /* its entries: topic | count << 16 */
    unsigned char slice_index[SLDA_PEER_HANDLE_BYTES];     /* the same for the rank's reduced word slice */
    unsigned char slice_entries[SLDA_PEER_HANDLE_BYTES];
    unsigned char barrier[SLDA_PEER_HANDLE_BYTES];         /* barrier counter (rank 0's is used) */
} slda_peer_handles;

int slda_peer_export(slda_engine* engine, slda_peer_handles* out);
int slda_peer_attach(slda_engine* engine, const slda_peer_handles* all_ranks);

#ifdef __cplusplus
}
#endif
#endif /* SABERLDA_H */
