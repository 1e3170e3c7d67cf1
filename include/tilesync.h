/*
 * tilesync.h — C ABI of libtilesync_b200.so, the B200 (sm_100a) implementation of
 * tile-level semaphore synchronization between dependent kernels (arXiv 2305.13450,
 * "CuSync").
 *
 * The reference (/root/reference) ships no native code: its hot-path API is the Python
 * policy layer `tilesync_sim.policies` plus the CUDA listings of the paper. Each entry
 * point below names the reference interface it replaces.
 *
 * Conventions
 *   - Plain C types only. Device pointers are `void*`/`int*`; streams are `void*`
 *     (a cudaStream_t, 0 = legacy default stream).
 *   - Every function returns a ts_status. On failure `ts_last_error()` returns a
 *     thread-local message. Status codes map onto the reference's exception types
 *     (/root/reference/pkg/src/tilesync_sim/errors.py:4-9, policies.py:102-112,
 *     gpu.py:63-67): TS_ERR_CONFIG -> ConfigError, TS_ERR_VALUE -> ValueError,
 *     TS_ERR_TYPE -> TypeError.
 *   - The library allocates no persistent device memory. The caller (PyTorch) owns
 *     every buffer; the library borrows pointers for the duration of one
 *     stream-ordered call.
 *   - Host functions are reentrant. One in-flight chain per semaphore array.
 */
#ifndef TILESYNC_B200_H
#define TILESYNC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TS_ABI_VERSION 6

/* ---- status codes ---------------------------------------------------------------- */
typedef enum {
  TS_OK = 0,
  TS_ERR_CONFIG = 1,   /* ConfigError  (errors.py:4-5)                     */
  TS_ERR_VALUE = 2,    /* ValueError   (gpu.py:63-67, policies.py:133,188) */
  TS_ERR_TYPE = 3,     /* TypeError    (policies.py:125,142,166,178,205)   */
  TS_ERR_CUDA = 4,     /* CUDA runtime/driver failure                      */
  TS_ERR_DEADLOCK = 5  /* device watchdog fired (engine.py:614-637)        */
} ts_status;

/* ---- policy and order kinds (policies.py:24-73) ---------------------------------- */
typedef enum {
  TS_POLICY_TILE = 0,    /* TileSync       policies.py:24-26 */
  TS_POLICY_ROW = 1,     /* RowSync        policies.py:29-31 */
  TS_POLICY_STRIDED = 2, /* StridedSync    policies.py:34-38, param = stride */
  TS_POLICY_CONV2D = 3   /* Conv2DTileSync policies.py:41-50, param = kk     */
} ts_policy_kind;

typedef enum {
  TS_ORDER_ROW_MAJOR = 0,        /* RowMajor        policies.py:56-58 */
  TS_ORDER_STRIDED_ROW_MAJOR = 1, /* StridedRowMajor policies.py:61-70, param = stride */
  TS_ORDER_BANDED_COLUMN_MAJOR = 2 /* extension: bands of `param` tile rows, column-major
                                      inside a band (weight-block reuse in L2)        */
} ts_order_kind;

/* ---- host mirrors of the policy layer --------------------------------------------
 * These run the exact __host__ __device__ functions the kernels use, so the Python
 * drop-in and the device agree by construction. */

/* ABI version (TS_ABI_VERSION). */
int ts_abi_version(void);

/* Thread-local message for the last non-OK status. */
const char* ts_last_error(void);

/* sem_count(policy, producer_grid) — policies.py:115-125 (+check_policy 102-112). */
int ts_sem_count(int policy, int param, int gx, int gy, int gz, int* out);

/* post_target(policy, tile, producer_grid) — policies.py:128-142. */
int ts_post_target(int policy, int param, int tx, int ty, int tz, int gx, int gy,
                   int gz, int* out);

/* consumer_wait(policy, consumer_tile, k_step, producer_grid, producer_z)
 * — policies.py:145-166. *sem = -1 encodes `None`. */
int ts_consumer_wait(int policy, int param, int tx, int ty, int tz, int k_step, int pgx,
                     int pgy, int pgz, int producer_z, int* sem, int* expected);

/* wait_steps(policy, k_steps) — policies.py:169-178. Writes up to `cap` steps. */
int ts_wait_steps(int policy, int param, int k_steps, int* out, int cap, int* n);

/* order_tile(order, grid, counter) — policies.py:181-205. */
int ts_order_tile(int order, int stride, int gx, int gy, int gz, int counter, int* x,
                  int* y, int* z);

/* avoid_wait_kernel(producer, consumer, gpu) — engine.py:173-180 ("+W"). */
int ts_avoid_wait_kernel(int prod_tiles, int prod_occ, int cons_tiles, int cons_occ,
                         int num_sms, int* out);

/* ---- chain launch ------------------------------------------------------------------
 * A chain is a list of tile stages (GeMM kernels C = epi(A x B^T)) plus dependency
 * edges. It replaces the paper's CuSync/CuStage host code and the
 * reference's Scenario (engine.py:71-131). */

#define TS_MAX_STAGES 4
#define TS_MAX_DEPS 4

typedef enum { TS_DTYPE_F16 = 0, TS_DTYPE_BF16 = 1 } ts_dtype;

typedef enum {
  TS_EPI_NONE = 0,   /* C = A x B^T                                        */
  TS_EPI_GELU = 1,   /* C = GeLU_tanh(A x B^T) (GPT-3 tanh form) */
  TS_EPI_SWIGLU = 2, /* C = SiLU(gate) * up, gate/up interleaved per tile  */
  TS_EPI_RELU = 3    /* C = max(A x B^T, 0) (conv layers, BN folded)      */
} ts_epilogue;

typedef enum {
  TS_MODE_STREAM = 0, /* one launch per stage on one stream, no semaphores (baseline) */
  TS_MODE_FUSED = 1,  /* one persistent launch over all stages' tiles, semaphores     */
  TS_MODE_CORESIDENT = 2 /* the paper's own form: one launch per stage,
                            each on its own stream, semaphores live, the consumer stage's
                            stream gated by the wait kernel — ts_chain_launch_coresident */
} ts_mode;

typedef enum {
  TS_FLAG_KEEP_SEMS = 1,   /* do not zero semaphores at exit (for final-value parity)  */
  TS_FLAG_NO_REORDER = 2,  /* disable "+R": load the dependent A tile before B         */
  TS_FLAG_NO_WATCHDOG = 4, /* spin forever instead of aborting a wait after ~4 s      */
  TS_FLAG_ROW_INTERLEAVE = 8, /* fused two-GeMM Row/TileSync chains: claim tiles row by
                              row across the stages (producer row r, consumer row r,
                              producer row r+1, ...) instead of stage by stage — for
                              inputs that arrive row by row (MlpChain.run_host); every
                              consumer item is still claimed after the producer items
                              it waits on                                               */
  TS_FLAG_CONV_HALO = 32,    /* convolution stages with Cin = Cout = 64 (cta_group 1,
                              tile_n 64): stage each tile's input rows + 3x3 halo ONCE in
                              shared memory (a 4-D TMA box; zero padding from the
                              out-of-bounds fill) and address the nine tap-shifted A views
                              as descriptor offsets of whole 128-B pixel rows, with the
                              layer's weight taps resident — instead of one im2col box per
                              tap (9x the input bytes). Tiles are 128 positions of an image
                              in a width-padded order (row stride W + 2; two junk columns
                              per row, not stored) or, for wide images, 128 positions of one
                              row; the stage grid is N x tiles-per-image. Every conv stage of
                              the chain must qualify                                         */
  TS_FLAG_BALANCED = 16      /* fused CTA-pair 256-wide GeMM chains: static stream-K
                              schedule. Each stage's flattened (tile in claim order,
                              K-block) space is cut into one equal range per work unit
                              (CTA pair); unit u runs its range of every stage in turn,
                              cut at tile boundaries. A segment that does not start its
                              tile writes an fp32 partial plane (workspace: fp32[units x 2
                              x 128 x tile_cols], indexed by unit) and counts it into the
                              tile half's counter (counters: int32[tiles x 2], zero); the
                              tile's head segment (K-block 0, the last item of its unit)
                              waits for those planes, sums them into its TMEM accumulator,
                              applies the epilogue, stores and posts once — the
                              reference's semantics of an unsplit tile (z = 1). Every unit
                              ends each stage within one K-block of the others, so no
                              wave runs partially filled (the B200 extension to the
                              paper's per-stage tile counters, engine.py:424-470)       */
} ts_flags;

typedef struct {
  const void* a; /* [m, k] row-major, lda elements                         */
  const void* b; /* [n, k] row-major (weights, K-major), ldb elements      */
  void* c;       /* [m, n_out] row-major, ldc elements                     */
  int m, n, k;   /* n = accumulator columns (for SwiGLU n_out = n / 2)      */
  int lda, ldb, ldc;
  int dtype;     /* ts_dtype  */
  int epilogue;  /* ts_epilogue */
  int order;     /* ts_order_kind */
  int order_stride;
  int splits;        /* split-K slices (the reference's z extent); 0/1 = none. Each
                        slice posts once; the last to arrive sums the fp32 partials and
                        applies the epilogue (GeMM stages, not SwiGLU) */
  float* workspace;  /* splits > 1: device fp32[tiles * splits * tile_m * tile_cols]
                        (tile_m = rows of a tile: 128 x cta_group, or tile_n swapped;
                        tile_cols = accumulator columns: the stage's tile width, or 128
                        swapped)                                                       */
  int* counters;     /* splits > 1: device int32[2 * tiles * cta_group] (per tile half:
                        slice arrivals, then partials ready), zero on entry (kept zero) */
  int kind;          /* ts_stage_kind */
  int conv_n, conv_h, conv_w; /* TS_STAGE_CONV2D: image batch, height, width (3x3 kernel,
                        stride 1, padding 1: output H x W = input H x W); m = n*h*w,
                        k = 9 * Cin, a = NHWC input (lda = Cin), b = KRSC weights
                        [n][3][3][Cin] (ldb >= 9 Cin), c = NHWC output [m, n]        */
  int tile_n;        /* this stage's tile width: 0 = the chain's tile_n; 384 or 512 = a
                        CTA-pair tile of two MMAs per K-block (256 x 384: 2 x N=192;
                        256 x 512: 2 x N=256) sharing one A box — fewer operand bytes
                        per MAC than 256 x 256. GeMM and conv stages of cta_group 2,
                        tile_n 256 chains that do not feed a dot stage */
  int* in_sem;       /* optional external gate on operand A (e.g. a chunked host->device
                        copy signalled by ts_stream_signal): a tile in activation-row tile
                        r waits in_sem[r] >= in_expected before its first A load; never
                        zeroed by the kernel (callers advance in_expected per launch) */
  int in_expected;
  int* out_sem;      /* optional: each tile (and split-K slice) of activation-row tile r
                        adds 1 to out_sem[r] after all its rows are stored (system-scope
                        release), so a copy stream can ts_stream_wait for finished rows;
                        never zeroed */
  int tail_tiles;    /* last-wave balancing (extension): the last `tail_tiles` tiles of this
                        stage in claim order run as `tail_splits` split-K slices each (the
                        others unsplit), so the final partial wave spreads over more SMs.
                        Only for a normal-layout GeMM stage with splits <= 1 that nothing
                        waits on (no outgoing dependency); workspace / counters sized for
                        tiles * tail_splits slices. 0 = off */
  int tail_splits;
} ts_stage_desc;

typedef enum {
  TS_STAGE_GEMM = 0,     /* C = epi(A x B^T) on tcgen05                                    */
  TS_STAGE_ATTN_DOT = 1, /* attention's fused dot: a = XQKV [m, 3n] with
                            [Q heads | K heads | V heads] 128-column head tiles, c = XDot
                            [m, n]; XDot = Softmax(Q*V)*K per head and row (column-tile
                            local, dropout p = 0); b unused. Tile = rows x tile_n columns
                            (tile_n / 128 heads).                                         */
  TS_STAGE_CONV2D = 2,   /* 3x3 "same" convolution as implicit GeMM (PAPER.md:190-204,
                            461-463): A gathered by an im2col TMA map, K order = input-
                            channel tile (the producer's column tile) outer, filter tap,
                            64-channel block inner, so Conv2DTileSync(9) waits once per
                            producer column tile (policies.py:161-165)                   */
  TS_STAGE_ALLREDUCE = 3 /* tensor-parallel all-reduce of the producer's output over peer
                            memory (extension; the "next" row of SURVEY.md §8f): c = this
                            rank's producer output [m, n] (ldc), summed in place across
                            ts_chain_desc.peers. Tile = the producer's tile; this rank owns
                            tiles t with t % world == rank: it waits for tile t's semaphore
                            on every rank (system-scope acquire over P2P), sums the N
                            partial tiles in fp32 and stores the result into every rank's
                            buffer, then adds 1 to every rank's done counter. The only
                            dependency into it: producer GeMM -> allreduce, TileSync. */
} ts_stage_kind;

#define TS_MAX_PEERS 8

/* Peer memory of a tensor-parallel group for TS_STAGE_ALLREDUCE (all device pointers
 * valid in this process: P2P-mapped / IPC-opened / symmetric memory; index = rank). */
typedef struct {
  int world, rank;             /* group size (1..TS_MAX_PEERS) and this rank             */
  void* bufs[TS_MAX_PEERS];    /* rank q's allreduce buffer (its stage c)                */
  int* sems[TS_MAX_PEERS];     /* rank q's semaphores of the producer -> allreduce dep   */
  int* done[TS_MAX_PEERS];     /* rank q's arrival counter (int32, zero before the first
                                  launch): each owner CTA adds 1 per tile half it
                                  finalized into rank q's buffer; rank q's kernel exits
                                  once it reaches epoch x tiles x cta_group              */
  int epoch;                   /* launch generation, >= 1, advanced by 1 per launch on
                                  every rank in lockstep. The producer -> all-reduce
                                  semaphores and the done counters are monotone (never
                                  reset by the kernel): launch e waits for e x count, so a
                                  peer's state from launch e-1 never satisfies a wait    */
} ts_peer_desc;

typedef struct {
  int producer, consumer; /* stage indices, producer < consumer                 */
  int operand;            /* 0 = consumer's A operand (the only one GeMMs read) */
  int policy, param;      /* ts_policy_kind + stride / kk                        */
  int* sem;               /* device int32[sem_count], zero on entry             */
} ts_dep_desc;

typedef struct {
  int n_stages;
  ts_stage_desc stages[TS_MAX_STAGES];
  int n_deps;
  ts_dep_desc deps[TS_MAX_DEPS];
  int mode;      /* ts_mode */
  int tile_n;    /* 64, 128 or 256; 0 = 256 */
  int cta_group; /* 1: one CTA per 128-row tile; 2: CTA pair per 256-row tile
                    (tcgen05 cta_group::2); 0 = 2 */
  int swap_ab;   /* 1: small-batch tiles — UMMA M over 128 weight rows, UMMA N = tile_n
                    (32/64/128/256) over activation rows; needs cta_group 1 */
  int flags;     /* ts_flags bitmask */
  int num_ctas;  /* persistent CTAs; 0 = one per SM */
  int* scratch;  /* device int32[TS_SCRATCH_INTS], zero on first use; kernels restore it */
  void* trace;   /* optional device ts_trace_rec[trace_cap]; NULL = no tracing */
  int trace_cap;
  const ts_peer_desc* peers; /* TS_STAGE_ALLREDUCE only (host pointer; copied at launch) */
  int cluster_pairs; /* 0/1: one CTA pair (or CTA) per cluster. 2: clusters of two CTA pairs
                        (cta_group 2, tile_n 256, every GeMM stage tile_n 512, no dot /
                        conv / all-reduce stage): a 256 x 512 tile runs as two 256 x 256
                        pair tiles that share the activation rows by TMA multicast (24 KB
                        instead of 32 KB of operands per SM and K-block) and keep their
                        accumulators double-buffered in TMEM. Grids, semaphores, posts and
                        waits are those of the 256 x 512 tile. */
} ts_chain_desc;

#define TS_SCRATCH_INTS 32
/* scratch layout: [0] work counter, [1] CTA exit counter, [2] trace count,
 *                 [3] watchdog flag (1 = a wait timed out), [4] dot claim counter,
 *                 [8 + d] producer posts of dependency d (done watermark),
 *                 [16 + 4 s + {0, 1, 2}] co-resident mode: stage s's work counter, exit
 *                 counter and started flag (set by every CTA of the stage's launch at
 *                 start — stage.start(); the wait kernel spins on it), rest reserved */

/* Device trace record (one event of the reference's JSONL schema, engine.py:220-248). */
typedef struct {
  uint64_t t_ns;     /* %globaltimer */
  int32_t kind;      /* 0 scheduled, 1 wait_begin, 2 wait_end, 3 post, 4 finished;
                        extensions: 5 mma_begin, 6 mma_end (value = ns the tile's MMAs
                        waited for operands after the first stage), 7 epilogue_begin
                        (accumulator ready), 8 epilogue_end (thread 0's stores issued) */
  int32_t stage;     /* stage index */
  int32_t tb;        /* claim index within the stage (reference `tb`) */
  int32_t k;         /* reference k-step, -1 = none */
  int32_t dep;       /* dependency index, -1 = none */
  int32_t sem;       /* semaphore index, -1 = none */
  int32_t value;     /* expected (wait_*) or post value (post), -1 = none */
  int16_t x, y;      /* tile coordinate */
  int16_t z, smid;   /* slice, SM id */
  int32_t clk;       /* low 32 bits of the SM cycle counter (clock64) */
} ts_trace_rec;

/* Validate `desc` on the host and enqueue the chain on `stream`. Returns before the
 * device work completes. */
int ts_chain_launch(const ts_chain_desc* desc, void* stream);

/* Number of work items (tiles) a fused launch of `desc` processes, and the tile grid
 * of stage `s` (rows x cols) as the reference Stage.grid sees it. */
int ts_chain_grid(const ts_chain_desc* desc, int s, int* gx, int* gy);

/* Paper's wait kernel: one thread on `stream` spins until every
 * flags[i] != 0 (each set by the producer's stage.start()). */
int ts_wait_kernel_launch(const int* flags, int n, void* stream);

/* The paper's co-resident form (reference engine Mode.FINE with its
 * scheduling gate, engine.py:173-204): desc->mode must be TS_MODE_CORESIDENT. Stage s
 * runs as its own launch on streams[s] (n_streams == desc->n_stages) over its tiles in
 * its tile order, with live semaphores (wait before the dependent A loads, post after the
 * stores). wait_kernel: 0 = off, 1 = on, 2 = auto (avoid_wait_kernel: skipped when the
 * producer's and the consumer's launch grids fit one wave together); when on, the
 * consumer stage's stream first runs ts_wait_kernel_launch on the started flags of its
 * producers (scratch layout above). launch_order: 0 = stage order, 1 = adversarial
 * (consumers enqueued before their producers: with the gate off and a consumer grid that
 * fills the GPU this deadlocks; the semaphore watchdog aborts it after ~4 s and sets
 * scratch[3]). grid: CTAs (CTA pairs for cta_group 2) per stage launch, NULL = one per
 * tile (the reference's one thread block per tile; a CTA that finds no tile left exits).
 * The caller orders the streams against each other across launches (each stage stream
 * waits for the previous launch to finish). */
int ts_chain_launch_coresident(const ts_chain_desc* desc, void* const* streams, int n_streams,
                               int wait_kernel, int launch_order, const int* grid);

/* Stream-ordered semaphore ops for overlapping copies with a chain (the paper's
 * producer -> consumer tile signal, with a copy engine on one side). Both run on the
 * stream's front end (cuStreamWriteValue32 / cuStreamWaitValue32), not on an SM, so they
 * make progress while a persistent chain occupies every SM:
 * ts_stream_signal writes `value` to *sem once the stream's earlier work (e.g. a copy)
 * is complete and visible; ts_stream_wait blocks `stream` until *sem >= value. */
int ts_stream_signal(int* sem, int value, void* stream);
int ts_stream_wait(const int* sem, int value, void* stream);

/* Work items the current device runs at once for a chain of this geometry: CTAs
 * (cta_group 1), CTA pairs (2) or two-pair clusters (cluster_pairs 2), capped at the
 * number of clusters that are co-resident on the device — the wave size the planner's
 * quantization arithmetic uses (reference gpu.waves, GpuConfig(num_sms)). */
int ts_chain_units(int tile_n, int cta_group, int cluster_pairs, int swap_ab, int dtype,
                   int* out);

/* SM count of the current device. */
int ts_device_sm_count(int* out);

#ifdef __cplusplus
}
#endif
#endif /* TILESYNC_B200_H */
