// ts_chain_kernel.cuh — persistent, warp-specialized tcgen05 GeMM over a chain of
// dependent tile stages, with the paper's tile-level semaphore protocol.
//
// One launch processes every tile of every stage. Work items are the stages' tiles laid
// end to end (stage 0's tiles first); a single global atomic counter hands them out, so
// any producer tile a consumer waits on was claimed earlier by a CTA that is already
// running it — the persistent replacement for the paper's wait kernel
// (engine.py:183-204). Within a stage, the n-th claim computes tile
// order_tile(order, grid, n) (the paper's stage.tile(); policies.py:181).
//
// CG = 1: one CTA per tile (UMMA M = 128). CG = 2: a CTA pair (cluster of 2 on one TPC)
// per tile, UMMA M = 256 with cta_group::2: each CTA loads its 128 rows of A and half
// of the B tile, halving per-SM operand traffic; the leader CTA issues the MMAs.
//
// Roles (256 threads per CTA):
//   warp 0 lane 0 : scheduler (leader) + TMA producer. For a consumer tile it issues the
//                   weight (B) tile first, then spins on the policy's semaphore
//                   (ld.acquire.gpu) and issues the dependent A tile ("+R",
//                   PAPER.md:534-540; kstep_duration engine.py:207-217).
//   warp 1        : tcgen05.mma issuer (leader only), fp32 accumulators in TMEM,
//                   double-buffered so the epilogue of tile i overlaps the mainloop of i+1.
//   warp 2        : TMEM allocator.
//   warps 4-7     : epilogue: tcgen05.ld -> GeLU/SwiGLU -> global stores; then the leader
//                   posts (fence + atom.release.gpu) to every outgoing dependency once the
//                   whole tile is stored (stage.post, PAPER.md:332,366-370;
//                   post_target policies.py:128-142).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include "tilesync.h"
#include "ts_policy.cuh"
#include "ts_ptx.cuh"

namespace ts {

constexpr int kBK = 64;         // K elements per smem stage = one 128-B swizzle row
constexpr int kTileRing = 4;
constexpr int kPostRing = 4;  // single-CTA kernels: posts handed to the post warp (warp 3)    // tile-id hand-off ring between scheduler and consumers
// Operand pipeline barriers are indexed by K-block sequence number (full: TMA bytes
// landed) and by commit group (empty: the MMAs that read a group of K-blocks are done),
// not by smem ring entry. One tcgen05.commit then frees several K-blocks (measured: each
// commit costs the tensor pipe a drain bubble), and the ring geometry (fixed slots or
// 16-KB chunks, 1-3 per K-block) is independent of the barriers.
constexpr int kFullRing = 16;    // > K-blocks in flight (<= 13)
constexpr int kCommitRing = 16;  // > commit groups in flight
// CTA pairs: the peer's "my stores of tile i are done" barrier ring. The peer's epilogue
// can run up to two tiles ahead of the leader's post (bounded by the two TMEM slots), so
// a 2-entry ring could see two phases complete before the leader waits — parity aliasing
// (observed as hangs when the leader's epilogue is slowed by split-K reductions or
// last-arriver dot tiles). Four entries keep every outstanding tile on its own barrier.
constexpr int kPeerRing = 4;
constexpr uint64_t kWatchdogNs = 4000000000ull;
constexpr int kStageGemm = 0;  // C = epi(A x B^T) on tcgen05
constexpr int kStageDot = 1;   // attention's fused softmax-dot over QKV column tiles
constexpr int kStageAllReduce = 3;  // TP all-reduce of the producer's tiles over peer memory
constexpr int kStageConv = 2;  // 3x3 "same" Conv2D as implicit GeMM (im2col TMA A operand)

// K-blocks per tcgen05.commit (flags bits 17-18: 1 -> 1, 2 -> 2, 3 -> 4; 0 -> default 1).
// One commit per K-block frees ring entries soonest; measured against 2 (scripts/flag_ab.py
// 17): equal or 1-3% faster on every chain (MLP B=256 146.5 -> 142.2 us, B=1024 headline
// 292 -> 286 us, attention S=512 147 -> 144.5 us); 4 per commit is 30% slower.
__host__ __device__ __forceinline__ int commit_group(int flags) {
  const int g = (flags >> 17) & 3;
  return g ? 1 << (g - 1) : 1;
}
// Ring-entry counter step without a division.
__device__ __forceinline__ int wrap_inc(int e, int n) { return e + 1 == n ? 0 : e + 1; }

struct StageParams {
  CUtensorMap tmap_a;  // activations [m, k] K-major, 128-B swizzle
  CUtensorMap tmap_b;  // weights [n, k] K-major, 128-B swizzle
  CUtensorMap tmap_a_half;  // two-pair clusters: activations, 64-row boxes (multicast halves)
  // split-K partial planes (chunked CTA-pair tiles): ws as fp32 [planes x 128 rows][tile
  // columns], 32-column x 128-row boxes, 128-B swizzle — the A operand of the reduction MMAs
  CUtensorMap tmap_ws;
  int red_mma;  // 1: tmap_ws is valid and split-K owners reduce on the tensor cores
  void* c;
  int m, n, k, ldc;
  int grid_x, grid_y;
  int order, order_stride;
  int epilogue;
  int k_blocks;
  int splits;    // split-K slices (the reference's z extent), >= 1
  float* ws;     // splits > 1: fp32 partial tiles [tiles][splits][BN][128]
  int* cnt;      // splits > 1: per-tile arrival counters (zero on entry and exit)
  int item_begin, item_end;
  int kind;    // kStageGemm or kStageDot
  int lda;     // activation leading dimension (elements), used by the dot stage
  const void* a;  // activations (dot stage reads them with generic loads)
  int in_dep;  // dependency feeding operand A, or -1
  int n_out_deps;
  int out_deps[TS_MAX_DEPS];
  // Last-arriver dot (fused mode): the dot stage's tiles are not claimed from the work
  // counter; the producer CTA whose post completes a dot tile's wait runs that tile
  // right away. `dot_dep` is this (producer) stage's dependency into such a dot stage.
  int dot_dep;       // producer side: dependency index, or -1
  int last_arriver;  // dot side: 1 when its tiles run on the last-arriving producer
  int wide;          // 1: two MMAs per K-block step (Cfg::kChunked): 2 x half_n columns
  int half_n;        // columns per MMA / accumulator slot: BN, or 192 (256 x 384 tiles)
  // kStageConv: NHWC input [conv_n, conv_h, conv_w, conv_cin] (tmap_a is an im2col map),
  // KRSC weights [n, 3, 3, conv_cin] (tmap_b over [n, 9 conv_cin]). K-block order:
  // input-channel tile (conv_subs x 64 channels) outer, filter tap, 64-channel sub-block
  // inner — a consumer k-step is one (producer column tile, tap) pair, as
  // Conv2DTileSync's k // kk map requires (policies.py:161-165). `halo` = producer row
  // tiles on each side a consumer tile's 3x3 window reaches (extra, untraced waits).
  int conv_h, conv_w, conv_cin, conv_subs, halo;
  // external row gates (ts_stage_desc.in_sem / out_sem): wait in_sem[tx] >= in_expected
  // before the first A load; add 1 to out_sem[tx] after the tile's stores
  int* in_sem;
  int in_expected;
  int* out_sem;
  int ar_cols;  // kStageAllReduce: columns of a tile (the producer's tile width)
  // last-wave balancing: the last tail_tiles tiles (claim order) run as tail_splits
  // split-K slices each; items = tiles - tail_tiles + tail_tiles * tail_splits
  int tail_tiles, tail_splits;
  // halo-staged convolution (TS_FLAG_CONV_HALO; Cin = Cout = 64, one CTA per 128-row
  // tile): the tile's input rows + 3x3 halo are loaded ONCE per tile into shared memory
  // (4-D TMA box, zero padding by out-of-bounds fill) and the nine tap-shifted A views are
  // UMMA descriptors offset by whole 128-B pixel rows; the layer's 9 weight taps stay
  // resident. hmode 1: a tile = 128 consecutive positions of one image in padded order
  // (row stride hs = W + 2, two junk columns per row); 2: a tile = 128 positions of one row
  // (hs = 130). 0: the im2col-per-tap path.
  int hmode, hs, htpi, htpr, hrows, hbytes;
  int hsub;  // 128-position sub-tiles per item (hmode 1: 2 when 256 positions' window fits)
  int hrpt;      // rows mode: image rows per tile (a tile = hrpt x hs positions)
  int hnb, hwin;  // window buffers in flight and their stride (bytes, 1024-aligned)
  CUtensorMap tmap_win;  // (C, W, H, N) box (64, hs, hrows, 1), 128-B swizzle
};

struct DepParams {
  int* sem;
  int policy, param;
  int pgx, pgy, pgz;    // producer grid (reference Stage.grid)
  int kb_per_kstep;     // consumer K-blocks per reference k-step
  int sem_n;
  int consumer;         // consumer stage index
  int producer;         // producer stage index
  int posts;            // producer posts in one launch (grid x*y*z): the done watermark
};

struct ChainParams {
  StageParams st[TS_MAX_STAGES];
  DepParams dep[TS_MAX_DEPS];
  int n_stages, n_deps, total_items;
  int item_lo, item_hi;  // this launch claims global items [item_lo, item_hi)
  int* scratch;
  // this launch's work / exit counters: scratch itself, or (co-resident mode: one launch
  // per stage on its own stream) the stage's block scratch + kCtlBase + kCtlInts * s,
  // whose [2] is the stage's "started" flag (stage.start())
  int* ctl;
  int coresident;
  int balanced;   // TS_FLAG_BALANCED: static stream-K assignment (0 = dynamic claims)
  int claim_batch;  // items per claim (> 1: one atomic per claim_batch items; set to 1)
  ts_trace_rec* trace;
  int trace_cap;
  int flags;
  int il_b1, il_b2;    // TS_FLAG_ROW_INTERLEAVE: items per row of stage 0 / 1 (0 = off)
  ts_peer_desc peers;  // kStageAllReduce: the tensor-parallel group
  int ar_done;         // tile halves every rank's owners finalize into this rank's buffer
};

// Tile geometry. Normal layout: UMMA M runs over activation rows (128 per CTA, 256 per
// CTA pair) and UMMA N = BN over weight rows. Swapped layout (SW, small batch): UMMA M
// runs over 128 weight rows and UMMA N = BN over activation rows, so every in-flight
// smem byte of the dominant operand is weight — the HBM-bound regime.
template <int BN, int CG, bool SW = false, bool QD = false>
struct Cfg {
  // CTA-pair 256-wide tiles stage operands through a ring of 16-KB chunks (one 128-row
  // x 64-K box each) instead of fixed slots, so a stage can use double-width tiles
  // (A + two B boxes per K-block, 256 x 512 outputs per pair): 25 % fewer operand bytes
  // per MAC, which is what bounds the 256 x 256 tile (L2 -> SM operand bandwidth).
  static constexpr bool kChunked = CG == 2 && BN == 256 && !SW;
  // Epilogue warps: 4 (one per TMEM lane quarter), or 8 for chunked tiles (two column
  // groups per lane quarter: a 256 x 512 tile's accumulator is single-buffered, so its
  // drain is on the MMA warp's critical path).
  // (QD: each pair's 256-column accumulator is double-buffered: 4 warps, 256 threads and
  // no register cap from a 384-thread CTA)
#ifndef TS_WIDE_EPI_GROUPS
#define TS_WIDE_EPI_GROUPS 2
#endif
  static constexpr int kEpiGroups = (kChunked && !QD) ? TS_WIDE_EPI_GROUPS : 1;
  static constexpr int kEpiThreads = 128 * kEpiGroups;
  static constexpr int kThreads = 128 + kEpiThreads;
  static constexpr int kChunkBytes = 16384;
  // One ring of 16-KB chunks, handed out in K-block order: a K-block takes its A chunk,
  // then one B chunk (two for a double-width tile), so 256 x 256 tiles keep 6 K-blocks
  // in flight and 256 x 512 tiles 4. (Separate 4-entry A / 8-entry B rings capped
  // 256 x 256 tiles at 4 K-blocks = 2048 MMA cycles of buffering, too little to cover
  // loaded HBM latency: 31-51% of the MMA floor against cuBLAS's 97% on the same tile.)
#ifndef TS_CHUNKS
#define TS_CHUNKS 12
#endif
  static constexpr int kChunks = TS_CHUNKS;
  static constexpr int kTileM = SW ? BN : 128 * CG;  // activation rows of a tile
  static constexpr int kTileN = SW ? 128 : BN;       // output columns of a tile
  static constexpr int kBRows = SW ? BN : BN / CG;   // rows of the UMMA-N operand per CTA
  static constexpr int kABytes = 128 * kBK * 2;      // UMMA-M operand stage
  static constexpr int kBBytes = kBRows * kBK * 2;   // UMMA-N operand stage
  static constexpr int kStageBytes = kABytes + kBBytes;
  // (single-CTA 64-wide kernels: 9 x 24 KB, so a halo-conv layer's windows get 144 KB next
  // to its 72 KB of resident weights)
  static constexpr bool kNarrow1 = !SW && CG == 1 && BN == 64;
  static constexpr int kStagesRaw = ((kNarrow1 ? 216 : 200) * 1024) / kStageBytes;
  static constexpr int kStagesMax = SW ? 12 : (kNarrow1 ? 9 : 8);
  static constexpr int kStages = kStagesRaw > kStagesMax ? kStagesMax : kStagesRaw;
  // Narrow swapped MMAs (128 x BN x 16, BN <= 64) are latency-bound when every one
  // accumulates into the same TMEM region; rotating over kAcc independent accumulators
  // (summed in the epilogue) keeps the tensor pipe busy.
  static constexpr int kAcc = SW ? (BN >= 256 ? 1 : 256 / BN > 8 ? 8 : 256 / BN) : 1;
  // (single-CTA 64-wide kernels: 128 columns, room for a halo-conv item's two sub-tiles)
  static constexpr int kAccCols =
      kAcc * BN * ((!kChunked && CG == 1 && !SW && BN == 64) ? 2 : 1);  // TMEM cols per buffer
  static constexpr int kTmemCols = 2 * kAccCols;       // two tile buffers
  static constexpr int kRing = kChunked ? kChunks : kStages;  // ring entries
  // chunked tiles: a 4-KB per-warp staging block after the ring turns the epilogue's
  // row-per-lane stores into 512-B coalesced ones (st.global from row-per-lane registers
  // touches 32 lines per instruction: measured ~25 GB/s per SM)
  static constexpr int kStageOff = kChunked ? kChunks * kChunkBytes : 0;
#ifndef TS_STAGE_WARP_BYTES
#define TS_STAGE_WARP_BYTES 4096
#endif
  // chunked tiles: a 4-KB tf32 identity (the B operand of the split-K reduction MMAs,
  // 32 x 32 for one CTA, this CTA's 16 rows of it for a pair) after the staging blocks
  // (chunked tiles: 2-KB blocks, half a warp's rows per pass, so that twelve ring chunks
  // and the identity fit: the eleven-chunk ring of an earlier build cost ~2% on the
  // 256 x 512 chains — three K-blocks in flight instead of four)
  static constexpr int kStageWarpBytes = kChunked ? 2048 : TS_STAGE_WARP_BYTES;
  static constexpr int kIdentOff = kStageOff + (kEpiThreads / 32) * kStageWarpBytes;
  static constexpr int kBarOffset = kChunked ? kIdentOff + 4096 : kStages * kStageBytes;
  // K-block full, commit-group empty; tmem full/empty x2; tile ring full/empty; peer_done
  // halo conv (hmode != 0, CG = 1, BN = 64): 9 weight taps (72 KB) then 2-4 window
  // buffers (StageParams::hnb x hwin bytes) in the (unused) operand ring
  static constexpr int kHaloRegion = kStages * kStageBytes;
  static constexpr bool kHaloOk = !kChunked && CG == 1 && !SW && BN == 64 &&
                                  9 * 8192 + 2 * 50176 <= kHaloRegion;
  static constexpr int kNumBars =
      kFullRing + kCommitRing + 4 + 2 * kTileRing + kPeerRing + 2 + 9 + 2 * kPostRing;
  // + tile ring ids, TMEM slot, flags and the last-arriver dot list (64 ints), ring-entry
  // owners (commit group that last read each entry)
  static constexpr int kSmemBytes =
      1024 + kBarOffset + kNumBars * 8 + 64 + 272 + 4 * kRing + 4 * kTileRing + 16 +
      4 * kPostRing;
  static_assert(kSmemBytes <= 227 * 1024, "shared memory budget");
  static_assert(kBRows % 8 == 0 && kBRows <= 256, "B box rows");
};

__device__ __forceinline__ int stage_of(const ChainParams& p, int g) {
  if (p.il_b1 > 0) return g % (p.il_b1 + p.il_b2) < p.il_b1 ? 0 : 1;
  int s = 0;
#pragma unroll 1
  while (s + 1 < p.n_stages && g >= p.st[s + 1].item_begin) ++s;
  return s;
}

__device__ __forceinline__ void trace_event(const ChainParams& p, uint64_t t, int kind,
                                            int stage, int tb, int k, int dep, int sem,
                                            int value, int x, int y, int z = 0) {
  if (p.trace == nullptr) return;
  int slot = atomicAdd(&p.scratch[2], 1);
  if (slot >= p.trace_cap) return;
  ts_trace_rec r;
  r.t_ns = t;
  r.kind = kind;
  r.stage = stage;
  r.tb = tb;
  r.k = k;
  r.dep = dep;
  r.sem = sem;
  r.value = value;
  r.x = static_cast<int16_t>(x);
  r.y = static_cast<int16_t>(y);
  r.z = static_cast<int16_t>(z);
  r.smid = static_cast<int16_t>(ptx::sm_id());
  r.clk = static_cast<int32_t>(clock64());  // SM cycles, for per-tile frequency
  p.trace[slot] = r;
}

// trace_event stamped now. The timer is read only when tracing: %globaltimer is an
// `asm volatile` read the compiler keeps even when trace_event returns at once, and two of
// them per consumer wait cost a fused conv pair ~8% (r02s3).
template <typename... A>
__device__ __forceinline__ void trace_now(const ChainParams& p, A... a) {
  if (p.trace == nullptr) return;
  trace_event(p, ptx::global_timer(), a...);
}

template <typename T>
struct AbFormat;
template <>
struct AbFormat<__half> {
  static constexpr uint32_t value = 0;
};
template <>
struct AbFormat<__nv_bfloat16> {
  static constexpr uint32_t value = 1;
};

__device__ __forceinline__ float relu(float x) { return fmaxf(x, 0.f); }

// GeLU in GPT-3's tanh form (GPT-2/3 "gelu_new"), with the hardware
// tanh: 0.5 x (1 + tanh(sqrt(2/pi) (x + 0.044715 x^3))).
__device__ __forceinline__ float gelu(float x) {
  const float u = x * fmaf(0.0356774081f, x * x, 0.7978845608f);
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(u));
  const float hx = 0.5f * x;
  return fmaf(hx, t, hx);
}

// Two GeLUs with one packed half-precision tanh (MUFU.TANH on f16x2: half the special-
// function issue slots of two f32 tanh.approx — the epilogue of a 256 x 512 tile runs
// 64 Ki GeLUs per CTA, which at 16 MUFU ops/clk/SM is ~4 K cycles with the f32 form).
// tanh's f16 rounding (<= 2^-11) is below the fp16/bf16 rounding of the stored output.
__device__ __forceinline__ void gelu2(float& a, float& b) {
  const float ua = a * fmaf(0.0356774081f, a * a, 0.7978845608f);
  const float ub = b * fmaf(0.0356774081f, b * b, 0.7978845608f);
  uint32_t h;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(ub), "f"(ua));  // hi = ub, lo = ua
  asm("tanh.approx.f16x2 %0, %0;" : "+r"(h));
  const __half2 t = *reinterpret_cast<const __half2*>(&h);
  const float ha = 0.5f * a, hb = 0.5f * b;
  a = fmaf(ha, __low2float(t), ha);
  b = fmaf(hb, __high2float(t), hb);
}

__device__ __forceinline__ float silu(float x) { return x / (1.0f + __expf(-x)); }

template <typename T>
__device__ __forceinline__ T to_elem(float v);
template <>
__device__ __forceinline__ __half to_elem<__half>(float v) {
  return __float2half_rn(v);
}
template <>
__device__ __forceinline__ __nv_bfloat16 to_elem<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}

template <typename T>
__device__ __forceinline__ uint32_t pack2(float a, float b);
template <>
__device__ __forceinline__ uint32_t pack2<__half>(float a, float b) {
  __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
template <>
__device__ __forceinline__ uint32_t pack2<__nv_bfloat16>(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// Spin until sem >= expected (the paper's wait_till, relaxed to >= so
// the semaphores stay monotone as in SemaphoreArray, policies.py:84-99). Exponential
// back-off keeps the polling traffic and issue slots of waiting SMs low.
__device__ __forceinline__ void sem_spin(const ChainParams& p, const int* sem, int expected) {
  // relaxed probes with back-off (an acquiring load per probe would invalidate L1 on
  // every iteration), then one acquiring load
  const bool watchdog = (p.flags & TS_FLAG_NO_WATCHDOG) == 0;
  // once a wait has timed out the launch is void: later waits return at once, so a
  // deadlocked launch (e.g. a co-resident consumer grid holding every SM) drains in one
  // watchdog period instead of one per wait
  if (watchdog && ptx::ld_relaxed_gpu(&p.scratch[3]) != 0) return;
  uint64_t t0 = ptx::global_timer();
  uint32_t ns = 32;
#pragma unroll 1
  while (ptx::ld_relaxed_gpu(sem) < expected) {
    __nanosleep(ns);
    if (ns < 256) ns <<= 1;
    if (watchdog && ptx::global_timer() - t0 > kWatchdogNs) {
      atomicExch(&p.scratch[3], 1);
      break;
    }
  }
  (void)ptx::ld_acquire_gpu(sem);
}

// sem_spin at system scope: a semaphore in a peer GPU's memory (all-reduce stage).
__device__ __forceinline__ void sem_spin_sys(const ChainParams& p, const int* sem, int expected) {
  const bool watchdog = (p.flags & TS_FLAG_NO_WATCHDOG) == 0;
  uint64_t t0 = ptx::global_timer();
  uint32_t ns = 32;
#pragma unroll 1
  while (ptx::ld_relaxed_sys(sem) < expected) {
    __nanosleep(ns);
    if (ns < 256) ns <<= 1;
    if (watchdog && ptx::global_timer() - t0 > kWatchdogNs) {
      atomicExch(&p.scratch[3], 1);
      break;
    }
  }
  (void)ptx::ld_acquire_sys(sem);
}

// Block until *s0 >= e0 and, for the optional extra semaphores (nullptr = none), *si >=
// ei. The first probes are acquiring loads issued back to back, so a satisfied wait
// costs one L2 round trip in the producer lane's critical path (two serialized loads
// per semaphore starved the MMA warp on short tiles). No arrays: they would live in
// local memory.
__device__ __forceinline__ void sem_wait5(const ChainParams& p, const int* s0, int e0,
                                          const int* s1 = nullptr, int e1 = 0,
                                          const int* s2 = nullptr, int e2 = 0,
                                          const int* s3 = nullptr, int e3 = 0,
                                          const int* s4 = nullptr, int e4 = 0) {
  const int v0 = ptx::ld_acquire_gpu(s0);
  const int v1 = s1 ? ptx::ld_acquire_gpu(s1) : 0;
  const int v2 = s2 ? ptx::ld_acquire_gpu(s2) : 0;
  const int v3 = s3 ? ptx::ld_acquire_gpu(s3) : 0;
  const int v4 = s4 ? ptx::ld_acquire_gpu(s4) : 0;
  if (v0 < e0) sem_spin(p, s0, e0);
  if (s1 && v1 < e1) sem_spin(p, s1, e1);
  if (s2 && v2 < e2) sem_spin(p, s2, e2);
  if (s3 && v3 < e3) sem_spin(p, s3, e3);
  if (s4 && v4 < e4) sem_spin(p, s4, e4);
}

__device__ __forceinline__ void sem_wait(const ChainParams& p, const int* sem, int expected) {
  sem_wait5(p, sem, expected);
}

// Producer-done watermark (extension, not a reference semantic): every producer post of
// dependency d also adds 1 to scratch[kDoneBase + d]. Once a consumer observes it at the
// dependency's total post count, every producer tile's stores are visible to it (the
// counter's release RMWs form one release sequence) and none of its later waits in this
// launch can block, so the producer lane stops probing semaphores for d. The counter is
// loaded together with the semaphores, so an unsatisfied watermark costs no extra round
// trip. Returns true when the watermark was reached.
constexpr int kDoneBase = 8;
// co-resident launches: stage s's work counter, exit counter and started flag at
// scratch[kCtlBase + kCtlInts * s + {0, 1, 2}] (TS_SCRATCH_INTS covers TS_MAX_STAGES)
constexpr int kCtlBase = 16;
constexpr int kCtlInts = 4;

__device__ __forceinline__ bool sem_wait_dep(const ChainParams& p, int d, const int* s0, int e0,
                                             const int* s1, int e1, const int* s2, int e2,
                                             const int* s3, int e3, const int* s4, int e4) {
  const int vd = ptx::ld_acquire_gpu(p.scratch + kDoneBase + d);
  const int v0 = ptx::ld_acquire_gpu(s0);
  const int v1 = s1 ? ptx::ld_acquire_gpu(s1) : 0;
  const int v2 = s2 ? ptx::ld_acquire_gpu(s2) : 0;
  const int v3 = s3 ? ptx::ld_acquire_gpu(s3) : 0;
  const int v4 = s4 ? ptx::ld_acquire_gpu(s4) : 0;
  if (vd >= p.dep[d].posts) return true;
  if (v0 < e0) sem_spin(p, s0, e0);
  if (s1 && v1 < e1) sem_spin(p, s1, e1);
  if (s2 && v2 < e2) sem_spin(p, s2, e2);
  if (s3 && v3 < e3) sem_spin(p, s3, e3);
  if (s4 && v4 < e4) sem_spin(p, s4, e4);
  return false;
}

template <typename T>
__device__ __forceinline__ void unpack8(const uint4& u, float (&f)[8]) {
  const T* h = reinterpret_cast<const T*>(&u);
#pragma unroll
  for (int j = 0; j < 8; ++j) f[j] = static_cast<float>(h[j]);
}

// The fused softmax-dot, two (row, head) items per warp instruction (lanes 0-15: item
// 2j, lanes 16-31: item 2j+1; 8 columns per lane), kDotBatch instruction pairs in flight:
// s = q*v over the head's 128 columns, p = softmax(s) (16-lane shuffle max and sum),
// out = p*k. Q, K, V are the head's column tiles at offsets h, heads + h and 2*heads + h
// (x128) of the QKV row, read through L2 (written by other SMs). All loads of a batch are
// issued before any is used: under a streaming GeMM the loaded L2 latency is ~1.5 us, and
// one item in flight made a 128 x 256 dot tile take ~40 us.
template <typename T, int kDotBatch>
__device__ __forceinline__ void dot_batch_warp(const StageParams& st, int row0, int hcount,
                                               int it0, int istep, int items, int h0,
                                               int lane) {
  const int heads = st.n / 128;
  const int half = lane >> 4, col = (lane & 15) * 8;
  uint4 qv[kDotBatch], kv[kDotBatch], vv[kDotBatch];
#pragma unroll
  for (int i = 0; i < kDotBatch; ++i) {
    const int it = it0 + i * istep + half;
    const int row = row0 + it / hcount;
    if (it < items && row < st.m) {
      const int h = h0 + it % hcount;
      const T* base = reinterpret_cast<const T*>(st.a) + static_cast<size_t>(row) * st.lda + col;
      qv[i] = __ldcg(reinterpret_cast<const uint4*>(base + h * 128));
      kv[i] = __ldcg(reinterpret_cast<const uint4*>(base + (heads + h) * 128));
      vv[i] = __ldcg(reinterpret_cast<const uint4*>(base + (2 * heads + h) * 128));
    }
  }
#pragma unroll
  for (int i = 0; i < kDotBatch; ++i) {
    const int it = it0 + i * istep + half;
    const int row = row0 + it / hcount;
    const bool ok = it < items && row < st.m;  // the two half-warps shuffle separately
    const T* q = reinterpret_cast<const T*>(&qv[i]);
    const T* k = reinterpret_cast<const T*>(&kv[i]);
    const T* v = reinterpret_cast<const T*>(&vv[i]);
    float sc[8], mx = -INFINITY;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      sc[j] = ok ? static_cast<float>(q[j]) * static_cast<float>(v[j]) : 0.f;
      mx = fmaxf(mx, sc[j]);
    }
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float sum = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      sc[j] = __expf(sc[j] - mx);
      sum += sc[j];
    }
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (!ok) continue;
    const float inv = 1.f / sum;
    const int h = h0 + it % hcount;
    uint32_t pk[4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
      pk[j] = pack2<T>(sc[2 * j] * inv * static_cast<float>(k[2 * j]),
                       sc[2 * j + 1] * inv * static_cast<float>(k[2 * j + 1]));
    T* out = reinterpret_cast<T*>(st.c) + static_cast<size_t>(row) * st.ldc + h * 128 + col;
    *reinterpret_cast<uint4*>(out) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
  }
}

// Split-K reduction of a normal tile, Z slices known at compile time: kS steps (4 rows x
// 32 columns of one 32-column chunk; lane l: row r0 + l / 8, columns (l % 8) * 4 .. + 4)
// with all kS x Z float4 loads in flight before any is summed — the loop is bound by L2
// latency under the MMA streams of the other SMs, so bytes in flight set its speed.
// emit(sidx, sum) stores step sidx.
template <int Z, int kS, typename Emit>
__device__ __forceinline__ void reduce_split_steps(const float* base, size_t zstride, int s0,
                                                   int sstride, int steps, int nr4, int lane,
                                                   uint64_t pol, Emit&& emit) {
  float4 v[kS][Z];
#pragma unroll
  for (int j = 0; j < kS; ++j) {
    const int sidx = s0 + j * sstride;
    const size_t off = (static_cast<size_t>(sidx / nr4) * 128 + (sidx % nr4) * 4) * 32 + lane * 4;
#pragma unroll
    for (int z = 0; z < Z; ++z)
      v[j][z] = sidx < steps ? ptx::ld_global_cg_f4_hint(base + z * zstride + off, pol)
                             : make_float4(0.f, 0.f, 0.f, 0.f);
  }
#pragma unroll
  for (int j = 0; j < kS; ++j) {
    const int sidx = s0 + j * sstride;
    if (sidx >= steps) break;
    float4 a = v[j][0];
#pragma unroll
    for (int z = 1; z < Z; ++z) {
      a.x += v[j][z].x;
      a.y += v[j][z].y;
      a.z += v[j][z].z;
      a.w += v[j][z].w;
    }
    emit(sidx, a);
  }
}

// diagnostic flag bit 12 (no semaphore waits) also skips the external row gates
__device__ __forceinline__ bool skip_in_gate(const ChainParams& p) { return (p.flags >> 12) & 1; }

struct Tile {
  int g, s, tb, tx, ty, tz;
  int z;  // split-K slices of this item's tile (st.splits, or tail_splits for a tail tile)
};

// Balanced (stream-K) schedule: the stage's flattened (tile in claim order, K-block) space
// is cut into `units` equal ranges of bal_width K-blocks; unit u runs [u w, (u + 1) w).
__device__ __forceinline__ int bal_width(const StageParams& st, int units) {
  const int total = st.grid_x * st.grid_y * st.k_blocks;
  return (total + units - 1) / units;
}

// A balanced item is the segment [kb0, kb1) of tile tb (packed (kb0 << 16) | kb1 in the
// tile ring). Role 0: the whole tile. Role 1 (kb0 > 0, the first item of its unit): writes
// an fp32 partial plane indexed by its unit and counts it into the tile half's counter; it
// does not post. Role 2 (the head: kb0 = 0, kb1 < k_blocks, the last item of its unit):
// waits for the planes of units ua..ub (every range that starts inside the tile), sums
// them into its TMEM accumulator, applies the epilogue, stores and posts once.

// Split-K slices of item g of stage st (see StageParams::tail_tiles).
__device__ __forceinline__ int item_slices(const StageParams& st, int tb) {
  if (st.tail_tiles > 0 && tb >= st.grid_x * st.grid_y - st.tail_tiles) return st.tail_splits;
  return st.splits;
}

// 32 packed 16-bit outputs (64 B) of one row: two 256-bit stores, or four 128-bit ones.
template <typename T>
__device__ __forceinline__ void store_row32(T* dst, const uint32_t (&pk)[16], bool v8ok) {
  if (v8ok) {
    ptx::st_global_v8(dst, pk);
    ptx::st_global_v8(dst + 16, pk + 8);
  } else {
    uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
    for (int q = 0; q < 4; ++q) d[q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
  }
}

__device__ __forceinline__ Tile decode(const ChainParams& p, int g) {
  Tile t;
  t.g = g;
  t.s = stage_of(p, g);
  const StageParams& st = p.st[t.s];
  t.tb = g - st.item_begin;
  if (p.il_b1 > 0) {
    // row-interleaved claims: row r = [b1 producer items | b2 consumer items]
    const int per = p.il_b1 + p.il_b2, r = g / per, j = g % per;
    t.tb = t.s == 0 ? r * p.il_b1 + j : r * p.il_b2 + (j - p.il_b1);
  }
  t.z = st.splits;
  const int base = st.grid_x * st.grid_y - st.tail_tiles;
  if (st.tail_tiles > 0 && t.tb >= base) {
    // tail tile (base + j / z), slice j % z
    const int j = t.tb - base;
    t.z = st.tail_splits;
    order_tile(st.order, st.order_stride, Grid3{st.grid_x, st.grid_y, 1}, base + j / t.z, &t.tx,
               &t.ty, &t.tz);
    t.tz = j % t.z;
    return t;
  }
  order_tile(st.order, st.order_stride, Grid3{st.grid_x, st.grid_y, st.splits}, t.tb, &t.tx,
             &t.ty, &t.tz);
  return t;
}

// Sum of one all-reduce tile's rows [r0, r0 + 128) over the group's buffers, stored back
// into every buffer (thread `tid` of `nthreads`). The peers' 16-byte vectors are staged
// with cp.async into `stage` (the operand ring, idle by the time an all-reduce item reaches
// the epilogue: every earlier GeMM item of this CTA has drained it and all later items
// are all-reduce items), up to 8 vectors x world per thread in flight without registers —
// the loop is bound by the latency of peer (NVLink) or HBM reads otherwise.
template <typename T>
__device__ __forceinline__ void allreduce_rows(const ChainParams& p, const StageParams& st, int r0,
                                               int ty, int tid, int nthreads, uint8_t* stage,
                                               int stage_bytes) {
  const int world = p.peers.world;
  const int rows = st.m - r0 < 128 ? st.m - r0 : 128;
  const int vpr = st.ar_cols / 8;  // 16-byte vectors per tile row
  const int total = rows > 0 ? rows * vpr : 0;
  const size_t base = static_cast<size_t>(r0) * st.ldc + static_cast<size_t>(ty) * st.ar_cols;
  const int slots = stage_bytes / (16 * nthreads) / world;  // vectors per thread in flight
  const int nb = slots > 8 ? 8 : (slots < 1 ? 1 : slots);
  uint4* sv = reinterpret_cast<uint4*>(stage);  // slot (i * world + q) * nthreads + tid
  auto offset = [&](int v) {
    return base + static_cast<size_t>(v / vpr) * st.ldc + (v % vpr) * 8;
  };
#pragma unroll 1
  for (int v0 = 0; v0 < total; v0 += nb * nthreads) {
#pragma unroll 1
    for (int i = 0; i < nb; ++i) {
      const int v = v0 + i * nthreads + tid;
      if (v >= total) break;
      const size_t off = offset(v);
#pragma unroll 1
      for (int q = 0; q < world; ++q)
        ptx::cp_async16(ptx::smem_u32(&sv[(i * world + q) * nthreads + tid]),
                        reinterpret_cast<const T*>(p.peers.bufs[q]) + off);
    }
    ptx::cp_async_wait_all();  // this thread's own slots only
#pragma unroll 1
    for (int i = 0; i < nb; ++i) {
      const int v = v0 + i * nthreads + tid;
      if (v >= total) break;
      float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll 1
      for (int q = 0; q < world; ++q) {
        float f[8];
        unpack8<T>(sv[(i * world + q) * nthreads + tid], f);
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] += f[j];
      }
      const uint4 o = make_uint4(pack2<T>(a[0], a[1]), pack2<T>(a[2], a[3]), pack2<T>(a[4], a[5]),
                                 pack2<T>(a[6], a[7]));
      const size_t off = offset(v);
#pragma unroll 1
      for (int q = 0; q < world; ++q)
        *reinterpret_cast<uint4*>(reinterpret_cast<T*>(p.peers.bufs[q]) + off) = o;
    }
  }
}

// QD: clusters of two CTA pairs (4 CTAs). A work item is a 256 x 512 tile (the reference
// tile of a double-width stage); pair p of the cluster computes its output columns
// [256 p, 256 p + 256) as a 256 x 256 cta_group::2 tile with its own double-buffered TMEM
// accumulator. Both pairs read the same 256 activation rows: every CTA loads 64 of its
// 128 rows and multicasts them to the same-half CTA of the other pair, so each SM pulls
// 24 KB of operands per 64-deep K-block instead of 32 KB (L2 -> SM bandwidth is what
// bounds unicast 256 x 256 tiles), while the epilogue of one tile overlaps the MMAs of the
// next (a 256 x 512 tile on one pair fills all of TMEM). Ring entries are freed by both
// pairs' MMA commits (empty barriers count 2); the cluster leader claims items, hands the
// id to the other three CTAs and posts once all four have stored.
// Halo-staged convolution geometry (StageParams::hmode). For tile tx: image n, first
// image row h0, first padded column w0 and the A base pixel inside the window buffer
// (the window starts at padded column 0 / w0 - 1 of image row h0 - 1).
struct HaloTile {
  int n, h0, w0, base;
};

__device__ __forceinline__ HaloTile halo_tile(const StageParams& st, int tx) {
  HaloTile h;
  h.n = tx / st.htpi;
  const int lt = tx - h.n * st.htpi;
  if (st.hmode == 1) {
    h.h0 = lt * st.hrpt;
    h.w0 = 0;
    h.base = 0;
  } else {
    const int rt = lt / st.htpr;  // row group (hrpt image rows) of the tile
    h.h0 = rt * st.hrpt;
    h.w0 = (lt - rt * st.htpr) * 128;
    h.base = 0;
  }
  return h;
}

// Output pixel of accumulator row m of halo tile `ht` (or -1: a junk position of the
// padded order / past the image edge).
__device__ __forceinline__ int halo_pixel(const StageParams& st, const HaloTile& ht, int m) {
  int h, w;
  if (st.hmode == 1) {
    if (m >= st.hrpt * st.hs) return -1;  // rows of the tile: hrpt x hs positions
    h = ht.h0 + m / st.hs;
    w = m % st.hs;
  } else {
    // sub-tile m / 128 = image row h0 + m / 128 of the segment
    h = ht.h0 + (m >> 7);
    w = ht.w0 + (m & 127);
  }
  if (h >= st.conv_h || w >= st.conv_w) return -1;
  return (ht.n * st.conv_h + h) * st.conv_w + w;
}

// Split-K owner, producer side: wait until the other slices' fp32 partial planes of this
// CTA's rows are written, then stream them in as 32-column x 128-row boxes (the A operand
// of the tensor-core reduction D += P x I), one ring chunk and one commit group per box.
// Out of line: the scheduler lane is the kernel's tightest register budget.
template <int CG, typename C>
__device__ __noinline__ void owner_plane_loads(const ChainParams& p, const StageParams& st,
                                               const Tile& t, int rank, bool leader,
                                               uint32_t plead, int acc_cols, uint8_t* smem,
                                               uint64_t* full, uint64_t* empty, int* owner,
                                               int& ea, uint32_t& kq, uint32_t& cid,
                                               uint64_t pol) {
  constexpr int R = C::kRing;
  const int half_id = (t.tx * st.grid_y + t.ty) * CG + rank;
  int* rdy = st.cnt + st.grid_x * st.grid_y * CG + half_id;
  sem_spin(p, rdy, t.z - 1);
  *rdy = 0;  // every writer has counted: restore the zero invariant
  ptx::fence_proxy_async_global();
  const int groups = acc_cols / 32;
#pragma unroll 1
  for (int pz = 0; pz < t.z - 1; ++pz) {
#pragma unroll 1
    for (int j = 0; j < groups; ++j) {
      const int e = ea;
      const int o = owner[e];
      if (o >= 0) {
        const uint32_t uo = static_cast<uint32_t>(o);
        ptx::mbar_wait(&empty[uo % kCommitRing], (uo / kCommitRing) & 1);
      }
      owner[e] = static_cast<int>(cid);
      ea = wrap_inc(ea, R);
      uint64_t* fb = &full[kq % kFullRing];
      if (leader) ptx::mbar_arrive_expect_tx(fb, CG * C::kChunkBytes);
      const int prow = (half_id * t.z + pz) * 128;
      if constexpr (CG == 2) {
        ptx::tma_load_2d_pair(smem + e * C::kChunkBytes, &st.tmap_ws, ptx::mapa(fb, plead),
                              j * 32, prow, pol);
      } else {
        ptx::tma_load_2d(smem + e * C::kChunkBytes, &st.tmap_ws, fb, j * 32, prow, pol);
      }
      ++kq;
      ++cid;
    }
  }
}

template <int BN, int CG, typename T, bool SW, bool QD = false>
__global__ void __launch_bounds__(Cfg<BN, CG, SW, QD>::kThreads, 1)
    chain_kernel(const __grid_constant__ ChainParams p) {
  using C = Cfg<BN, CG, SW, QD>;
  static_assert(!QD || (CG == 2 && BN == 256 && !SW), "two-pair clusters: 256-wide CTA pairs");
  constexpr int NP = QD ? 2 : 1;  // CTA pairs per cluster
  constexpr int kEpiThreads = C::kEpiThreads;
  constexpr int kEpiWarps = kEpiThreads / 32;
  static_assert(!SW || CG == 1, "swapped tiles use single-CTA MMAs");
  constexpr int S = C::kStages;
  constexpr int R = C::kRing;  // smem ring entries (slots, or chunks when kChunked)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;                       // S x [128 x 64]
  uint8_t* sB = smem + S * C::kABytes;      // S x [BN/CG x 64]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kBarOffset);
  uint64_t* full = bars;               // [kFullRing], by K-block sequence number
  uint64_t* empty = bars + kFullRing;  // [kCommitRing], by commit group
  uint64_t* tmem_full = empty + kCommitRing;
  uint64_t* tmem_empty = tmem_full + 2;
  uint64_t* ti_full = tmem_empty + 2;
  uint64_t* ti_empty = ti_full + kTileRing;
  uint64_t* peer_done = ti_empty + kTileRing;
  uint64_t* dot_msg = peer_done + kPeerRing;  // peer CTA: leader's list of released dot tiles
  uint64_t* dot_done = dot_msg + 1;           // leader: peer finished its half of them
  // halo conv: weights landed, window landed [2], window consumed by the MMAs [2]
  uint64_t* hw_full = dot_done + 1;
  uint64_t* win_full = hw_full + 1;    // [4]
  uint64_t* win_empty = win_full + 4;  // [4]
  uint64_t* post_full = win_empty + 4;           // [kPostRing]: a post request is queued
  uint64_t* post_empty = post_full + kPostRing;  // [kPostRing]: the post warp took it
  int* ti_item = reinterpret_cast<int*>(post_empty + kPostRing);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ti_item + kTileRing);
  int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);
  int* split_flag = last_flag + 1;
  int* dot_count = split_flag + 1;  // last-arriver dot tiles released by a post
  int* dot_list = dot_count + 1;    // [0, 32): dot tile columns, [32, 64): their tb
  int* owner = dot_list + 64;       // [R]: commit group that last read each ring entry
  int* ti_kb = owner + R;           // [kTileRing]: balanced segment K range per ring slot
  int* bst = ti_kb + kTileRing;     // [3]: balanced scheduler state (stage, next, end)
  int* post_req = bst + 4;          // [kPostRing]: item ids queued for the post warp
  const bool bal = p.balanced != 0;
  // single-CTA kernels: the post warp takes the posts when a stage of this launch posts
  // and the launch has at least four items per CTA (a short launch is latency-bound: the
  // hand-off to another warp delays the consumer; measured +0.6-1 us at B <= 8)
  bool any_post = false;
  if constexpr (CG == 1) {
    for (int s = 0; s < p.n_stages; ++s) any_post |= p.st[s].n_out_deps > 0;
    any_post = any_post && p.item_hi - p.item_lo >= 4 * static_cast<int>(gridDim.x);
  }
  const int unit = static_cast<int>(blockIdx.x) / (CG * NP);  // this CTA's work unit
  const int units = static_cast<int>(gridDim.x) / (CG * NP);  // all co-resident (host cap)

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t qrank = CG == 2 ? ptx::cluster_rank() : 0;  // rank in the cluster
  // (compile-time 0 / identities without QD, so one-pair kernels keep their registers)
  const uint32_t rank = QD ? (qrank & 1) : qrank;     // CTA within its pair (row half)
  const uint32_t pair = QD ? (qrank >> 1) : 0;        // pair within the cluster (column half)
  const uint32_t plead = QD ? (qrank & ~1u) : 0;      // this pair's leader
  const bool leader = rank == 0;                      // pair leader: MMA issuer, TMEM owner
  const bool uleader = QD ? qrank == 0 : leader;      // cluster leader: scheduler, posts

  if (threadIdx.x == 0) {
    for (int i = 0; i < kFullRing; ++i) ptx::mbar_init(&full[i], 1);
    for (int i = 0; i < kCommitRing; ++i) ptx::mbar_init(&empty[i], NP);  // every pair's commit
    for (int i = 0; i < R; ++i) owner[i] = -1;
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&tmem_full[i], 1);
      ptx::mbar_init(&tmem_empty[i], CG * kEpiWarps);
    }
    for (int i = 0; i < kPeerRing; ++i)
      ptx::mbar_init(&peer_done[i], NP * CG > 1 ? NP * CG - 1 : 1);  // the other CTAs' stores
    ptx::mbar_init(dot_msg, 1);
    ptx::mbar_init(dot_done, 1);
    ptx::mbar_init(hw_full, 1);
    for (int i = 0; i < 4; ++i) {
      ptx::mbar_init(&win_full[i], 1);
      ptx::mbar_init(&win_empty[i], 1);
    }
    for (int i = 0; i < kPostRing; ++i) {
      ptx::mbar_init(&post_full[i], 1);
      ptx::mbar_init(&post_empty[i], 1);
    }
    for (int i = 0; i < kTileRing; ++i) {
      ptx::mbar_init(&ti_full[i], 1);
      // every pair's MMA warp + every epilogue warp of the cluster + the other CTAs'
      // producer lanes
      ptx::mbar_init(&ti_empty[i], NP + NP * CG * kEpiWarps + (NP * CG - 1));
    }
    *dot_count = 0;
    ptx::fence_barrier_init();
  }
  if constexpr (C::kChunked && !QD) {
    // tf32 identity rows of this CTA (K-major, 128-B swizzle: element (n, k) of an 8-row
    // group at n * 128 + ((k / 4) ^ (n & 7)) * 16 + (k % 4) * 4); a CTA pair's B operand
    // of N = 32 is split by rows: rank r holds rows [16 r, 16 r + 16)
    float* id = reinterpret_cast<float*>(smem + C::kIdentOff);
    for (int i = threadIdx.x; i < 1024; i += C::kThreads) {
      const int n = i >> 5, k = i & 31;
      const int ng = (CG == 2 ? 16 * static_cast<int>(rank) : 0) + n;  // global N row
      id[(n * 128 + (((k >> 2) ^ (n & 7)) << 4) + ((k & 3) << 2)) >> 2] = (k == ng) ? 1.f : 0.f;
    }
    ptx::fence_proxy_async_shared();
  }
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < p.n_stages; ++s) {
      if (p.st[s].kind == kStageDot || p.st[s].kind == kStageAllReduce)
        continue;  // pointwise stages have no tensor maps
      ptx::tma_prefetch_desc(&p.st[s].tmap_a);
      ptx::tma_prefetch_desc(&p.st[s].tmap_b);
    }
  }
  // stage.start(): a co-resident launch marks its stage as started,
  // which releases the wait kernel on the consumer stage's stream
  if (p.coresident && threadIdx.x == 0) atomicExch(&p.ctl[2], 1);
  __syncthreads();  // barrier init (thread 0) before the allocator warp writes tmem_slot
  if (warp == 2) ptx::tmem_alloc<C::kTmemCols, CG>(tmem_slot);
  ptx::tc_fence_before();
  if constexpr (CG == 2) {
    ptx::cluster_sync();
  } else {
    __syncthreads();
  }
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // Receive the next tile id from the ring (and release the slot).
  auto ring_take = [&](int it, bool remote_release, int& kbr) -> int {
    const int slot = it % kTileRing;
    if constexpr (CG == 2) {
      ptx::mbar_wait_cluster(&ti_full[slot], (it / kTileRing) & 1);
    } else {
      ptx::mbar_wait(&ti_full[slot], (it / kTileRing) & 1);
    }
    // CTA pairs: lane 0 reads the id and is the lane that releases the slot, the others get
    // it by shuffle (no lane's shared-memory read ordered only through another lane's
    // arrive; measured +4% on the B=1024 pair chain). Single CTAs keep the warp-wide read
    // (the shuffle measured 7-10% slower on ResNet 8x28x28x128).
    int g;
    if constexpr (CG == 2) {
      g = lane == 0 ? ti_item[slot] : 0;
      kbr = lane == 0 ? ti_kb[slot] : 0;
      g = __shfl_sync(0xffffffffu, g, 0);
      kbr = __shfl_sync(0xffffffffu, kbr, 0);
    } else {
      g = ti_item[slot];
      kbr = ti_kb[slot];
      __syncwarp();
    }
    if (lane == 0) {
      if (remote_release) {
        ptx::mbar_arrive_remote(ptx::mapa(&ti_empty[slot], 0));
      } else {
        ptx::mbar_arrive(&ti_empty[slot]);
      }
    }
    return g;
  };

  if (warp == 0) {
    // ===================== scheduler + TMA producer =====================
    if (lane == 0) {
      const bool reorder = (p.flags & TS_FLAG_NO_REORDER) == 0;
      // L2 hints: activations (A) are re-read by every column tile -> evict_last.
      // Weights (B) are re-read by every row tile of the same column; they stream once
      // only when the stage has a single row of tiles -> evict_first there.
      const uint64_t pol_first = ptx::policy_evict_first();
      const uint64_t pol_normal = ptx::policy_evict_normal();
      const uint64_t pol_last = ptx::policy_evict_last();
      const int b_hint = (p.flags >> 8) & 3;
      // ring entries: ea = next A entry (slot, or A chunk), eb = next B chunk (chunked)
      int ea = 0;         // next ring entry (slot, or chunk when kChunked)
      uint32_t kq = 0;    // K-blocks issued (full barrier index)
      uint32_t cid = 0;   // commit group of the K-block being issued
      const int group = commit_group(p.flags);
      uint32_t done_mask = 0;  // dependencies whose producer-done watermark was observed
      // Claim ring entry e for commit group `cid` once the MMAs of the group that last
      // read it are done.
      auto claim = [&](int e) {
        const int o = owner[e];
        if (o >= 0) {
          const uint32_t uo = static_cast<uint32_t>(o);
          ptx::mbar_wait(&empty[uo % kCommitRing], (uo / kCommitRing) & 1);
        }
        owner[e] = static_cast<int>(cid);
      };
      int hi = 0, pw_stage = -1;  // halo conv: windows issued, stage of the resident weights
      int cb_next = 0, cb_left = 0;  // claim batching (halo-conv kernels)
      // balanced schedule state (shared memory: the scheduler lane's registers are the
      // kernel's tightest): stage, next and end position in the stage's flattened space
      if (bal) {
        bst[0] = 0;
        bst[1] = -1;
        bst[2] = 0;
      }
#pragma unroll 1
      for (int it = 0;; ++it) {
        int g, kbr = 0;
        const int slot = it % kTileRing;
        if (uleader) {
          ptx::mbar_wait(&ti_empty[slot], ((it / kTileRing) & 1) ^ 1);  // no data: slot reuse
          if (bal) {
            // static stream-K assignment: this unit's K-block range of each stage in turn,
            // cut at tile boundaries (the first segment may start inside a tile, the last
            // may end inside one)
            g = -1;
            int bs = bst[0], bpos = bst[1], bend = bst[2];
            while (bs < p.n_stages) {
              const StageParams& sb = p.st[bs];
              const int kbs = sb.k_blocks;
              if (bpos < 0) {
                const int total = sb.grid_x * sb.grid_y * kbs;
                const int w = bal_width(sb, units);
                bpos = unit * w;
                bend = bpos + w < total ? bpos + w : total;
              }
              if (bpos < bend) {
                const int tile = bpos / kbs, k0 = bpos % kbs;
                const int k1 = kbs < k0 + (bend - bpos) ? kbs : k0 + (bend - bpos);
                g = sb.item_begin + tile;
                kbr = (k0 << 16) | k1;
                bpos += k1 - k0;
                break;
              }
              ++bs;
              bpos = -1;
            }
            bst[0] = bs;
            bst[1] = bpos;
            bst[2] = bend;
          } else if (C::kHaloOk && p.claim_batch > 1) {
            // short halo-conv tiles: one claim RMW (a loaded L2 round trip in the
            // scheduler lane) per claim_batch consecutive items
            if (cb_left == 0) {
              cb_next = p.item_lo + atomicAdd(&p.ctl[0], p.claim_batch);
              cb_left = p.claim_batch;
            }
            g = cb_next < p.item_hi ? cb_next : -1;
            ++cb_next;
            --cb_left;
            if (g < 0) cb_left = 0;
          } else {
            g = p.item_lo + atomicAdd(&p.ctl[0], 1);
            if (g >= p.item_hi) g = -1;
          }
          ti_item[slot] = g;
          ti_kb[slot] = kbr;
          ptx::mbar_arrive(&ti_full[slot]);
          if constexpr (CG == 2) {
#pragma unroll
            for (int r = 1; r < NP * CG; ++r) {
              ptx::st_cluster_u32(ptx::mapa(&ti_item[slot], r), static_cast<uint32_t>(g));
              ptx::st_cluster_u32(ptx::mapa(&ti_kb[slot], r), static_cast<uint32_t>(kbr));
              ptx::mbar_arrive_remote(ptx::mapa(&ti_full[slot], r));
            }
          }
        } else {
          ptx::mbar_wait_cluster(&ti_full[slot], (it / kTileRing) & 1);
          g = ti_item[slot];
          kbr = ti_kb[slot];
          ptx::mbar_arrive_remote(ptx::mapa(&ti_empty[slot], 0));
        }
        if (g < 0) break;
        const Tile t = decode(p, g);
        const StageParams& st = p.st[t.s];
        if (uleader)
          trace_now(p, 0, t.s, t.tb, -1, -1, -1, -1, t.tx, t.ty, t.tz);
        if (st.kind == kStageDot || st.kind == kStageAllReduce)
          continue;  // pointwise stages: the epilogue warps run them
        if constexpr (C::kHaloOk) {
          if (st.hmode) {
            // (1) the stage's nine weight taps, resident for all its tiles: reload once the
            // MMAs of every earlier window (the old weights' readers) have completed
            if (t.s != pw_stage) {
              for (int j = hi - st.hnb; j < hi; ++j)
                if (j >= 0) ptx::mbar_wait(&win_empty[j % st.hnb], (j / st.hnb) & 1);
              ptx::mbar_arrive_expect_tx(hw_full, 9 * 8192);
              for (int tap = 0; tap < 9; ++tap)
                ptx::tma_load_2d(smem + tap * 8192, &st.tmap_b, hw_full, tap * kBK, t.ty * 64,
                                 ptx::policy_evict_last());
              pw_stage = t.s;
            }
            const HaloTile ht = halo_tile(st, t.tx);
            // (2) stage.wait(): the producer tiles whose rows the window covers (the
            // reference's Conv2DTileSync wait of k-step 0 is tile tx itself; the 3x3 halo
            // rows ride along untraced)
            const int d = st.in_dep;
            if (d >= 0 && !((p.flags >> 12) & 1)) {
              const DepParams& dp = p.dep[d];
              if (uleader)
                trace_now(p, 1, t.s, t.tb, 0, d, t.tx, dp.pgz, t.tx, t.ty, t.tz);
              const int base_t = ht.n * st.htpi;
              // producer tiles [u, u + n) (contiguous semaphores), probed five at a time in
              // one round trip (one sem_wait_dep per tile serialized 2-6 loaded-L2 round
              // trips per item until the producer-done watermark was seen)
              auto wait_range = [&](int u, int n) {
                for (; n > 0 && !((done_mask >> d) & 1); u += 5, n -= 5) {
                  const int* s0 = dp.sem + u;
                  if (sem_wait_dep(p, d, s0, dp.pgz, n > 1 ? s0 + 1 : nullptr, dp.pgz,
                                   n > 2 ? s0 + 2 : nullptr, dp.pgz, n > 3 ? s0 + 3 : nullptr,
                                   dp.pgz, n > 4 ? s0 + 4 : nullptr, dp.pgz))
                    done_mask |= 1u << d;
                }
              };
              const int hlo = ht.h0 > 0 ? ht.h0 - 1 : 0;
              const int hhi0 = ht.h0 + st.hrpt;  // last input row the window reads
              const int hhi = hhi0 < st.conv_h - 1 ? hhi0 : st.conv_h - 1;
              if (st.hmode == 1) {
                wait_range(base_t + hlo / st.hrpt, hhi / st.hrpt - hlo / st.hrpt + 1);
              } else {
                const int s0 = ht.w0 > 0 ? (ht.w0 - 1) / 128 : 0;
                const int s1 = (ht.w0 + 128 < st.conv_w - 1 ? ht.w0 + 128 : st.conv_w - 1) / 128;
                for (int rg = hlo / st.hrpt; rg <= hhi / st.hrpt; ++rg)
                  wait_range(base_t + rg * st.htpr + s0, s1 - s0 + 1);
              }
              if (uleader)
                trace_now(p, 2, t.s, t.tb, 0, d, t.tx, dp.pgz, t.tx, t.ty, t.tz);
              ptx::fence_proxy_async_global();
            }
            // (3) the window: input rows h0 - 1 .. h0 + hrows - 2 (+ halo columns), once
            const int b = hi % st.hnb;
            if (hi >= st.hnb) ptx::mbar_wait(&win_empty[b], ((hi / st.hnb) & 1) ^ 1);
            ptx::mbar_arrive_expect_tx(&win_full[b], st.hbytes);
            ptx::tma_load_4d(smem + 9 * 8192 + b * st.hwin, &st.tmap_win, &win_full[b], 0,
                             st.hmode == 1 ? -1 : ht.w0 - 1, ht.h0 - 1, ht.n,
                             ptx::policy_evict_normal());
            ++hi;
            continue;
          }
        }
        // activation (dependent) and weight (independent) tile rows of this CTA
        const int act_row = SW ? t.tx * BN : t.tx * C::kTileM + static_cast<int>(rank) * 128;
        // a double-width tile's second B box (output columns [BN, 2 BN) of the pair
        // tile) starts BN weight rows further; each CTA holds its 128-row half of both
        // QD: a double-width tile runs as one 256-wide MMA tile per pair (no second B box)
        const int wide = (C::kChunked && !QD) ? st.wide : 0;
        const int hn = C::kChunked ? st.half_n : BN;  // columns per MMA
        const int w_row = SW ? t.ty * 128
                             : t.ty * (hn << (QD ? 1 : wide)) + static_cast<int>(pair) * hn +
                                   static_cast<int>(rank) * (hn / CG);
        const int d = st.in_dep;
        const int bh = b_hint ? b_hint : (st.grid_x == 1 ? 1 : 2);
        const uint64_t pol_b = bh == 1 ? pol_first : (bh == 2 ? pol_normal : pol_last);
        const int ah = (p.flags >> 10) & 3;
        const uint64_t pol_a = ah == 1 ? pol_first : (ah == 2 ? pol_normal : pol_last);
        // diagnostic only (flag bit 12): time the chain without semaphore waits
        const bool no_wait = (p.flags >> 12) & 1;
        // K-blocks of this split-K slice, or of this balanced segment
        const int k_per = bal ? (kbr & 0xffff) - (kbr >> 16) : st.k_blocks / t.z;
        const int kb_begin = bal ? kbr >> 16 : t.tz * k_per;
        const int kb_end = kb_begin + k_per;
        // stage.wait() for reference k-step `ks` (policies.py:145-166)
        auto wait_kstep = [&](int ks) {
          const DepParams& dp = p.dep[d];
          const Grid3 pg{dp.pgx, dp.pgy, dp.pgz};
          // the producer-done watermark was observed (and fenced) earlier in this launch:
          // every wait of d is satisfied, and the fence after that observation orders all
          // later TMA reads of this thread (traced launches still record the wait events)
          if (((done_mask >> d) & 1) && p.trace == nullptr) return;
          Wait w = consumer_wait(dp.policy, dp.param, t.tx, t.ty, ks, pg, dp.pgz);
          if (w.sem < 0) return;
          if (uleader)
            trace_now(p, 1, t.s, t.tb, ks, d, w.sem, w.expected, t.tx,
                        t.ty, t.tz);
          // Halo (extension): a 3x3 window of output rows [m0, m0 + tile_m) reads input
          // pixels up to W + 1 rows away, i.e. the same k-step's producer tiles of
          // neighbouring row tiles; the reference map names only row tx. Those waits ride
          // along untraced (their wait_end is not an event of the reference model).
          // halo rows tx-2 .. tx+2 (halo <= 2, checked on the host)
          auto halo_sem = [&](int dx, int& e) -> const int* {
            const int x = t.tx + dx;
            if (dx < -st.halo || dx > st.halo || x < 0 || x >= dp.pgx) return nullptr;
            const Wait h = consumer_wait(dp.policy, dp.param, x, t.ty, ks, pg, dp.pgz);
            e = h.expected;
            return h.sem >= 0 ? dp.sem + h.sem : nullptr;
          };
          int e1 = 0, e2 = 0, e3 = 0, e4 = 0;
          const int* h1 = halo_sem(-1, e1);
          const int* h2 = halo_sem(1, e2);
          const int* h3 = halo_sem(-2, e3);
          const int* h4 = halo_sem(2, e4);
          if ((p.flags >> 23) & 1)  // diagnostic flag bit 23: no watermark
            sem_wait5(p, dp.sem + w.sem, w.expected, h1, e1, h2, e2, h3, e3, h4, e4);
          else if (!((done_mask >> d) & 1) &&
                   sem_wait_dep(p, d, dp.sem + w.sem, w.expected, h1, e1, h2, e2, h3, e3, h4, e4))
            done_mask |= 1u << d;
          if (uleader)
            trace_now(p, 2, t.s, t.tb, ks, d, w.sem, w.expected, t.tx,
                        t.ty, t.tz);
          ptx::fence_proxy_async_global();
        };
        // conv: the first output pixel of this CTA's rows, as NHW coordinates
        const bool conv = st.kind == kStageConv;
        int cq = 0, cp = 0, cn = 0;
        if (conv) {
          cq = act_row % st.conv_w;
          cp = (act_row / st.conv_w) % st.conv_h;
          cn = act_row / (st.conv_w * st.conv_h);
        }
        if (st.in_sem != nullptr && !skip_in_gate(p)) {
          // external gate: the rows of this tile were copied in (ts_stream_signal)
          sem_wait(p, st.in_sem + t.tx, st.in_expected);
          ptx::fence_proxy_async_global();
        }
        const bool waits = d >= 0 && !no_wait;
        const int kbpk = waits ? p.dep[d].kb_per_kstep : 1;
        // K-loop rotation. At small batch every tile reads the same few activation lines
        // for a given K-block; if all tiles walked K in the same order they would hit one
        // L2 line at a time (measured: 1.9 TB/s instead of 6.4). Starting each weight
        // column block at a different K-block spreads those reads while tiles sharing a
        // weight block (same ty) stay in lockstep for L2 reuse. Allowed when the policy
        // has no k-step ordering to respect (no dependency, or a single wait at k-step 0).
        const bool ordered = waits && !(p.dep[d].policy == kRow || p.dep[d].policy == kStrided);
        const int rot = (ordered || conv || (p.flags >> 14) & 1) ? 0 : (t.ty * 37 + 5) % k_per;
        // Deep "+R": a Row/Strided consumer waits once (k-step 0) before any activation
        // load, so it issues the weight boxes of as many K-blocks as the ring holds first,
        // then waits, then issues their activation boxes — the weights stream while the
        // producer rows finish (flag bit 21 disables it).
        const int per_kb = C::kChunked ? 2 + wide : 1;  // ring entries per K-block
        const int cap = R / per_kb;
        // Ordered policies (Tile, Conv2D) defer the waits of the k-steps inside the first
        // `pre` K-blocks the same way (their later k-steps wait inline), which hides the
        // loaded latency of a satisfied wait (~2 us of L2 round trip) behind weight loads.
        // Only for Row/Strided consumers (one wait, at k-step 0). Not for convolution
        // consumers — their im2col A boxes are the heavy operand and front-loading the small
        // weight boxes delayed them (flag bit 21: ResNet 8x56x56x64 39.7 -> 33.0 us,
        // 32x56x56x64 107 -> 90 us) — nor for ordered (Tile/Conv2D) GeMM consumers, where
        // deferring the first waits cost 1-5% (TileSync MLP B=1024 341 vs 336 us, attention
        // S=512 153 vs 147 us).
        const bool deep = waits && reorder && !conv && !((p.flags >> 21) & 1) &&
                          (p.dep[d].policy == kRow || p.dep[d].policy == kStrided);
        const int pre = deep ? (k_per < cap ? k_per : cap) : 0;
        const int ea_start = ea;
        const uint32_t kq_start = kq;
        auto all_waits = [&]() {
          // every wait of the slice (only k-step 0 waits for Row/Strided)
          for (int ks = 0; ks * kbpk < st.k_blocks; ++ks) wait_kstep(ks);
        };
        // conv: K-block kb = (channel tile, tap, 64-channel sub-block)
        // returns (c0 << 4) | tap
        auto conv_coords = [&](int kb) -> int {
          const int per_tile = 9 * st.conv_subs;
          const int rem = kb % per_tile;
          return ((((kb / per_tile) * st.conv_subs + rem % st.conv_subs) * kBK) << 4) | (rem / st.conv_subs);
        };
        // the activation (A) box of K-block kb into `dst`, completing on barrier fb; conv:
        // cc = conv_coords(kb)
        auto load_a = [&](uint8_t* dst, uint64_t* fb, int kb, int cc) {
          const uint32_t fbc = CG == 2 ? ptx::mapa(fb, plead) : 0;
          if (conv) {
            // im2col box: 128 consecutive output pixels' inputs at filter tap (r, s), 64
            // channels from c0; the map's bounding box starts at (-1, -1), so pixel
            // (p, q) sits at box coordinate (p - 1, q - 1) and the tap adds (r, s);
            // outside the image the TMA fills zeros (the 3x3 "same" padding).
            const int c0 = cc >> 4, tap = cc & 15;
            const uint16_t r = static_cast<uint16_t>(tap / 3), s = static_cast<uint16_t>(tap % 3);
            if constexpr (CG == 2) {
              ptx::tma_load_im2col_pair(dst, &st.tmap_a, fbc, c0, cq - 1, cp - 1, cn, s, r, pol_a);
            } else {
              ptx::tma_load_im2col(dst, &st.tmap_a, fb, c0, cq - 1, cp - 1, cn, s, r, pol_a);
            }
          } else if constexpr (QD) {
            // this CTA's 64 of its half's 128 rows, to the same half of both pairs
            const uint16_t mask = static_cast<uint16_t>((1u << rank) | (1u << (2 + rank)));
            ptx::tma_load_2d_pair_mc(dst + pair * (C::kChunkBytes / 2), &st.tmap_a_half, fbc,
                                     kb * kBK, act_row + static_cast<int>(pair) * 64, mask, pol_a);
          } else if constexpr (CG == 2) {
            ptx::tma_load_2d_pair(dst, &st.tmap_a, fbc, kb * kBK, act_row, pol_a);
          } else {
            ptx::tma_load_2d(dst, &st.tmap_a, fb, kb * kBK, act_row, pol_a);
          }
        };
        if (deep && !ordered) {
        } else if (waits && rot != 0) {
          all_waits();  // before any load
        } else if (waits) {
          // A split-K slice of a consumer still performs every k-step's wait of the
          // reference model (each z-slice of a tile runs all k-steps, engine.py:469-514):
          // the ones before its K range up front (they cover the k-step it starts in) ...
          // (a balanced segment waits only for what it reads: the k-step it starts inside;
          // Row / Strided: k-step 0, the row's single wait)
          int ks_lo = 0, ks_hi = (kb_begin + kbpk - 1) / kbpk;
          if (bal) {
            ks_lo = ordered ? kb_begin / kbpk : 0;
            ks_hi = ordered ? ks_hi : (kb_begin > 0 ? 1 : 0);
          }
          for (int ks = ks_lo; ks < ks_hi; ++ks) wait_kstep(ks);
        }
        // conv K-block coordinates, advanced without divisions (rot = 0 for conv)
        int cv_sub = 0, cv_tap = 0, cv_ct = 0;
        if (conv) {
          const int per_tile = 9 * st.conv_subs;
          cv_ct = kb_begin / per_tile;
          cv_tap = (kb_begin % per_tile) / st.conv_subs;
          cv_sub = kb_begin % st.conv_subs;
        }
#pragma unroll 1
        for (int i = 0, kb = kb_begin + rot, gi = 0; i < k_per; ++i) {
          // diagnostic only (flag bit 15): stream the weights, skip the activation loads
          const bool skip_act = (p.flags >> 15) & 1;
          // normal layout: activations -> UMMA-M operand, weights -> UMMA-N; swapped:
          // weights -> UMMA-M, activations -> UMMA-N. Chunked: one A chunk, 1-2 B chunks.
          const int e0 = ea;
          claim(e0);
          ea = wrap_inc(ea, R);
          int e1 = 0, e2 = 0;
          if constexpr (C::kChunked) {
            e1 = ea;
            claim(e1);
            ea = wrap_inc(ea, R);
            if (wide) {
              e2 = ea;
              claim(e2);
              ea = wrap_inc(ea, R);
            }
          }
          uint64_t* fb = &full[kq % kFullRing];
          const uint32_t fbc = CG == 2 ? ptx::mapa(fb, plead) : 0;  // the pair leader's barrier
          if (leader) {
            const int nc = 2 + wide;
            // chunked: A box (128 rows) + 1-2 B boxes of hn / 2 rows, 128 B each
            const int bytes = C::kChunked ? (skip_act ? 0 : C::kChunkBytes) + (nc - 1) * (hn / 2) * 128
                                          : (skip_act ? (SW ? C::kABytes : C::kBBytes)
                                                      : C::kStageBytes);
            ptx::mbar_arrive_expect_tx(fb, CG * bytes);
          }
          uint8_t* act_dst;
          uint8_t* w_dst;
          if constexpr (C::kChunked) {
            act_dst = smem + e0 * C::kChunkBytes;
            w_dst = smem + e1 * C::kChunkBytes;
          } else {
            act_dst = SW ? sB + e0 * C::kBBytes : sA + e0 * C::kABytes;
            w_dst = SW ? sA + e0 * C::kABytes : sB + e0 * C::kBBytes;
          }
          // weight K coordinate; conv: K-block kb = (channel tile, tap, sub-block)
          int wk = kb * kBK, cc = 0;
          if (conv) {
            const int c0 = (cv_ct * st.conv_subs + cv_sub) * kBK;
            cc = (c0 << 4) | cv_tap;
            wk = cv_tap * st.conv_cin + c0;  // KRSC: [tap][cin] inside a weight row
            if (++cv_sub == st.conv_subs) {
              cv_sub = 0;
              if (++cv_tap == 9) {
                cv_tap = 0;
                ++cv_ct;
              }
            }
          }
          auto load_b = [&]() {
            if constexpr (CG == 2) {
              ptx::tma_load_2d_pair(w_dst, &st.tmap_b, fbc, wk, w_row, pol_b);
              if (C::kChunked && wide)
                ptx::tma_load_2d_pair(smem + e2 * C::kChunkBytes, &st.tmap_b, fbc, wk,
                                      w_row + hn, pol_b);
            } else {
              ptx::tma_load_2d(w_dst, &st.tmap_b, fb, wk, w_row, pol_b);
            }
          };
          if (reorder) load_b();
          if (i >= pre && waits && rot == 0 && kb % kbpk == 0) wait_kstep(kb / kbpk);
          if (!skip_act && i >= pre) load_a(act_dst, fb, kb, cc);  // deep "+R": first `pre` later
          if (!reorder) load_b();
          ++kq;
          if (++gi == group || i + 1 == k_per) {  // the K-block closes a commit group
            ++cid;
            gi = 0;
          }
          if (++kb == kb_end) kb = kb_begin;
          if (i + 1 == pre) {
            // the ring holds the weights of K-blocks [0, pre): wait, then their activations
            if (!ordered) {
              all_waits();
            } else {
              for (int j = 0; j < pre; ++j) {  // the k-steps starting in [kb_begin, +pre)
                const int kbj = kb_begin + j;
                if (kbj % kbpk == 0) wait_kstep(kbj / kbpk);
              }
            }
            for (int j = 0; j < pre && !skip_act; ++j) {
              const int ej = (ea_start + j * per_kb) % R;
              const int kbj = kb_begin + (rot + j) % k_per;
              uint8_t* dst = C::kChunked ? smem + ej * C::kChunkBytes
                                         : (SW ? sB + ej * C::kBBytes : sA + ej * C::kABytes);
              load_a(dst, &full[(kq_start + j) % kFullRing], kbj, conv ? conv_coords(kbj) : 0);
            }
          }
        }
        // ... and the ones after it once its loads are issued.
        if (waits && rot == 0 && !(deep && !ordered) && !bal)
          for (int ks = (kb_end + kbpk - 1) / kbpk; ks * kbpk < st.k_blocks; ++ks) wait_kstep(ks);
        if constexpr (C::kChunked && !QD) {
          // Split-K owner (the last slice of a CTA-pair tile): once the other slices' fp32
          // partial planes of this CTA's rows are written, stream them in as 32-column x
          // 128-row boxes — the A operand of the tensor-core reduction D += P x I (see the
          // MMA warp) — so the sum is TMA-fed and bandwidth-bound instead of a register
          // loop at loaded-L2 latency. One ring chunk and one commit per box.
          if (st.red_mma && !bal && t.z >= 2 && t.tz == t.z - 1 && !((p.flags >> 29) & 1)) {
            owner_plane_loads<CG, C>(p, st, t, static_cast<int>(rank), leader, plead, hn << wide,
                                     smem, full, empty, owner, ea, kq, cid, pol_first);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== tcgen05.mma issuer (leader) =====================
    if (leader) {
      // UMMA shape: M = 128 per CTA (256 for a pair), N = BN in both layouts
      constexpr uint32_t kIdesc = ptx::idesc_f16(128 * CG, BN, AbFormat<T>::value);
      int ea = 0;  // ring entry of the next K-block's A operand, as the producer
      uint32_t kq = 0;    // K-blocks consumed (full barrier index)
      uint32_t cid = 0;   // commit group
      const int group = commit_group(p.flags);
      uint32_t u = 0;  // TMEM accumulator-slot uses (a double-width tile takes two)
      int hm = 0, mw_stage = -1, mw_count = 0;  // halo conv: windows, resident-weight loads
      // halo conv fast path: the current halo stage's item range and constants in registers
      // (set by the general path below; measured ~2.9k cycles per item of parameter-block
      // reads and bookkeeping in the issuing warp otherwise, profiles/r02y_conv_halo.txt)
      int hc_lo = 0, hc_hi = 0, hc_hnb = 1, hc_hwin = 0, hc_hs8 = 0, hc_hsub = 1;
      uint64_t hc_sub = 0;
#pragma unroll 1
      for (int it = 0;; ++it) {
        int kbr;
        const int g = ring_take(it, QD && !uleader, kbr);
        if (g < 0) break;
        if constexpr (C::kHaloOk) {
          if (g >= hc_lo && g < hc_hi) {
            ptx::mbar_wait(&tmem_empty[u & 1], ((u >> 1) & 1) ^ 1);
            ptx::tc_fence_after();
            const uint32_t d_tmem = tmem_base + (u & 1) * C::kAccCols;
            const int hq = hm / hc_hnb, b = hm - hq * hc_hnb;
            ptx::mbar_wait(&win_full[b], hq & 1);
            ptx::tc_fence_after();
            if (lane == 0) {
              const uint64_t ad0 =
                  ptx::smem_desc_k_sw128(ptx::smem_u32(smem + 9 * 8192 + b * hc_hwin));
              const uint64_t bd0 = ptx::smem_desc_k_sw128(ptx::smem_u32(smem));
              if (hc_hsub > 1) {
#pragma unroll 1
                for (int tap = 0; tap < 9; ++tap) {
                  const int r = tap / 3, s = tap - 3 * (tap / 3);
                  const uint64_t ad = ad0 + static_cast<uint64_t>(r * hc_hs8 + s * 8);
                  const uint64_t bdd = bd0 + static_cast<uint64_t>(tap * 512);
                  ptx::umma_f16_kblock<CG>(d_tmem, ad, bdd, kIdesc, tap != 0);
                  ptx::umma_f16_kblock<CG>(d_tmem + 64, ad + hc_sub, bdd, kIdesc, tap != 0);
                }
              } else {
#pragma unroll 1
                for (int tap = 0; tap < 9; ++tap) {
                  const int r = tap / 3, s = tap - 3 * (tap / 3);
                  const uint64_t ad = ad0 + static_cast<uint64_t>(r * hc_hs8 + s * 8);
                  const uint64_t bdd = bd0 + static_cast<uint64_t>(tap * 512);
                  ptx::umma_f16_kblock<CG>(d_tmem, ad, bdd, kIdesc, tap != 0);
                }
              }
              ptx::umma_commit(&win_empty[b]);
              ptx::umma_commit(&tmem_full[u & 1]);
            }
            ++hm;
            __syncwarp();
            u += 1;
            continue;
          }
        }
        const StageParams& sp = p.st[stage_of(p, g)];
        if (sp.kind == kStageDot || sp.kind == kStageAllReduce)
          continue;  // no MMA, no accumulator buffer
        const int kblocks = (C::kHaloOk && sp.hmode) ? 0
                            : bal ? (kbr & 0xffff) - (kbr >> 16)
                                  : sp.k_blocks / item_slices(sp, g - sp.item_begin);
        const int wide = (C::kChunked && !QD) ? sp.wide : 0;
        // instruction descriptor: N = the stage's columns per MMA (chunked stages)
        const uint32_t idesc = C::kChunked ? ptx::idesc_f16(128 * CG, sp.half_n, AbFormat<T>::value)
                                           : kIdesc;
        // TMEM reuse only (for pairs, tcgen05 fences order the peer's loads)
        for (int j = 0; j <= wide; ++j)
          ptx::mbar_wait(&tmem_empty[(u + j) & 1], (((u + j) >> 1) & 1) ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + (u & 1) * C::kAccCols;
        const uint32_t d_tmem2 = tmem_base + ((u + 1) & 1) * C::kAccCols;
        const bool tr = p.trace != nullptr;
        const bool no_mma = (p.flags >> 13) & 1;  // diagnostic only: skip the MMAs
        uint64_t starve_ns = 0;  // time this tile's MMAs waited for operand stages
        if constexpr (C::kHaloOk) {
          if (sp.hmode) {
            // halo conv tile: nine taps x four K = 16 MMAs over one staged window; tap
            // (r, s)'s A is the window shifted by r window rows + s pixels (whole 128-B
            // rows: the 128-B swizzle is address based, so any row offset is a valid
            // K-major descriptor start), B the resident tap weights
            const int stg_i = stage_of(p, g);
            if (stg_i != mw_stage) {
              ptx::mbar_wait(hw_full, mw_count & 1);
              ++mw_count;
              mw_stage = stg_i;
            }
            const int b = hm % sp.hnb;
            ptx::mbar_wait(&win_full[b], (hm / sp.hnb) & 1);
            ptx::tc_fence_after();
            if (!tr && !no_mma) {  // later items of this stage take the fast path above
              hc_lo = sp.item_begin;
              hc_hi = sp.item_end;
              hc_hnb = sp.hnb;
              hc_hwin = sp.hwin;
              hc_hs8 = sp.hs * 8;
              hc_hsub = sp.hsub;
              hc_sub = static_cast<uint64_t>((sp.hmode == 1 ? 128 : sp.hs) * 8);
            }
            if (lane == 0) {
              // (a tile's window always starts at its base pixel: halo_tile's base is 0, so
              // the MMA warp needs no tile decode — integer divisions by runtime grid sizes
              // in the single issuing thread, on the per-item critical path)
              if (tr) {
                const Tile t5 = decode(p, g);
                trace_now(p, 5, t5.s, t5.tb, -1, -1, -1, -1, t5.tx, t5.ty);
              }
              // tap (r, s): A = the window from row r * hs + s (16-B descriptor units: 8 per
              // 128-B row), B = tap weights (8 KB = 512 units apart)
              const uint64_t ad0 = ptx::smem_desc_k_sw128(ptx::smem_u32(smem + 9 * 8192 + b * sp.hwin));
              const uint64_t bd0 = ptx::smem_desc_k_sw128(ptx::smem_u32(smem));
              const int hs8 = sp.hs * 8;
              if (sp.hsub > 1) {
                // two sub-tiles into accumulator columns [64, 128): the window rows 128 + ...
                // (rows mode) or one image row further (segment mode), in 16-B units
                const uint64_t sub_off = (sp.hmode == 1 ? 128 : sp.hs) * 8;
#pragma unroll 1
                for (int tap = 0; tap < 9; ++tap) {
                  const int r = tap / 3, s = tap - 3 * (tap / 3);
                  const uint64_t ad = ad0 + static_cast<uint64_t>(r * hs8 + s * 8);
                  const uint64_t bdd = bd0 + static_cast<uint64_t>(tap * 512);
                  if (!no_mma) {
                    ptx::umma_f16_kblock<CG>(d_tmem, ad, bdd, kIdesc, tap != 0);
                    ptx::umma_f16_kblock<CG>(d_tmem + 64, ad + sub_off, bdd, kIdesc, tap != 0);
                  }
                }
              } else {
#pragma unroll 1
                for (int tap = 0; tap < 9; ++tap) {
                  const int r = tap / 3, s = tap - 3 * (tap / 3);
                  const uint64_t ad = ad0 + static_cast<uint64_t>(r * hs8 + s * 8);
                  const uint64_t bdd = bd0 + static_cast<uint64_t>(tap * 512);
                  // (one accumulator: a second one for alternating taps measured no faster
                  // and doubles the epilogue's TMEM reads, the other pacing resource)
                  if (!no_mma) ptx::umma_f16_kblock<CG>(d_tmem, ad, bdd, kIdesc, tap != 0);
                }
              }
              ptx::umma_commit(&win_empty[b]);
            }
            ++hm;
            __syncwarp();
          }
        }
#pragma unroll 1
        for (int kb = 0, gi = 0; kb < kblocks; ++kb) {
          uint64_t* fb = &full[kq % kFullRing];
          const uint32_t ph = (kq / kFullRing) & 1;
          if ((p.flags >> 19) & 1) {
            // diagnostic only (flag bit 19): MMA pipe rate without waiting for operands
          } else if (tr && !ptx::mbar_test_wait(fb, ph)) {
            const uint64_t t0 = ptx::global_timer();
            ptx::mbar_wait(fb, ph);
            if (kb > 0) starve_ns += ptx::global_timer() - t0;
          } else {
            ptx::mbar_wait(fb, ph);
          }
          if (tr && kb == 0 && lane == 0) {
            const Tile t = decode(p, g);
            trace_now(p, 5, t.s, t.tb, -1, -1, -1, -1, t.tx, t.ty);
          }
          ptx::tc_fence_after();
          if (lane == 0) {
            if constexpr (C::kChunked) {
              // A chunk; B chunk(s): output columns [0, BN) and, double width, [BN, 2 BN)
              auto desc = [&](int e) {
                return ptx::smem_desc_k_sw128(ptx::smem_u32(smem + e * C::kChunkBytes));
              };
              const uint64_t ad = desc(ea);
              const int eb = wrap_inc(ea, R), eb2 = wrap_inc(eb, R);
              if (no_mma) {
              } else if (wide) {
                // both halves' MMAs interleaved: no two consecutive MMAs into one
                // accumulator (at the tcgen05 floor; 4 + 4 back to back ran ~3-25% slower)
                ptx::umma_f16_kblock2<CG>(d_tmem, d_tmem2, ad, desc(eb), desc(eb2), idesc, kb != 0);
              } else {
                ptx::umma_f16_kblock<CG>(d_tmem, ad, desc(eb), idesc, kb != 0);
              }
            } else {
              const int rs = ea;
              const uint32_t a_addr = ptx::smem_u32(sA + rs * C::kABytes);
              const uint32_t b_addr = ptx::smem_u32(sB + rs * C::kBBytes);
              if (no_mma) {
              } else if constexpr (SW && C::kAcc > 1) {
                // rotate independent accumulators (sub-step `step` -> step % kAcc), the
                // K-block's four MMAs in one issue sequence
                const int step = kb * (kBK / 16);
                uint32_t dd[4], mask = 0;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                  dd[k] = d_tmem + ((step + k) % C::kAcc) * BN;
                  mask |= (step + k >= C::kAcc ? 1u : 0u) << k;
                }
                ptx::umma_f16_kblock4(dd[0], dd[1], dd[2], dd[3], ptx::smem_desc_k_sw128(a_addr),
                                      ptx::smem_desc_k_sw128(b_addr), kIdesc, mask);
              } else {
                // the K-block's four MMAs back to back in one issue sequence
                ptx::umma_f16_kblock<CG>(d_tmem, ptx::smem_desc_k_sw128(a_addr),
                                         ptx::smem_desc_k_sw128(b_addr), kIdesc, kb != 0);
              }
            }
            // one commit frees every ring entry of the group's K-blocks
            if (gi + 1 == group || kb + 1 == kblocks) {
              if constexpr (QD) {
                ptx::umma_commit_pair_mask(&empty[cid % kCommitRing], 0xF);  // all 4 CTAs' rings
              } else if constexpr (CG == 2) {
                ptx::umma_commit_pair(&empty[cid % kCommitRing]);
              } else {
                ptx::umma_commit(&empty[cid % kCommitRing]);
              }
            }
          }
          if (++gi == group || kb + 1 == kblocks) {
            ++cid;
            gi = 0;
          }
          ea = wrap_inc(ea, R);
          if constexpr (C::kChunked) {
            for (int c = 0; c <= wide; ++c) ea = wrap_inc(ea, R);
          }
          ++kq;
          __syncwarp();
        }
        if constexpr (C::kChunked && !QD) {
          // split-K owner: D[:, 32 j .. 32 j + 32) += P_z[:, 32 j ..] x I for every other
          // slice's plane P_z (kind::tf32: the partial enters the fp32 accumulator at tf32
          // precision, 2^-11 relative — below the fp16/bf16 output rounding), one ring
          // chunk per 32-column box, committed box by box like a K-block
          if (!bal) {
            const Tile tt = decode(p, g);
            if (sp.red_mma && tt.z >= 2 && tt.tz == tt.z - 1 && !((p.flags >> 29) & 1)) {
              const int hn = sp.half_n;
              const int groups = (hn << wide) / 32;
              const uint32_t idesc_r = ptx::idesc_tf32(128 * CG, 32);
              const uint64_t bd = ptx::smem_desc_k_sw128(ptx::smem_u32(smem + C::kIdentOff));
#pragma unroll 1
              for (int rb = 0; rb < (tt.z - 1) * groups; ++rb) {
                const int col = (rb % groups) * 32;
                ptx::mbar_wait(&full[kq % kFullRing], (kq / kFullRing) & 1);
                ptx::tc_fence_after();
                if (lane == 0) {
                  const uint32_t dcol = tmem_base + ((u + col / hn) & 1) * C::kAccCols + (col % hn);
                  if (!no_mma && !((p.flags >> 30) & 1))  // bit 30: diagnostic, no reduction MMAs
                    ptx::umma_tf32_kblock<CG>(dcol, ptx::smem_desc_k_sw128(
                                                        ptx::smem_u32(smem + ea * C::kChunkBytes)),
                                              bd, idesc_r);
                  if constexpr (CG == 2) {
                    ptx::umma_commit_pair(&empty[cid % kCommitRing]);
                  } else {
                    ptx::umma_commit(&empty[cid % kCommitRing]);
                  }
                }
                ++cid;
                ea = wrap_inc(ea, R);
                ++kq;
                __syncwarp();
              }
            }
          }
        }
        if (lane == 0) {
          for (int j = 0; j <= wide; ++j) {
            if constexpr (QD) {
              ptx::umma_commit_pair_mask(&tmem_full[(u + j) & 1],
                                         static_cast<uint16_t>(3u << plead));  // this pair
            } else if constexpr (CG == 2) {
              ptx::umma_commit_pair(&tmem_full[(u + j) & 1]);
            } else {
              ptx::umma_commit(&tmem_full[(u + j) & 1]);
            }
          }
          if (tr) {
            const Tile t = decode(p, g);
            trace_now(p, 6, t.s, t.tb, -1, -1, -1,
                        static_cast<int>(starve_ns > 0x7fffffff ? 0x7fffffff : starve_ns), t.tx,
                        t.ty);
          }
        }
        __syncwarp();
        u += 1 + wide;
      }
    }
  } else if (CG == 1 && warp == 3) {
    // ===================== post warp (single-CTA kernels) =====================
    // stage.post() of items the epilogue queued: the release fence waits for the tile's
    // stores to be performed (~3k cycles after a 128-row store burst) — here, off the
    // epilogue warps' per-item path. Ordering: the epilogue's stores, its named barrier,
    // thread 128's arrive (release, CTA) -> this wait (acquire) -> the GPU-scope fence ->
    // the release RMW on the consumer's semaphore.
    if (lane == 0 && any_post) {
#pragma unroll 1
      for (int q = 0;; ++q) {
        const int ps = q % kPostRing;
        ptx::mbar_wait(&post_full[ps], (q / kPostRing) & 1);
        const int g = post_req[ps];
        ptx::mbar_arrive(&post_empty[ps]);
        if (g < 0) break;
        const Tile t = decode(p, g);
        const StageParams& st = p.st[t.s];
        __threadfence();
        ptx::fence_proxy_async_global();
        for (int i = 0; i < st.n_out_deps; ++i) {
          const int d = st.out_deps[i];
          const DepParams& dp = p.dep[d];
          const int idx = post_target(dp.policy, dp.param, t.tx, t.ty,
                                      Grid3{dp.pgx, dp.pgy, dp.pgz});
          if (p.st[dp.consumer].kind == kStageAllReduce) {
            __threadfence_system();
            ptx::atom_add_release_sys(dp.sem + idx, 1);
          } else {
            ptx::red_add_release_gpu(dp.sem + idx, 1);
          }
          ptx::red_add_release_gpu(p.scratch + kDoneBase + d, 1);
        }
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ===================== epilogue =====================
    const int ew = warp & 3;         // TMEM lanes [32*ew, 32*ew+32) (a warp's lane quarter)
    const int eg = (warp - 4) >> 2;  // column group (chunked tiles: 0 or 1)
    // Coalesced row stores through this warp's staging block: every lane holds 128 B of
    // its row (32 words); they go to shared memory (16-B granules XOR-swizzled by row)
    // and come back as 4 rows x 128 B per instruction, written with 16-B stores to
    // dst(row_in_warp, granule) (nullptr = skip).
    uint32_t* stg =
        reinterpret_cast<uint32_t*>(smem + C::kStageOff + (warp - 4) * C::kStageWarpBytes);
    // split-K partial planes: written evict_last, read evict_first, so they stay in L2
    // between the slices instead of round-tripping through HBM under the weight streams
    // (diagnostic flag bit 26: no hints)
    auto stage_rows_hint = [&](const uint32_t (&v)[32], auto&& dst, uint64_t pol_el) {
      if constexpr (C::kStageWarpBytes >= 4096) {
#pragma unroll
        for (int g = 0; g < 8; ++g)
          *reinterpret_cast<uint4*>(stg + lane * 32 + ((g ^ (lane & 7)) * 4)) =
              make_uint4(v[4 * g], v[4 * g + 1], v[4 * g + 2], v[4 * g + 3]);
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int rr = 4 * i + (lane >> 3), g = lane & 7;
          const uint4 q = *reinterpret_cast<const uint4*>(stg + rr * 32 + ((g ^ (rr & 7)) * 4));
          uint4* d = dst(rr, g);
          if (d != nullptr) ptx::st_global_v4_hint(d, q, pol_el);
        }
        __syncwarp();
      } else {
        // 2-KB block: rows [16 h, 16 h + 16) per pass
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if ((lane >> 4) == h) {
            const int lr = lane & 15;
#pragma unroll
            for (int g = 0; g < 8; ++g)
              *reinterpret_cast<uint4*>(stg + lr * 32 + ((g ^ (lr & 7)) * 4)) =
                  make_uint4(v[4 * g], v[4 * g + 1], v[4 * g + 2], v[4 * g + 3]);
          }
          __syncwarp();
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int rr = 4 * i + (lane >> 3), g = lane & 7;
            const uint4 q = *reinterpret_cast<const uint4*>(stg + rr * 32 + ((g ^ (rr & 7)) * 4));
            uint4* d = dst(16 * h + rr, g);
            if (d != nullptr) ptx::st_global_v4_hint(d, q, pol_el);
          }
          __syncwarp();
        }
      }
    };
    auto stage_rows = [&](const uint32_t (&v)[32], auto&& dst) {
      stage_rows_hint(v, dst, (p.flags >> 26) & 1 ? ptx::policy_evict_normal()
                                                  : ptx::policy_evict_last());
    };
    uint32_t local = 0;  // GeMM tiles (peer_done parity)
    int npost = 0;       // single-CTA kernels: posts queued for the post warp (thread 128)
    uint32_t u = 0;      // TMEM accumulator-slot uses, as counted by the MMA warp
    uint32_t tmem_empty_remote[2] = {0, 0};
    if constexpr (CG == 2) {
      if (!leader) {
        for (int i = 0; i < 2; ++i) tmem_empty_remote[i] = ptx::mapa(&tmem_empty[i], plead);
      }
    }
    // Compute dot tile (tx, ty) of stage ds with the 128 epilogue threads (its wait is
    // already satisfied), then post to its consumers (thread 128).
    // Compute dot tile (tx, ty) — all its rows (half < 0) or one CTA's 128 of a pair's 256
    // (half 0 / 1) — and, if `post`, post it to its consumers (thread 128).
    auto run_dot_rows = [&](int ds, int tx, int ty, int tb, int half) {
      const StageParams& sd = p.st[ds];
      asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
      ptx::fence_acq_rel_gpu();
      if (threadIdx.x == 128 && half <= 0)
        trace_now(p, 7, ds, tb, -1, -1, -1, -1, tx, ty);
      // a dot tile covers BN / 128 heads (the paper's stride H / (8 Ty));
      // one warp per (row, head), warps striding over the tile's rows x heads
      constexpr int kHeads = BN >= 128 ? BN / 128 : 1;
      const int items = (half < 0 ? C::kTileM : 128) * kHeads;
      const int row0 = tx * C::kTileM + (half > 0 ? 128 : 0);
      // loads in flight per warp: 2 x kB items (fewer for 384-thread CTAs, 168 registers)
      constexpr int kB = C::kChunked ? 2 : 4;
#pragma unroll 1
      for (int it0 = (warp - 4) * 2; it0 < items; it0 += kEpiWarps * 2 * kB)
        dot_batch_warp<T, kB>(sd, row0, kHeads, it0, kEpiWarps * 2, items, ty * kHeads, lane);
      asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
    };
    auto post_dot = [&](int ds, int tx, int ty, int tb) {
      const StageParams& sd = p.st[ds];
      if (threadIdx.x == 128) {
        const uint64_t tnow = p.trace ? ptx::global_timer() : 0;  // traced launches only
        trace_event(p, tnow, 8, ds, tb, -1, -1, -1, -1, tx, ty);
        __threadfence();
        ptx::fence_proxy_async_global();
        for (int i = 0; i < sd.n_out_deps; ++i) {
          const int d = sd.out_deps[i];
          const DepParams& dp = p.dep[d];
          const int idx = post_target(dp.policy, dp.param, tx, ty, Grid3{dp.pgx, dp.pgy, dp.pgz});
          const int old = ptx::atom_add_release_gpu(dp.sem + idx, 1);
          ptx::atom_add_release_gpu(p.scratch + kDoneBase + d, 1);
          trace_event(p, tnow, 3, ds, tb, -1, d, idx, old + 1, tx, ty);
        }
        trace_event(p, tnow, 4, ds, tb, -1, -1, -1, -1, tx, ty);
      }
    };
    auto run_dot = [&](int ds, int tx, int ty, int tb) {
      run_dot_rows(ds, tx, ty, tb, -1);
      post_dot(ds, tx, ty, tb);
    };
    // last-arriver dot tiles split over a CTA pair (diagnostic flag bit 28: leader only)
    const bool dsplit = CG == 2 && !((p.flags >> 28) & 1);
    uint32_t dmsg = 0, ddone = 0;  // dot_msg / dot_done phases (peer / leader)
#pragma unroll 1
    for (int it = 0;; ++it) {
      int kbr;
      const int g = ring_take(it, CG == 2 && !uleader, kbr);
      if (g < 0) break;
      const Tile t = decode(p, g);
      const StageParams& st = p.st[t.s];
      // balanced segment role (see Tile): 0 whole tile, 1 not the head, 2 head
      const int brole = !bal ? 0
                        : ((kbr >> 16) > 0 ? 1 : ((kbr & 0xffff) == st.k_blocks ? 0 : 2));
      if (st.kind == kStageAllReduce) {
        // Tensor-parallel all-reduce of one producer tile (extension): this
        // rank owns tiles lin = tb * world + rank. Wait for the tile's post on every rank
        // (system-scope acquire over P2P), sum the world partial tiles in fp32, store the
        // sum into every rank's buffer, then count the tile into every rank's done counter.
        // Each CTA of a pair handles its 128 rows.
        const int world = p.peers.world;
        const int lin = t.tb * world + p.peers.rank;
        const int tx = lin / st.grid_y, ty = lin % st.grid_y;
        const DepParams& dp = p.dep[st.in_dep];
        if (threadIdx.x == 128) {
          // the group's semaphores are monotone across launches (epoch scheme): launch e
          // waits for e x pgz posts, so a peer's value from launch e-1 never satisfies it
          const int idx = post_target(dp.policy, dp.param, tx, ty, Grid3{dp.pgx, dp.pgy, dp.pgz});
          for (int q = 0; q < world; ++q)
            sem_spin_sys(p, p.peers.sems[q] + idx, dp.pgz * p.peers.epoch);
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
        ptx::fence_acq_rel_sys();
        allreduce_rows<T>(p, st, tx * C::kTileM + static_cast<int>(rank) * 128, ty,
                          threadIdx.x - 128, kEpiThreads, smem,
                          C::kChunked ? C::kStageOff : C::kStages * C::kStageBytes);
        asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
        if (threadIdx.x == 128) {
          __threadfence_system();
          for (int q = 0; q < world; ++q) ptx::atom_add_release_sys(p.peers.done[q], 1);
        }
        continue;
      }
      if (st.kind == kStageDot) {
        // Attention's fused dot: XDot = Dropout(Softmax(XQ . XV)) . XK,
        // column-tile local as its StridedSync dependency defines it — tile (r, h) reads
        // only head h's Q, K and V column tiles of row tile r. Dropout p = 0 (inference).
        // The leader CTA computes the whole tile; its peer (CTA pairs) has nothing to do.
        if (CG == 2 && !leader) continue;
        if (threadIdx.x == 128 && st.in_dep >= 0 && !((p.flags >> 12) & 1)) {
          const DepParams& dp = p.dep[st.in_dep];
          Wait w = consumer_wait(dp.policy, dp.param, t.tx, t.ty, 0, Grid3{dp.pgx, dp.pgy, dp.pgz},
                                 dp.pgz);
          if (w.sem >= 0) {
            trace_now(p, 1, t.s, t.tb, 0, st.in_dep, w.sem, w.expected,
                        t.tx, t.ty, t.tz);
            sem_wait(p, dp.sem + w.sem, w.expected);
            trace_now(p, 2, t.s, t.tb, 0, st.in_dep, w.sem, w.expected,
                        t.tx, t.ty, t.tz);
          }
        }
        run_dot(t.s, t.tx, t.ty, t.tb);
        continue;
      }
      const int wide = (C::kChunked && !QD) ? st.wide : 0;
      const int hn = C::kChunked ? st.half_n : BN;  // accumulator columns per slot
      for (int j = 0; j <= wide; ++j)  // arrived by the MMA commits
        ptx::mbar_wait(&tmem_full[(u + j) & 1], ((u + j) >> 1) & 1);
      ptx::tc_fence_after();
      if (threadIdx.x == 128 && uleader && p.trace != nullptr)  // epilogue begin (extension)
        trace_now(p, 7, t.s, t.tb, -1, -1, -1, -1, t.tx, t.ty, t.tz);
      const uint32_t lane_base = tmem_base + (static_cast<uint32_t>(ew * 32) << 16);
      const uint32_t t_lane = lane_base + (u & 1) * C::kAccCols;
      // accumulator column x of this tile (a double-width tile spans both slots)
      auto tcol = [&](int x) -> uint32_t {
        return lane_base + ((u + x / hn) & 1) * C::kAccCols + (x % hn);
      };
      auto release_slot = [&](int j) {
        ptx::tc_fence_before();
        if (lane == 0) {
          const uint32_t sl = (u + j) & 1;
          if (CG == 2 && !leader) {
            ptx::mbar_arrive_remote(tmem_empty_remote[sl]);
          } else {
            ptx::mbar_arrive(&tmem_empty[sl]);
          }
        }
      };
      auto release_tmem = [&]() {
        for (int j = 0; j <= wide; ++j) release_slot(j);
      };
      if constexpr (SW) {
        // Swapped tile: TMEM lane = output column, TMEM column = activation row.
        const int ncl = ew * 32 + lane;
        const int ncol = t.ty * 128 + ncl;
        const int b0 = t.tx * BN;
        const int rows = st.m - b0 < BN ? st.m - b0 : BN;
        const bool gl = st.epilogue == TS_EPI_GELU;
        T* cout = reinterpret_cast<T*>(st.c) + ncol;
        // accumulators the MMA warp actually wrote (fewer than kAcc for very short K)
        const int steps = (st.k_blocks / st.splits) * (kBK / 16);
        const int n_acc = steps < C::kAcc ? steps : C::kAcc;
        // 32 activation rows [col, col+32) of this thread's output column, summed over the
        // rotating accumulators
        auto load_sum = [&](int col, float (&v)[32]) {
          uint32_t r[32];
          ptx::tmem_ld_32x32b_x32(t_lane + col, r);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
#pragma unroll 1
          for (int a = 1; a < n_acc; ++a) {
            ptx::tmem_ld_32x32b_x32(t_lane + a * BN + col, r);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] += __uint_as_float(r[j]);
          }
        };
        if (st.splits == 1) {
#pragma unroll 1
          for (int cc = 0; cc < BN / 32; ++cc) {
            float v[32];
            load_sum(cc * 32, v);
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int b = cc * 32 + j;
              const float o = gl ? gelu(v[j]) : v[j];
              if (b < rows) cout[static_cast<size_t>(b0 + b) * st.ldc] = to_elem<T>(o);
            }
          }
          release_tmem();
        } else {
          // Split-K slice (reference z > 1): publish the fp32 partial, count arrivals;
          // the last slice to arrive sums all partials, applies the epilogue, stores.
          const int tile_id = t.tx * st.grid_y + t.ty;
          float* part = st.ws + (static_cast<size_t>(tile_id) * st.splits + t.tz) * BN * 128;
#pragma unroll 1
          for (int cc = 0; cc < BN / 32; ++cc) {
            float v[32];
            load_sum(cc * 32, v);
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              if (cc * 32 + j < rows) part[(cc * 32 + j) * 128 + ncl] = v[j];
            }
          }
          release_tmem();
          __threadfence();
          asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
          if (threadIdx.x == 128) {
            const int old = atomicAdd(&st.cnt[tile_id], 1);
            *split_flag = (old == st.splits - 1);
            if (old == st.splits - 1) st.cnt[tile_id] = 0;  // restore the zero invariant
          }
          asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
          if (*split_flag) {
            ptx::fence_acq_rel_gpu();
            const float* base = st.ws + static_cast<size_t>(tile_id) * st.splits * BN * 128;
            // 8 activation rows at a time so 8 x splits L2 loads are in flight together
#pragma unroll 1
            for (int b8 = 0; b8 < rows; b8 += 8) {
              float s[8];
#pragma unroll
              for (int j = 0; j < 8; ++j) s[j] = 0.f;
#pragma unroll 1
              for (int z = 0; z < st.splits; ++z) {
                const float* src = base + (static_cast<size_t>(z) * BN + b8) * 128 + ncl;
                float v[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) v[j] = b8 + j < rows ? __ldcg(src + j * 128) : 0.f;
#pragma unroll
                for (int j = 0; j < 8; ++j) s[j] += v[j];
              }
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                if (b8 + j < rows) {
                  const float o = gl ? gelu(s[j]) : s[j];
                  cout[static_cast<size_t>(b0 + b8 + j) * st.ldc] = to_elem<T>(o);
                }
              }
            }
          }
        }
      } else {
      const int row = t.tx * C::kTileM + static_cast<int>(rank) * 128 + ew * 32 + lane;
      bool row_ok = row < st.m;
      T* crow = reinterpret_cast<T*>(st.c) + static_cast<size_t>(row) * st.ldc;
      if constexpr (C::kHaloOk) {
        if (st.hmode) {
          // halo conv: accumulator row -> output pixel (junk positions are not stored)
          const int px = halo_pixel(st, halo_tile(st, t.tx), ew * 32 + lane);
          row_ok = px >= 0;
          crow = reinterpret_cast<T*>(st.c) + static_cast<size_t>(px < 0 ? 0 : px) * st.ldc;
        }
      }
      const int acc_cols = hn << wide;  // accumulator columns of this tile (this pair's)
      // first output column of this pair's accumulator (QD: the pair's half of the unit)
      const int col0 = QD ? (2 * t.ty + static_cast<int>(pair)) * acc_cols : t.ty * acc_cols;
      // full-sector (32-B) stores when the output rows are 32-B aligned
      const bool v8ok = ((reinterpret_cast<uintptr_t>(st.c) | (st.ldc * sizeof(T))) & 31) == 0;
      constexpr int G = C::kEpiGroups;
      if (C::kChunked && !QD &&
          (bal ? brole != 0
               : (!((p.flags >> 29) & 1) &&
                  (st.red_mma ? (t.z >= 2 && t.tz < t.z - 1) : (t.z >= 2 && t.z <= 4))))) {
        // Split-K slice (the reference's z > 1) of a CTA-pair tile, reduced into the
        // accumulator of the LAST slice to arrive (per tile half = per CTA): each slice
        // takes an arrival index from cnt[half]; the first z - 1 write their fp32 partial
        // (plane `arrival`, layout [16-column chunk][4][128 rows][4 floats]: each 16-B
        // store / load instruction of a warp covers 512 contiguous bytes) and count it
        // into rdy[half]; the last
        // waits for rdy == z - 1, adds the planes to its TMEM accumulator chunk by chunk,
        // applies the epilogue and stores. Against every slice writing a plane and the
        // last re-reading all z of them: one plane less written and read per tile, and
        // the last slice's own partial never leaves TMEM. Every slice still posts once
        // below (consumers wait for expected x z; each post follows its own slice's work,
        // and the count completes only after the reducing slice has stored).
        // Two slices: a + b is exact in either order, so the result does not depend on
        // which slice arrives last. Three or four: a reduction order that depends on the
        // arrival order would round differently run to run, so the owner is static — the
        // last slice in claim order (claimed last, it finishes last in the common case)
        // sums planes 0 .. z-2 in slice order into its accumulator; slices 0 .. z-2
        // write their planes and never wait. z > 4 takes the all-planes path below.
        // (diagnostic flag bit 29: the all-planes path for z = 2..4 as well)
        // Balanced (stream-K) segments use the same machinery with static roles: a
        // segment that does not start its tile writes the plane of its unit and counts it
        // into the tile half's ready counter; the head segment (K-block 0, the last item of
        // its unit) waits for the ua..ub planes and reduces them into its accumulator.
        const int tile_id = bal ? t.tb : t.tx * st.grid_y + t.ty;
        const int half_id = tile_id * CG * NP + static_cast<int>(qrank);
        int* cnt = st.cnt + half_id;
        int* rdy = bal ? cnt : st.cnt + st.grid_x * st.grid_y * CG * NP + half_id;
        const size_t plane = static_cast<size_t>(128) * acc_cols;
        // balanced head: the planes of units ua..ub (the ranges that start inside the tile)
        const int bw = bal ? bal_width(st, units) : 1;
        const int ua = bal ? (t.tb * st.k_blocks) / bw + 1 : 0;
        float* planes = bal ? st.ws + (static_cast<size_t>(ua) * CG * NP + qrank) * plane
                            : st.ws + static_cast<size_t>(half_id) * t.z * plane;
        const size_t pstride = bal ? static_cast<size_t>(CG * NP) * plane : plane;
        const int nparts = bal ? ((t.tb + 1) * st.k_blocks - 1) / bw - ua + 1 : t.z - 1;
        const int rl_row = ew * 32 + lane;
        const int row0 = t.tx * C::kTileM + static_cast<int>(rank) * 128;
        const int valid = st.m - row0 < 128 ? (st.m - row0 > 0 ? st.m - row0 : 0) : 128;
        const bool mine_ok = rl_row < valid;
        const int span = acc_cols / G;
        int arrival;
        if (bal) {
          arrival = brole == 1 ? 0 : nparts;
        } else if (st.red_mma) {
          // a writer slice (the owner, the last slice, reduces on the tensor cores and
          // takes the plain epilogue below)
          arrival = t.tz;
        } else if (t.z > 2) {
          arrival = t.tz == t.z - 1 ? nparts : t.tz;  // static owner: the last slice
        } else {
          if (threadIdx.x == 128) *split_flag = atomicAdd(cnt, 1);
          asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
          arrival = *split_flag;
        }
        if (arrival < nparts) {
          float* mine = bal ? st.ws + (static_cast<size_t>(unit) * CG * NP + qrank) * plane
                            : planes + static_cast<size_t>(arrival) * plane;
#pragma unroll 1
          for (int j = 0; j <= wide; ++j) {
            const int lo = max(eg * span, j * hn), hi = min((eg + 1) * span, (j + 1) * hn);
#pragma unroll 1
            for (int x = lo; x < hi && ew * 32 < valid; x += 16) {  // warp-uniform skip
              uint32_t r[16];
              ptx::tmem_ld_32x32b_x16(tcol(x), r);
              ptx::tmem_ld_wait();
              if (mine_ok && !st.red_mma) {
                uint4* d = reinterpret_cast<uint4*>(mine + (static_cast<size_t>(x / 16) * 512 + rl_row) * 4);
#pragma unroll
                for (int q = 0; q < 4; ++q)
                  d[q * 128] = make_uint4(r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]);
              } else if (mine_ok) {
                // row-major [128 rows][tile columns] fp32: the owner's reduction boxes,
                // written evict_last so they are still in L2 when the owner streams them
                float* d = mine + static_cast<size_t>(rl_row) * acc_cols + x;
                const uint64_t pel = ptx::policy_evict_last();
#pragma unroll
                for (int q = 0; q < 4; ++q)
                  ptx::st_global_v4_hint(d + 4 * q, make_uint4(r[4 * q], r[4 * q + 1], r[4 * q + 2],
                                                               r[4 * q + 3]), pel);
              }
            }
            release_slot(j);
          }
          __threadfence();
          asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
          if (threadIdx.x == 128) {
            if (uleader && p.trace != nullptr)  // partial written (extension)
              trace_now(p, 9, t.s, t.tb, -1, -1, -1, -1, t.tx, t.ty, t.tz);
            ptx::fence_proxy_async_global();  // the owner reads the plane with TMA
            ptx::atom_add_release_gpu(rdy, 1);
          }
        } else {
          if (threadIdx.x == 128) {
            sem_spin(p, rdy, nparts);
            *cnt = 0;  // every slice has arrived and every writer has counted: restore zero
            *rdy = 0;
          }
          asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
          ptx::fence_acq_rel_gpu();
          const bool gl = st.epilogue == TS_EPI_GELU;
          const bool rl = st.epilogue == TS_EPI_RELU;
          T* out = crow + col0;
          // kPC chunks (16 columns each) at a time: first the z - 1 planes' 16 floats per
          // chunk for this thread's row are loaded and summed (kPC x 4 float4 loads in
          // flight per lane: the loop is bound by loaded L2 latency, so bytes in flight set
          // its speed), then each chunk's accumulator is read from TMEM, added, activated
          // and stored.
#ifndef TS_OWNER_CHUNKS
#define TS_OWNER_CHUNKS 3
#endif
          constexpr int kPC = TS_OWNER_CHUNKS;
#pragma unroll 1
          for (int j = 0; j <= wide; ++j) {
            const int lo = max(eg * span, j * hn), hi = min((eg + 1) * span, (j + 1) * hn);
#pragma unroll 1
            for (int x0 = lo; x0 < hi; x0 += 16 * kPC) {
              float4 pa[kPC][4];
#pragma unroll
              for (int c = 0; c < kPC; ++c)
#pragma unroll
                for (int q = 0; q < 4; ++q) pa[c][q] = make_float4(0.f, 0.f, 0.f, 0.f);
              if (mine_ok) {
#pragma unroll 1
                for (int z = 0; z < nparts; ++z) {
#pragma unroll
                  for (int c = 0; c < kPC; ++c) {
                    if (x0 + 16 * c >= hi) break;
                    const float4* s4 = reinterpret_cast<const float4*>(
                        planes + static_cast<size_t>(z) * pstride +
                        (static_cast<size_t>((x0 + 16 * c) / 16) * 512 + rl_row) * 4);
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                      const float4 v = __ldcg(s4 + q * 128);
                      pa[c][q].x += v.x;
                      pa[c][q].y += v.y;
                      pa[c][q].z += v.z;
                      pa[c][q].w += v.w;
                    }
                  }
                }
              }
#pragma unroll
              for (int c = 0; c < kPC; ++c) {
                const int x = x0 + 16 * c;
                if (x >= hi) break;
                uint32_t r[16];
                ptx::tmem_ld_32x32b_x16(tcol(x), r);
                ptx::tmem_ld_wait();
                uint32_t pk[8];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  float v0 = __uint_as_float(r[4 * q]) + pa[c][q].x;
                  float v1 = __uint_as_float(r[4 * q + 1]) + pa[c][q].y;
                  float v2 = __uint_as_float(r[4 * q + 2]) + pa[c][q].z;
                  float v3 = __uint_as_float(r[4 * q + 3]) + pa[c][q].w;
                  if (gl) {
                    gelu2(v0, v1);
                    gelu2(v2, v3);
                  } else if (rl) {
                    v0 = relu(v0);
                    v1 = relu(v1);
                    v2 = relu(v2);
                    v3 = relu(v3);
                  }
                  pk[2 * q] = pack2<T>(v0, v1);
                  pk[2 * q + 1] = pack2<T>(v2, v3);
                }
                if (row_ok) {
                  if (v8ok) {
                    ptx::st_global_v8(out + x, pk);
                  } else {
                    uint4* d = reinterpret_cast<uint4*>(out + x);
                    d[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                    d[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
                  }
                }
              }
            }
            release_slot(j);
          }
        }
      } else if (t.z > 1 && !(C::kChunked && !QD && st.red_mma && !bal && t.tz == t.z - 1 &&
                                !((p.flags >> 29) & 1))) {
        // (a tensor-core-reduced owner slice — its accumulator already holds every slice —
        // takes the plain epilogue below)
        // Split-K slice (the reference's z > 1) of a normal tile: publish this CTA's fp32
        // partial rows, count arrivals per (tile, CTA); the last slice to arrive sums all
        // partials, applies the epilogue and stores. Every slice still posts once below
        // (consumers wait for expected x z), and each post follows its own stores, so
        // the count only reaches its target after the summing slice has stored.
        const int tile_id = t.tx * st.grid_y + t.ty;
        const int rl_row = ew * 32 + lane;  // this thread's row inside the CTA's 128
        // partial plane of one CTA: [acc_cols / 32 chunks][128 rows][32 floats], so a
        // warp's 32 rows of one chunk are 4 KB contiguous (coalesced writes and reads)
        const size_t plane = static_cast<size_t>(128) * acc_cols;
        float* mine = st.ws + (static_cast<size_t>(tile_id * t.z + t.tz) * (CG * NP) + qrank) * plane;
        const int span = acc_cols / G;
        // only rows < m carry data (small batch: a 128-row tile may hold a single row)
        const int row0 = t.tx * C::kTileM + static_cast<int>(rank) * 128;
        const int valid = st.m - row0 < 128 ? (st.m - row0 > 0 ? st.m - row0 : 0) : 128;
#pragma unroll 1
        for (int j = 0; j <= wide; ++j) {
          const int lo = max(eg * span, j * hn), hi = min((eg + 1) * span, (j + 1) * hn);
#pragma unroll 1
          for (int x = lo; x < hi && ew * 32 < valid; x += 32) {  // warp-uniform skip
            uint32_t r[32];
            ptx::tmem_ld_32x32b_x32(tcol(x), r);
            ptx::tmem_ld_wait();
            if constexpr (C::kChunked) {
              // plane rows of this warp are 32 consecutive 128-B rows of chunk x / 32
              float* wbase = mine + (static_cast<size_t>(x / 32) * 128 + ew * 32) * 32;
              stage_rows(r, [&](int rr, int g) -> uint4* {
                return ew * 32 + rr < valid ? reinterpret_cast<uint4*>(wbase + rr * 32 + g * 4)
                                            : nullptr;
              });
            } else if (rl_row < valid) {
              float* dst = mine + (static_cast<size_t>(x / 32) * 128 + rl_row) * 32;
#pragma unroll
              for (int q = 0; q < 4; ++q) ptx::st_global_v8(dst + 8 * q, r + 8 * q);
            }
          }
          release_slot(j);
        }
        __threadfence();
        asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
        if (threadIdx.x == 128 && uleader && p.trace != nullptr)  // partials written (ext.)
          trace_now(p, 9, t.s, t.tb, -1, -1, -1, -1, t.tx, t.ty, t.tz);
        if (threadIdx.x == 128) {
          const int half_id = tile_id * CG * NP + static_cast<int>(qrank);
          const int old = atomicAdd(&st.cnt[half_id], 1);
          *split_flag = (old == t.z - 1);
          if (old == t.z - 1) st.cnt[half_id] = 0;  // restore the zero invariant
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
        if (*split_flag) {
          ptx::fence_acq_rel_gpu();
          // Reduction, warp-cooperative: one step = 4 rows x 32 columns of one chunk
          // (512 B per slice, lane l: row r0 + l / 8, columns (l % 8) * 4 .. + 4).
          const float* base = st.ws + static_cast<size_t>(tile_id) * t.z * (CG * NP) * plane +
                              static_cast<size_t>(qrank) * plane;
          const bool gl = st.epilogue == TS_EPI_GELU;
          const bool rl = st.epilogue == TS_EPI_RELU;
          const int nr4 = (valid + 3) / 4;          // 4-row groups holding data
          const int steps = (acc_cols / 32) * nr4;  // chunks x row groups
          auto emit = [&](int sidx, float4 s) {
            const int chunk = sidx / nr4, r0 = (sidx % nr4) * 4;
            float o[4] = {s.x, s.y, s.z, s.w};
            if (gl) {
              gelu2(o[0], o[1]);
              gelu2(o[2], o[3]);
            } else if (rl) {
#pragma unroll
              for (int q = 0; q < 4; ++q) o[q] = relu(o[q]);
            }
            const int grow = row0 + r0 + (lane >> 3);
            if (grow < st.m) {
              T* dst = reinterpret_cast<T*>(st.c) + static_cast<size_t>(grow) * st.ldc +
                       col0 + chunk * 32 + (lane & 7) * 4;
              *reinterpret_cast<uint2*>(dst) = make_uint2(pack2<T>(o[0], o[1]), pack2<T>(o[2], o[3]));
            }
          };
          const size_t zs = static_cast<size_t>(CG * NP) * plane;
          const int ss = kEpiWarps;
          const uint64_t pol_ef =
              (p.flags >> 26) & 1 ? ptx::policy_evict_normal() : ptx::policy_evict_first();
          // ~16 float4 loads in flight per lane for the common slice counts (diagnostic
          // flag bit 20 forces the generic loop)
          const int zsel = (p.flags >> 20) & 1 ? 0 : t.z;
          if (zsel == 2) {
#pragma unroll 1
            for (int s0 = warp - 4; s0 < steps; s0 += ss * 8)
              reduce_split_steps<2, 8>(base, zs, s0, ss, steps, nr4, lane, pol_ef, emit);
          } else if (zsel == 3) {
#pragma unroll 1
            for (int s0 = warp - 4; s0 < steps; s0 += ss * 5)
              reduce_split_steps<3, 5>(base, zs, s0, ss, steps, nr4, lane, pol_ef, emit);
          } else if (zsel == 4) {
#pragma unroll 1
            for (int s0 = warp - 4; s0 < steps; s0 += ss * 4)
              reduce_split_steps<4, 4>(base, zs, s0, ss, steps, nr4, lane, pol_ef, emit);
          } else {
          // generic slice count: kSB steps per iteration, 4 slices' loads at a time
          constexpr int kSB = C::kChunked ? 2 : 4;
#pragma unroll 1
          for (int s0 = warp - 4; s0 < steps; s0 += kEpiWarps * kSB) {
            float4 a[kSB];
#pragma unroll
            for (int j = 0; j < kSB; ++j) a[j] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 1
            for (int z0 = 0; z0 < t.z; z0 += 4) {
              float4 v[kSB][4];
#pragma unroll
              for (int j = 0; j < kSB; ++j) {
                const int sidx = s0 + j * kEpiWarps;
                const size_t off =
                    (static_cast<size_t>(sidx / nr4) * 128 + (sidx % nr4) * 4) * 32 + lane * 4;
#pragma unroll
                for (int zz = 0; zz < 4; ++zz)
                  v[j][zz] = (sidx < steps && z0 + zz < t.z)
                                 ? __ldcg(reinterpret_cast<const float4*>(base + (z0 + zz) * zs + off))
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
              }
#pragma unroll
              for (int j = 0; j < kSB; ++j) {
#pragma unroll
                for (int zz = 0; zz < 4; ++zz) {
                  a[j].x += v[j][zz].x;
                  a[j].y += v[j][zz].y;
                  a[j].z += v[j][zz].z;
                  a[j].w += v[j][zz].w;
                }
              }
            }
#pragma unroll
            for (int j = 0; j < kSB; ++j) {
              const int sidx = s0 + j * kEpiWarps;
              if (sidx >= steps) break;
              emit(sidx, a[j]);
            }
          }
          }
        }
      } else if (st.epilogue == TS_EPI_SWIGLU) {
        // gate = accumulator columns [0, acc_cols/2), up = the matching upper half; each
        // column group stores its 1/G of the output columns
        const int half = acc_cols / 2;
        const int span = half / G;
        T* out = crow + (QD ? (2 * t.ty + static_cast<int>(pair)) * half : t.ty * half) + eg * span;
#pragma unroll 1
        for (int cc = 0; cc < span / 32; ++cc) {
          const int x = eg * span + cc * 32;
          uint32_t gr[32], ur[32];
          ptx::tmem_ld_32x32b_x32(tcol(x), gr);
          ptx::tmem_ld_32x32b_x32(tcol(half + x), ur);
          ptx::tmem_ld_wait();
          uint32_t pk[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            float g0 = __uint_as_float(gr[2 * j]), g1 = __uint_as_float(gr[2 * j + 1]);
            float u0 = __uint_as_float(ur[2 * j]), u1 = __uint_as_float(ur[2 * j + 1]);
            pk[j] = pack2<T>(silu(g0) * u0, silu(g1) * u1);
          }
          if (row_ok) store_row32<T>(out + cc * 32, pk, v8ok);
        }
        release_tmem();
      } else {
        T* out = crow + col0;
        const bool gl = st.epilogue == TS_EPI_GELU;
        const bool rl = st.epilogue == TS_EPI_RELU;
        // Column group eg stores accumulator columns [eg * span, (eg + 1) * span); slot
        // by slot, so a slot is handed back to the MMA warp as soon as every group is
        // done with it (a group arrives on a slot it does not read right away).
        const int span = acc_cols / G;
        // 16 accumulator columns -> activation -> 16-bit -> one 32-B row segment
        auto emit16 = [&](int x, const uint32_t (&r)[16]) {
          uint32_t pk[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            float v0 = __uint_as_float(r[2 * q]), v1 = __uint_as_float(r[2 * q + 1]);
            if (gl) {
              gelu2(v0, v1);
            } else if (rl) {
              v0 = relu(v0);
              v1 = relu(v1);
            }
            pk[q] = pack2<T>(v0, v1);
          }
          if (row_ok) {
            if (v8ok) {
              ptx::st_global_v8(out + x, pk);
            } else {
              uint4* d = reinterpret_cast<uint4*>(out + x);
              d[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
              d[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
            }
          }
        };
#pragma unroll 1
        for (int j = 0; j <= wide; ++j) {
          const int lo = max(eg * span, j * hn), hi = min((eg + 1) * span, (j + 1) * hn);
          // 16 columns per TMEM load. Measured per 256 x 512 tile drain (M=1024 probe):
          // this loop 8.1 us; 32-column loads with the f32 tanh 9.2 us; a two-deep
          // software pipeline of TMEM loads 11 us (it spills at the 168-register cap of the
          // 384-thread pair kernel; with 4 epilogue warps and no cap, 16 us); staging
          // 64-column chunks through shared memory for 512-B coalesced stores 14 us.
#pragma unroll 1
          for (int x = lo; x < hi; x += 16) {
            uint32_t ra[16];
            if ((p.flags >> 24) & 1) {  // diagnostic only (bit 24): no TMEM reads
#pragma unroll
              for (int q = 0; q < 16; ++q) ra[q] = 0;
            } else {
              ptx::tmem_ld_32x32b_x16(tcol(x), ra);
              ptx::tmem_ld_wait();
            }
            emit16(x, ra);
          }
          if constexpr (C::kHaloOk) {
            if (st.hmode && st.hsub > 1) {
              // a halo-conv item's second sub-tile: item rows 128 + ..., accumulator
              // columns [64, 128) of the same buffer
              const int px = halo_pixel(st, halo_tile(st, t.tx), 128 + ew * 32 + lane);
              row_ok = px >= 0;
              out = reinterpret_cast<T*>(st.c) + static_cast<size_t>(px < 0 ? 0 : px) * st.ldc +
                    col0;
#pragma unroll 1
              for (int x = lo; x < hi; x += 16) {
                uint32_t ra[16];
                ptx::tmem_ld_32x32b_x16(t_lane + 64 + x, ra);
                ptx::tmem_ld_wait();
                emit16(x, ra);
              }
            }
          }
          release_slot(j);
        }
      }
      }  // normal layout
      if (threadIdx.x == 128 && uleader && p.trace != nullptr)  // epilogue stores issued
        trace_now(p, 8, t.s, t.tb, -1, -1, -1, -1, t.tx, t.ty, t.tz);
      // stage.post(): every epilogue thread's stores (of both CTAs of a pair)
      // happen-before the release below.
      asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
      // single-CTA kernels, untraced items without a last-arriver dot or row gate: the
      // post warp makes the post (see above)
      const bool apost = CG == 1 && any_post && p.trace == nullptr && st.dot_dep < 0 &&
                         st.out_sem == nullptr && st.n_out_deps > 0 && brole != 1;
      if (threadIdx.x == 128 && apost) {
        const int ps = npost % kPostRing;
        ptx::mbar_wait(&post_empty[ps], ((npost / kPostRing) & 1) ^ 1);
        post_req[ps] = g;
        ptx::mbar_arrive(&post_full[ps]);
        ++npost;
      } else if (threadIdx.x == 128) {
        if (CG == 2 && !uleader) {
          __threadfence();
          ptx::mbar_arrive_remote(ptx::mapa(&peer_done[local % kPeerRing], 0));
        } else {
          if constexpr (CG == 2)
            ptx::mbar_wait_cluster(&peer_done[local % kPeerRing], (local / kPeerRing) & 1);
          const uint64_t tnow = p.trace ? ptx::global_timer() : 0;  // traced launches only
          // a balanced segment that does not start its tile only contributed a partial:
          // the tile is posted once, by its head segment after the reduction
          const bool posts = brole != 1;
          if (st.n_out_deps > 0 && posts) {
            // release: the epilogue's stores (ordered before this thread by the named
            // barrier) become visible before the post; diagnostic flag bit 22 times the
            // post without the full fence
            if (!((p.flags >> 22) & 1)) __threadfence();
            ptx::fence_proxy_async_global();
            for (int i = 0; i < st.n_out_deps; ++i) {
              const int d = st.out_deps[i];
              const DepParams& dp = p.dep[d];
              const int idx = post_target(dp.policy, dp.param, t.tx, t.ty,
                                          Grid3{dp.pgx, dp.pgy, dp.pgz});
              // an all-reduce consumer reads this semaphore (and the tile) from peer GPUs
              const bool sys = p.st[dp.consumer].kind == kStageAllReduce;
              if (sys) __threadfence_system();
              int old = 0;
              if (sys) {
                old = ptx::atom_add_release_sys(dp.sem + idx, 1);
              } else if (p.trace != nullptr || d == st.dot_dep) {
                old = ptx::atom_add_release_gpu(dp.sem + idx, 1);  // the value is used below
              } else {
                ptx::red_add_release_gpu(dp.sem + idx, 1);
              }
              ptx::red_add_release_gpu(p.scratch + kDoneBase + d, 1);
              trace_event(p, tnow, 3, t.s, t.tb, -1, d, idx, old + 1, t.tx, t.ty, t.tz);
              if (d == st.dot_dep) {
                // Which dot tiles of this row did this post complete? (the wait of tile
                // (x, c) at k-step 0 is on semaphore idx and now reached its threshold)
                const StageParams& sd = p.st[dp.consumer];
                // time read after the atomic: later than every post it counted
                const uint64_t tfire = p.trace ? ptx::global_timer() : 0;
                int n = 0;
                for (int c = 0; c < sd.grid_y; ++c) {
                  Wait w = consumer_wait(dp.policy, dp.param, t.tx, c, 0,
                                         Grid3{dp.pgx, dp.pgy, dp.pgz}, dp.pgz);
                  if (w.sem == idx && w.expected == old + 1) {
                    const int tb = atomicAdd(&p.scratch[4], 1);
                    dot_list[n] = c;
                    dot_list[32 + n] = tb;
                    ++n;
                    // the dot tile is scheduled the moment its wait is satisfied
                    trace_event(p, tfire, 0, dp.consumer, tb, -1, -1, -1, -1, t.tx, c);
                    trace_event(p, tfire, 1, dp.consumer, tb, 0, d, idx, w.expected, t.tx, c);
                    trace_event(p, tfire, 2, dp.consumer, tb, 0, d, idx, w.expected, t.tx, c);
                  }
                }
                *dot_count = n;
                if (dsplit) {
                  // hand the list to the peer CTA, which computes the lower 128 rows
                  for (int i = 0; i < n; ++i) {
                    ptx::st_cluster_u32(ptx::mapa(&dot_list[i], 1), static_cast<uint32_t>(dot_list[i]));
                    ptx::st_cluster_u32(ptx::mapa(&dot_list[32 + i], 1),
                                        static_cast<uint32_t>(dot_list[32 + i]));
                  }
                  ptx::st_cluster_u32(ptx::mapa(dot_count, 1), static_cast<uint32_t>(n));
                  ptx::mbar_arrive_remote(ptx::mapa(dot_msg, 1));
                }
              }
            }
          }
          if (st.out_sem != nullptr && posts) {
            // the tile's rows (both CTAs of a pair) are stored: let a copy stream read
            // them (a PCIe agent, hence system scope)
            __threadfence_system();
            atomicAdd(st.out_sem + t.tx, 1);
          }
          trace_event(p, tnow, 4, t.s, t.tb, -1, -1, -1, -1, t.tx, t.ty, t.tz);
        }
      }
      if (st.dot_dep >= 0 && (leader || dsplit)) {
        // last-arriver dot tiles released by this tile's posts; split over a CTA pair the
        // leader computes rows [0, 128) of each and the peer (told by the leader's list)
        // rows [128, 256), and the leader posts once the peer's rows are stored
        if (!leader) {
          ptx::mbar_wait_cluster(dot_msg, dmsg & 1);
          ++dmsg;
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
        const int n = *dot_count;
        const int ds = p.dep[st.dot_dep].consumer;
        const int half = dsplit ? (leader ? 0 : 1) : -1;
        for (int i = 0; i < n; ++i) run_dot_rows(ds, t.tx, dot_list[i], dot_list[32 + i], half);
        if (leader) {
          if (dsplit && n > 0) {
            if (threadIdx.x == 128) ptx::mbar_wait_cluster(dot_done, ddone & 1);
            ++ddone;
          }
          for (int i = 0; i < n; ++i) post_dot(ds, t.tx, dot_list[i], dot_list[32 + i]);
        } else if (n > 0 && threadIdx.x == 128) {
          __threadfence();
          ptx::mbar_arrive_remote(ptx::mapa(dot_done, 0));
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
        if (leader && threadIdx.x == 128) *dot_count = 0;
      }
      ++local;
      u += 1 + wide;
    }
    if (CG == 1 && threadIdx.x == 128 && any_post) {  // end of the post warp's queue
      const int ps = npost % kPostRing;
      ptx::mbar_wait(&post_empty[ps], ((npost / kPostRing) & 1) ^ 1);
      post_req[ps] = -1;
      ptx::mbar_arrive(&post_full[ps]);
    }
  }

  // ---- teardown: free TMEM; the last CTA out restores the zero invariant -------------
  ptx::tc_fence_before();
  if constexpr (CG == 2) {
    ptx::cluster_sync();
  } else {
    __syncthreads();
  }
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<C::kTmemCols, CG>(tmem_base);
  }
  if (threadIdx.x == 0) {
    __threadfence();
    const int prev = atomicAdd(&p.ctl[1], 1);
    *last_flag = (prev == static_cast<int>(gridDim.x) - 1);
  }
  __syncthreads();
  if (*last_flag) {
    __threadfence();
    // All-reduce stage in this launch: this rank's buffer is final once every owner (on
    // every rank) has counted its tiles into the done counter. The counter and the
    // producer -> all-reduce semaphores are monotone (epoch e waits for e x count) and
    // never reset here: a reset could race with a faster peer's next launch reading them.
    bool ar_here = false;
    for (int s = 0; s < p.n_stages; ++s)
      if (p.st[s].kind == kStageAllReduce && p.st[s].item_begin >= p.item_lo &&
          p.st[s].item_end <= p.item_hi)
        ar_here = true;
    if (ar_here) {
      if (threadIdx.x == 0) sem_spin_sys(p, p.peers.done[p.peers.rank], p.ar_done * p.peers.epoch);
      __syncthreads();
    }
    if (p.coresident) {
      // One stage per launch: the consumer's launch is the last reader of its incoming
      // dependencies' semaphores and watermarks, and of its producers' started flags.
      const int s = stage_of(p, p.item_lo);
      for (int d = 0; d < p.n_deps; ++d) {
        if (p.dep[d].consumer != s) continue;
        if ((p.flags & TS_FLAG_KEEP_SEMS) == 0)
          for (int i = threadIdx.x; i < p.dep[d].sem_n; i += C::kThreads) p.dep[d].sem[i] = 0;
        if (threadIdx.x == 0) {
          p.scratch[kDoneBase + d] = 0;
          p.scratch[kCtlBase + kCtlInts * p.dep[d].producer + 2] = 0;
        }
      }
      if (threadIdx.x == 0) {
        p.ctl[0] = 0;
        p.ctl[1] = 0;
        bool waited_on = false;  // nothing consumes this stage: nobody else resets its flag
        for (int d = 0; d < p.n_deps; ++d) waited_on = waited_on || p.dep[d].producer == s;
        if (!waited_on) p.ctl[2] = 0;
      }
      __threadfence();
    } else {
      if ((p.flags & TS_FLAG_KEEP_SEMS) == 0) {
        for (int d = 0; d < p.n_deps; ++d) {
          if (p.st[p.dep[d].consumer].kind == kStageAllReduce) continue;  // epoch-monotone
          for (int i = threadIdx.x; i < p.dep[d].sem_n; i += C::kThreads) p.dep[d].sem[i] = 0;
        }
      }
      if (threadIdx.x == 0) {
        p.scratch[0] = 0;
        p.scratch[1] = 0;
        p.scratch[4] = 0;  // last-arriver dot claim counter
      }
      if (threadIdx.x < TS_MAX_DEPS) p.scratch[kDoneBase + threadIdx.x] = 0;  // watermarks
      __threadfence();
    }
  }
}

}  // namespace ts
