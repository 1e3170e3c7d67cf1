// ts_abi.cu — the extern "C" boundary of libtilesync_b200.so (declared in
// include/tilesync.h). Host-side validation mirrors the reference's structural checks
// (validate_scenario, /root/reference/pkg/src/tilesync_sim/engine.py:134-170; check_policy,
// policies.py:102-112) so errors surface as the same exception types before any launch.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <mutex>
#include <string>

#include "tilesync.h"
#include "ts_launch.h"
#include "ts_policy.cuh"

namespace ts_host {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(TS_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

}  // namespace ts_host

namespace {

using ts_host::cuda_fail;
using ts_host::fail;
using ts_host::launch_one;
using ts_host::prepare;

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// Encoded tensor maps, keyed by everything that enters the encoding (pointer, shape,
// stride, dtype, box, kind): ts_chain_launch re-derives every map of a chain on each call,
// and cuTensorMapEncode* costs microseconds of host time per map against 30-70 us chains
// ("may cache TMA descriptors keyed by (ptr, shape, stride)"). A small
// per-thread table with round-robin replacement; an entry is only reused on an exact key
// match, so a freed-and-reallocated buffer at the same address with the same geometry maps
// to the same (still correct) descriptor.
struct TmapKey {
  const void* ptr;
  long long d[6];
  bool operator==(const TmapKey& o) const {
    if (ptr != o.ptr) return false;
    for (int i = 0; i < 6; ++i)
      if (d[i] != o.d[i]) return false;
    return true;
  }
};

struct TmapCache {
  static constexpr int kEntries = 64;
  TmapKey key[kEntries];
  CUtensorMap map[kEntries];
  int used = 0, next = 0;
  const CUtensorMap* find(const TmapKey& k) const {
    for (int i = 0; i < used; ++i)
      if (key[i] == k) return &map[i];
    return nullptr;
  }
  void put(const TmapKey& k, const CUtensorMap& m) {
    const int i = used < kEntries ? used++ : next;
    next = (i + 1) % kEntries;
    key[i] = k;
    map[i] = m;
  }
};

thread_local TmapCache g_tmaps;

// K-major [rows, k] 16-bit matrix, leading dimension `ld` elements, box {64, box_rows}.
int make_tmap(CUtensorMap* m, const void* ptr, int rows, int k, int ld, int dtype,
              int box_rows) {
  const TmapKey key{ptr, {0, rows, k, ld, dtype, box_rows}};
  if (const CUtensorMap* hit = g_tmaps.find(key)) {
    *m = *hit;
    return TS_OK;
  }
  EncodeTiledFn enc = encode_fn();
  if (!enc) return fail(TS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (driver too old?)");
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(k), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 2};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(ts::kBK), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, dtype == TS_DTYPE_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                             : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                   2, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(TS_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d) rows=%d k=%d ld=%d", (int)r,
                rows, k, ld);
  g_tmaps.put(key, *m);
  return TS_OK;
}

// Split-K partial planes of a CTA-pair 256-wide stage: the fp32 workspace viewed as
// [rows][cols] (rows = planes x 128), 32-column x 128-row boxes with 128-B swizzle — the A
// operand of the owner slice's reduction MMAs (kind::tf32).
int make_tmap_ws(CUtensorMap* m, const float* ptr, long long rows, int cols) {
  const TmapKey key{ptr, {2, rows, cols, 0, 0, 0}};
  if (const CUtensorMap* hit = g_tmaps.find(key)) {
    *m = *hit;
    return TS_OK;
  }
  EncodeTiledFn enc = encode_fn();
  if (!enc) return fail(TS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (driver too old?)");
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * 4};
  cuuint32_t box[2] = {32, 128};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(TS_ERR_CUDA, "cuTensorMapEncodeTiled (workspace) failed (%d) rows=%lld cols=%d",
                (int)r, rows, cols);
  g_tmaps.put(key, *m);
  return TS_OK;
}

// Halo-staged convolution window: NHWC input as a 4-D (C, W, H, N) tensor, box (64
// channels, bw pixels, bh rows, 1 image), 128-B swizzle (one pixel = one 128-B row); boxes
// start at column -1 / row -1, the out-of-bounds fill supplies the zero padding.
int make_tmap_window(CUtensorMap* m, const void* ptr, int n, int h, int w, int ldc_px, int dtype,
                     int bw, int bh) {
  const TmapKey key{ptr, {3, n, h, w, static_cast<long long>(ldc_px) * 4 + dtype,
                          (static_cast<long long>(bw) << 16) | bh}};
  if (const CUtensorMap* hit = g_tmaps.find(key)) {
    *m = *hit;
    return TS_OK;
  }
  EncodeTiledFn enc = encode_fn();
  if (!enc) return fail(TS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (driver too old?)");
  cuuint64_t dims[4] = {64, static_cast<cuuint64_t>(w), static_cast<cuuint64_t>(h),
                        static_cast<cuuint64_t>(n)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(ldc_px) * 2,
                           static_cast<cuuint64_t>(ldc_px) * 2 * w,
                           static_cast<cuuint64_t>(ldc_px) * 2 * w * h};
  cuuint32_t box[4] = {64, static_cast<cuuint32_t>(bw), static_cast<cuuint32_t>(bh), 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(m, dtype == TS_DTYPE_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                             : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                   4, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(TS_ERR_CUDA, "cuTensorMapEncodeTiled (conv window) failed (%d) n=%d h=%d w=%d", (int)r,
                n, h, w);
  g_tmaps.put(key, *m);
  return TS_OK;
}

using EncodeIm2colFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const int*,
                                    const int*, cuuint32_t, cuuint32_t, const cuuint32_t*,
                                    CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeIm2colFn encode_im2col_fn() {
  static EncodeIm2colFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeIm2colFn>(p);
  });
  return fn;
}

// im2col map over an NHWC activation tensor for a 3x3, stride-1, padding-1 convolution:
// the pixel bounding box spans [-1, H-2] x [-1, W-2] (lower corner -pad, upper corner
// pad - (R-1)), so output pixel (p, q) is box coordinate (p-1, q-1) and filter tap (r, s)
// is the im2col offset; each load is `pixels` consecutive output pixels x 64 channels.
int make_tmap_im2col(CUtensorMap* m, const void* ptr, int n, int h, int w, int c, int ldc_px,
                     int dtype, int pixels) {
  // kind 1 (im2col); n, h, w, c and the pixel stride fully determine the map
  const TmapKey key{ptr, {1 + (static_cast<long long>(pixels) << 8), n, h, w, c,
                          static_cast<long long>(ldc_px) * 4 + dtype}};
  if (const CUtensorMap* hit = g_tmaps.find(key)) {
    *m = *hit;
    return TS_OK;
  }
  EncodeIm2colFn enc = encode_im2col_fn();
  if (!enc) return fail(TS_ERR_CUDA, "cuTensorMapEncodeIm2col unavailable (driver too old?)");
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(c), static_cast<cuuint64_t>(w),
                        static_cast<cuuint64_t>(h), static_cast<cuuint64_t>(n)};
  const cuuint64_t px = static_cast<cuuint64_t>(ldc_px) * 2;
  cuuint64_t strides[3] = {px, px * w, px * w * h};
  int lower[2] = {-1, -1};
  int upper[2] = {-1, -1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(m, dtype == TS_DTYPE_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                             : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                   4, const_cast<void*>(ptr), dims, strides, lower, upper, ts::kBK,
                   static_cast<cuuint32_t>(pixels), estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(TS_ERR_CUDA, "cuTensorMapEncodeIm2col failed (%d) n=%d h=%d w=%d c=%d", (int)r, n,
                h, w, c);
  g_tmaps.put(key, *m);
  return TS_OK;
}

int sm_count() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  return n;
}

template <typename T>
int launch_bn1(int bn, const ts::ChainParams& p, int units, cudaStream_t s) {
  switch (bn) {
    case 64: return launch_one<64, 1, T, false, false>(p, units, s);
    case 128: return launch_one<128, 1, T, false, false>(p, units, s);
    case 256: return launch_one<256, 1, T, false, false>(p, units, s);
  }
  return fail(TS_ERR_VALUE, "tile_n must be 64, 128 or 256 (got %d)", bn);
}

template <typename T>
int launch_bn2(int bn, const ts::ChainParams& p, int units, cudaStream_t s) {
  switch (bn) {
    case 128: return launch_one<128, 2, T, false, false>(p, units, s);
    case 256: return launch_one<256, 2, T, false, false>(p, units, s);
  }
  return fail(TS_ERR_VALUE, "cta_group 2 needs tile_n 128 or 256 (got %d)", bn);
}

template <typename T>
int launch_swapped(int bn, const ts::ChainParams& p, int units, cudaStream_t s) {
  switch (bn) {
    case 32: return launch_one<32, 1, T, true, false>(p, units, s);
    case 64: return launch_one<64, 1, T, true, false>(p, units, s);
    case 128: return launch_one<128, 1, T, true, false>(p, units, s);
    case 256: return launch_one<256, 1, T, true, false>(p, units, s);
  }
  return fail(TS_ERR_VALUE, "swapped tile_n must be 32, 64, 128 or 256 (got %d)", bn);
}

int launch_dispatch(int bn, int cg, int swap, int dtype, const ts::ChainParams& p, int units,
                    cudaStream_t s, int np = 1) {
  if (np == 2) {  // validated: cta_group 2, tile_n 256, normal layout
    return dtype == TS_DTYPE_BF16 ? launch_one<256, 2, __nv_bfloat16, false, true>(p, units, s)
                                  : launch_one<256, 2, __half, false, true>(p, units, s);
  }
  if (swap) {
    return dtype == TS_DTYPE_BF16 ? launch_swapped<__nv_bfloat16>(bn, p, units, s)
                                  : launch_swapped<__half>(bn, p, units, s);
  }
  if (cg == 2) {
    if (bn == 64) return fail(TS_ERR_VALUE, "cta_group 2 needs tile_n >= 128");
    return dtype == TS_DTYPE_BF16 ? launch_bn2<__nv_bfloat16>(bn, p, units, s)
                                  : launch_bn2<__half>(bn, p, units, s);
  }
  return dtype == TS_DTYPE_BF16 ? launch_bn1<__nv_bfloat16>(bn, p, units, s)
                                : launch_bn1<__half>(bn, p, units, s);
}

int tile_n_of(const ts_chain_desc* d) { return d->tile_n == 0 ? 256 : d->tile_n; }
int cluster_pairs_of(const ts_chain_desc* d) { return d->cluster_pairs == 0 ? 1 : d->cluster_pairs; }
int cta_group_of(const ts_chain_desc* d) {
  if (d->swap_ab) return 1;
  return d->cta_group == 0 ? 2 : d->cta_group;
}

// 1 if GeMM/conv stage `st` uses two MMAs per K-block step (CTA-pair tiles of
// ts_stage_desc.tile_n = 512: 2 x 256 columns, or 384: 2 x 192 columns), 0 for the
// chain's tile width, -1 if its tile_n is not allowed.
int stage_wide(const ts_stage_desc& st, int bn, int cg, int swap) {
  if (st.tile_n == 0 || st.tile_n == (swap ? 128 : bn)) return 0;
  if ((st.kind == TS_STAGE_GEMM || st.kind == TS_STAGE_CONV2D) && !swap && cg == 2 && bn == 256 &&
      (st.tile_n == 512 || st.tile_n == 384))
    return 1;
  return -1;
}

// Columns per MMA (and per TMEM accumulator slot) of stage `st`.
int stage_half_n(const ts_stage_desc& st, int bn, int cg, int swap) {
  return stage_wide(st, bn, cg, swap) > 0 ? st.tile_n / 2 : bn;
}

// Output columns one tile of stage `st` writes (the producer "column tile" width that a
// consumer k-step covers).
int out_tile_cols(const ts_stage_desc& st, int bn, int cg, int swap) {
  if (swap) return 128;
  const int w = stage_wide(st, bn, cg, swap) > 0 ? st.tile_n : bn;
  return st.epilogue == TS_EPI_SWIGLU ? w / 2 : w;
}

// Validate the descriptor and fill kernel parameters (everything but tensor maps when
// `with_tmaps` is false, so ts_chain_grid works without a GPU).
int build_params(const ts_chain_desc* d, ts::ChainParams* p, bool with_tmaps) {
  if (d == nullptr) return fail(TS_ERR_VALUE, "null chain descriptor");
  const int bn = tile_n_of(d);
  const int swap = d->swap_ab ? 1 : 0;
  if (swap) {
    if (bn != 32 && bn != 64 && bn != 128 && bn != 256)
      return fail(TS_ERR_VALUE, "swapped tile_n must be 32, 64, 128 or 256 (got %d)", d->tile_n);
    if (d->cta_group == 2) return fail(TS_ERR_VALUE, "swap_ab tiles use cta_group 1");
  } else if (bn != 64 && bn != 128 && bn != 256) {
    return fail(TS_ERR_VALUE, "tile_n must be 64, 128 or 256 (got %d)", d->tile_n);
  }
  const int cg = cta_group_of(d);
  if (cg != 1 && cg != 2) return fail(TS_ERR_VALUE, "cta_group must be 1 or 2 (got %d)", d->cta_group);
  if (cg == 2 && bn == 64) return fail(TS_ERR_VALUE, "cta_group 2 needs tile_n >= 128");
  const int np = cluster_pairs_of(d);
  if (np != 1 && np != 2) return fail(TS_ERR_VALUE, "cluster_pairs must be 0, 1 or 2 (got %d)", d->cluster_pairs);
  if (np == 2 && (cg != 2 || bn != 256 || swap))
    return fail(TS_ERR_CONFIG, "two-pair clusters need cta_group 2 and tile_n 256 (normal layout)");
  // reference-grid tile: rows of activations x columns of output
  const int tile_m = swap ? bn : 128 * cg;
  const int tile_n = swap ? 128 : bn;
  if (d->n_stages < 1 || d->n_stages > TS_MAX_STAGES)
    return fail(TS_ERR_CONFIG, "n_stages must be in [1, %d]", TS_MAX_STAGES);
  if (d->n_deps < 0 || d->n_deps > TS_MAX_DEPS)
    return fail(TS_ERR_CONFIG, "n_deps must be in [0, %d]", TS_MAX_DEPS);
  if (d->mode != TS_MODE_STREAM && d->mode != TS_MODE_FUSED && d->mode != TS_MODE_CORESIDENT)
    return fail(TS_ERR_CONFIG, "unknown mode %d", d->mode);
  std::memset(p, 0, sizeof(*p));
  p->n_stages = d->n_stages;
  p->n_deps = d->n_deps;
  p->flags = d->flags;
  p->scratch = d->scratch;
  p->ctl = d->scratch;
  p->coresident = 0;
  p->balanced = (d->flags & TS_FLAG_BALANCED) ? 1 : 0;
  // one item per claim: batching halo-conv claims (2 / 4 / 8 per atomic) measured 1-95%
  // slower once items carry two sub-tiles — the claim is not the per-item cost, the tail
  // balance is (profiles/r02y_conv_halo.txt, r02pp)
  p->claim_batch = 1;
  p->trace = static_cast<ts_trace_rec*>(d->trace);
  p->trace_cap = d->trace ? d->trace_cap : 0;
  const int dtype = d->stages[0].dtype;
  int items = 0;
  for (int s = 0; s < d->n_stages; ++s) {
    const ts_stage_desc& st = d->stages[s];
    ts::StageParams& sp = p->st[s];
    if (st.dtype != TS_DTYPE_F16 && st.dtype != TS_DTYPE_BF16)
      return fail(TS_ERR_TYPE, "stage %d: unknown dtype %d", s, st.dtype);
    if (st.dtype != dtype) return fail(TS_ERR_CONFIG, "stage %d: all stages must share a dtype", s);
    if (np == 2 && st.kind != TS_STAGE_GEMM)
      return fail(TS_ERR_CONFIG, "stage %d: two-pair clusters run GeMM stages only", s);
    if (st.kind == TS_STAGE_ATTN_DOT) {
      if (swap) return fail(TS_ERR_CONFIG, "stage %d: the attention dot stage needs normal tiles", s);
      if (st.m < 1 || st.n < bn || st.n % bn)
        return fail(TS_ERR_CONFIG, "stage %d: dot width %d must be a positive multiple of tile_n %d", s, st.n, bn);
      if (st.lda < 3 * st.n || st.lda % 8 || st.ldc < st.n || st.ldc % 8)
        return fail(TS_ERR_VALUE, "stage %d: dot needs lda >= 3n and ldc >= n (multiples of 8)", s);
      if (!st.a || !st.c) return fail(TS_ERR_VALUE, "stage %d: null operand pointer", s);
      if (st.tile_n != 0 && st.tile_n != bn)
        return fail(TS_ERR_CONFIG, "stage %d: the dot stage uses the chain's tile width", s);
      if ((reinterpret_cast<uintptr_t>(st.a) | reinterpret_cast<uintptr_t>(st.c)) & 15)
        return fail(TS_ERR_VALUE, "stage %d: operands must be 16-byte aligned", s);
      if (st.order != TS_ORDER_ROW_MAJOR && st.order != TS_ORDER_BANDED_COLUMN_MAJOR)
        return fail(TS_ERR_CONFIG, "stage %d: unsupported order for the dot stage", s);
      sp.kind = ts::kStageDot;
      sp.a = st.a;
      sp.lda = st.lda;
      sp.c = st.c;
      sp.m = st.m;
      sp.n = st.n;
      sp.ldc = st.ldc;
      sp.grid_x = (st.m + tile_m - 1) / tile_m;
      sp.grid_y = st.n / bn;  // one tile = tile_n columns = tile_n / 128 heads
      sp.splits = 1;
      sp.order = st.order;
      sp.order_stride = st.order == TS_ORDER_ROW_MAJOR ? 1 : (st.order_stride < 1 ? 1 : st.order_stride);
      sp.epilogue = TS_EPI_NONE;
      sp.item_begin = items;
      items += sp.grid_x * sp.grid_y;
      sp.item_end = items;
      sp.in_dep = -1;
      sp.n_out_deps = 0;
      sp.dot_dep = -1;
      sp.last_arriver = 0;
      continue;
    }
    if (st.kind == TS_STAGE_ALLREDUCE) {
      // tensor-parallel all-reduce of the producer's output tiles over peer memory
      const ts_peer_desc* pr = d->peers;
      if (pr == nullptr) return fail(TS_ERR_VALUE, "stage %d: the allreduce stage needs peers", s);
      if (pr->world < 1 || pr->world > TS_MAX_PEERS || pr->rank < 0 || pr->rank >= pr->world)
        return fail(TS_ERR_VALUE, "stage %d: peers world %d / rank %d invalid", s, pr->world, pr->rank);
      for (int q = 0; q < pr->world; ++q)
        if (!pr->bufs[q] || !pr->sems[q] || !pr->done[q] ||
            (reinterpret_cast<uintptr_t>(pr->bufs[q]) & 15))
          return fail(TS_ERR_VALUE, "stage %d: peer %d has a null or misaligned pointer", s, q);
      if (pr->bufs[pr->rank] != st.c)
        return fail(TS_ERR_VALUE, "stage %d: peers.bufs[rank] must be this stage's c", s);
      if (pr->epoch < 1) return fail(TS_ERR_VALUE, "stage %d: peers.epoch must be >= 1", s);
      // The epilogue stages peer vectors in the operand ring, which is idle only when no
      // GeMM item follows; a second all-reduce stage would share p->peers / p->ar_done.
      if (s != d->n_stages - 1)
        return fail(TS_ERR_CONFIG, "stage %d: the allreduce stage must be the chain's last stage", s);
      if (swap) return fail(TS_ERR_CONFIG, "stage %d: the allreduce stage needs normal tiles", s);
      int prod = -1;
      for (int i = 0; i < d->n_deps; ++i)
        if (d->deps[i].consumer == s) prod = d->deps[i].producer;
      if (prod < 0 || prod >= s || d->stages[prod].kind != TS_STAGE_GEMM)
        return fail(TS_ERR_CONFIG, "stage %d: the allreduce stage needs one earlier GeMM producer", s);
      const ts_stage_desc& pd = d->stages[prod];
      if (pd.c != st.c || pd.ldc != st.ldc || pd.m != st.m || pd.epilogue == TS_EPI_SWIGLU ||
          pd.n != st.n)
        return fail(TS_ERR_CONFIG, "stage %d: the allreduce stage sums its producer's output in place", s);
      if (st.ldc % 8) return fail(TS_ERR_VALUE, "stage %d: ldc must be a multiple of 8", s);
      const ts::StageParams& pp = p->st[prod];
      sp.kind = ts::kStageAllReduce;
      sp.c = st.c;
      sp.m = st.m;
      sp.n = st.n;
      sp.ldc = st.ldc;
      sp.grid_x = pp.grid_x;
      sp.grid_y = pp.grid_y;
      sp.ar_cols = out_tile_cols(pd, bn, cg, swap);
      sp.splits = 1;
      sp.order = TS_ORDER_ROW_MAJOR;
      sp.order_stride = 1;
      sp.epilogue = TS_EPI_NONE;
      const int tiles = pp.grid_x * pp.grid_y;
      sp.item_begin = items;
      items += (tiles - pr->rank + pr->world - 1) / pr->world;  // tiles t % world == rank
      sp.item_end = items;
      sp.in_dep = -1;
      sp.n_out_deps = 0;
      sp.dot_dep = -1;
      sp.last_arriver = 0;
      p->peers = *pr;
      p->ar_done = tiles * cg;
      continue;
    }
    if (st.kind != TS_STAGE_GEMM && st.kind != TS_STAGE_CONV2D)
      return fail(TS_ERR_TYPE, "stage %d: unknown stage kind %d", s, st.kind);
    const bool conv = st.kind == TS_STAGE_CONV2D;
    sp.kind = conv ? ts::kStageConv : ts::kStageGemm;
    if (st.epilogue < TS_EPI_NONE || st.epilogue > TS_EPI_RELU)
      return fail(TS_ERR_TYPE, "stage %d: unknown epilogue %d", s, st.epilogue);
    if (swap && st.epilogue == TS_EPI_RELU)
      return fail(TS_ERR_CONFIG, "stage %d: the ReLU epilogue needs the normal tile layout", s);
    if (conv) {
      if (swap) return fail(TS_ERR_CONFIG, "stage %d: convolutions need the normal tile layout", s);
      if (st.epilogue == TS_EPI_SWIGLU)
        return fail(TS_ERR_CONFIG, "stage %d: no SwiGLU epilogue on a convolution", s);
      if (st.conv_n < 1 || st.conv_h < 1 || st.conv_w < 1 ||
          static_cast<long long>(st.conv_n) * st.conv_h * st.conv_w != st.m)
        return fail(TS_ERR_VALUE, "stage %d: conv m=%d must equal n*h*w (%d*%d*%d)", s, st.m,
                    st.conv_n, st.conv_h, st.conv_w);
      if (st.k % 9 != 0 || (st.k / 9) % ts::kBK != 0)
        return fail(TS_ERR_CONFIG, "stage %d: conv k=%d must be 9 x Cin with Cin a multiple of %d", s,
                    st.k, ts::kBK);
      if (st.lda < st.k / 9)
        return fail(TS_ERR_VALUE, "stage %d: conv lda (pixel stride) %d < Cin %d", s, st.lda, st.k / 9);
      if (st.conv_h > 32767 || st.conv_w > 32767)
        return fail(TS_ERR_VALUE, "stage %d: image too large for the im2col map", s);
    }
    if (swap && st.epilogue == TS_EPI_SWIGLU)
      return fail(TS_ERR_CONFIG, "stage %d: the SwiGLU epilogue needs the normal tile layout", s);
    if (st.m < 1 || st.n < 1 || st.k < 1)
      return fail(TS_ERR_VALUE, "stage %d: m, n, k must be >= 1", s);
    const int wide = stage_wide(st, bn, cg, swap);
    if (wide < 0)
      return fail(TS_ERR_CONFIG, "stage %d: tile_n %d unsupported (0, %d, or 384 / 512 with "
                  "cta_group 2 and chain tile_n 256)", s, st.tile_n, tile_n);
    const int half_n = stage_half_n(st, bn, cg, swap);
    const int stage_tile_n = swap ? tile_n : half_n << wide;
    if (np == 2 && !(wide == 1 && half_n == 256))
      return fail(TS_ERR_CONFIG, "stage %d: two-pair clusters need tile_n 512 stages", s);
    if (st.n % stage_tile_n != 0)
      return fail(TS_ERR_CONFIG, "stage %d: n=%d is not a multiple of the tile width %d", s, st.n,
                  stage_tile_n);
    const int splits = st.splits < 1 ? 1 : st.splits;
    if (st.k % (ts::kBK * splits) != 0)
      return fail(TS_ERR_CONFIG, "stage %d: k=%d is not a multiple of %d x %d split(s)", s, st.k,
                  ts::kBK, splits);
    // SwiGLU needs gate and up summed before SiLU(g) * u: only the tensor-core reduction
    // (flag bit 27: the owner slice's accumulator holds the full sum before its plain
    // epilogue) supports split-K under it
    if (splits > 1 && !swap && st.epilogue == TS_EPI_SWIGLU &&
        !(((d->flags >> 27) & 1) && cg == 2 && bn == 256 && np == 1))
      return fail(TS_ERR_CONFIG, "stage %d: split-K under the SwiGLU epilogue needs the "
                  "tensor-core reduction (flag bit 27, cta_group 2, tile_n 256)", s);
    if (splits > 1 && (st.workspace == nullptr || st.counters == nullptr))
      return fail(TS_ERR_VALUE, "stage %d: split-K needs a workspace and counters", s);
    const int n_out = st.epilogue == TS_EPI_SWIGLU ? st.n / 2 : st.n;
    if ((!conv && st.lda < st.k) || st.ldb < st.k || st.ldc < n_out || st.lda % 8 || st.ldb % 8 || st.ldc % 8)
      return fail(TS_ERR_VALUE, "stage %d: leading dimensions must cover the rows and be multiples of 8", s);
    if (!st.a || !st.b || !st.c) return fail(TS_ERR_VALUE, "stage %d: null operand pointer", s);
    if ((reinterpret_cast<uintptr_t>(st.a) | reinterpret_cast<uintptr_t>(st.b) |
         reinterpret_cast<uintptr_t>(st.c)) & 15)
      return fail(TS_ERR_VALUE, "stage %d: operands must be 16-byte aligned", s);
    sp.c = st.c;
    sp.m = st.m;
    sp.n = st.n;
    sp.k = st.k;
    sp.ldc = st.ldc;
    sp.grid_x = (st.m + tile_m - 1) / tile_m;
    sp.grid_y = st.n / stage_tile_n;
    sp.wide = wide;
    sp.half_n = half_n;
    sp.in_sem = st.in_sem;
    sp.in_expected = st.in_expected;
    sp.out_sem = st.out_sem;
    if (conv) {
      sp.conv_h = st.conv_h;
      sp.conv_w = st.conv_w;
      sp.conv_cin = st.k / 9;
      sp.conv_subs = 1;  // K channel tile = 64 unless a producer's column tile sets it
      sp.halo = (st.conv_w + 1 + tile_m - 1) / tile_m;
      if (d->flags & TS_FLAG_CONV_HALO) {
        // halo-staged tiles (see StageParams::hmode): Cin = Cout = 64 on single-CTA 64-wide
        // tiles; rows mode while the window (rows the 128 positions span + 2 halo rows) fits
        // 56 KB, else one 128-position segment of a row per tile
        if (cg != 1 || bn != 64 || swap || st.k != 9 * 64 || st.n != 64 || splits != 1 ||
            st.conv_w + 2 > 256 || st.tile_n != 0)
          return fail(TS_ERR_CONFIG, "stage %d: halo-staged convolution needs Cin = Cout = 64, "
                      "cta_group 1, tile_n 64, no split-K, width <= 254", s);
        const int srow = st.conv_w + 2;
        // window space of the BN = 64 kernel: its 9 x 24 KB operand ring minus the resident
        // weight taps (9 x 8 KB)
        constexpr int kHaloWindowBytes = 9 * 24576 - 9 * 8192;
        if (srow <= 128) {
          // rows mode: a tile = the whole width-padded rows that fit 128 positions
          sp.hmode = 1;
          sp.hs = srow;
          sp.hrpt = 128 / srow < st.conv_h ? 128 / srow : st.conv_h;
          sp.hsub = 1;
          // two 128-position sub-tiles per item (rows that fit 256 positions) when their
          // window still fits two buffers and the layer still has two items per SM: one
          // claim, window, commit and accumulator hand-off per two tiles (the per-item
          // pipeline cost dominates 128 x 64 tiles; B=256 56x56x64: 325 -> 248 us)
          const int rpt2 = 256 / srow < st.conv_h ? 256 / srow : st.conv_h;
          if (rpt2 * srow > 128 &&
              kHaloWindowBytes / (((rpt2 + 2) * srow * 128 + 1023) / 1024 * 1024) >= 2 &&
              static_cast<long long>(st.conv_n) * ((st.conv_h + rpt2 - 1) / rpt2) >=
                  2LL * sm_count()) {
            sp.hrpt = rpt2;
            sp.hsub = 2;
          }
          sp.hrows = sp.hrpt + 2;
          sp.htpi = (st.conv_h + sp.hrpt - 1) / sp.hrpt;
          sp.htpr = 0;
        } else {
          sp.hmode = 2;
          sp.hsub = 1;
          sp.hs = 130;
          sp.hrows = 3;
          sp.hrpt = 1;
          sp.htpr = (st.conv_w + 127) / 128;
          // two image rows of the segment per item (a 4-row window) when two such windows
          // fit and the layer keeps two items per SM
          if (st.conv_h >= 2 && kHaloWindowBytes / ((4 * 130 * 128 + 1023) / 1024 * 1024) >= 2 &&
              static_cast<long long>(st.conv_n) * ((st.conv_h + 1) / 2) * sp.htpr >=
                  2LL * sm_count()) {
            sp.hrpt = 2;
            sp.hrows = 4;
            sp.hsub = 2;
          }
          sp.htpi = (st.conv_h + sp.hrpt - 1) / sp.hrpt * sp.htpr;
        }
        sp.hbytes = sp.hrows * sp.hs * 128;
        sp.hwin = (sp.hbytes + 1023) / 1024 * 1024;
        sp.hnb = kHaloWindowBytes / sp.hwin;  // the BN = 64 kernel's operand ring
        if (sp.hnb > 4) sp.hnb = 4;
        if (sp.hnb < 2)
          return fail(TS_ERR_CONFIG, "stage %d: conv window of %d bytes too large", s, sp.hbytes);
        sp.halo = 0;  // the window waits cover the halo rows
      } else if (sp.halo > 2) {
        return fail(TS_ERR_CONFIG, "stage %d: image width %d needs a 3x3 halo of %d row tiles "
                    "(at most 2; use larger tiles)", s, st.conv_w, sp.halo);
      }
    }
    if (sp.hmode) sp.grid_x = st.conv_n * sp.htpi;  // per-image re-tiling (halo conv)
    sp.splits = splits;
    sp.ws = st.workspace;
    sp.cnt = st.counters;
    if (st.order != TS_ORDER_ROW_MAJOR && st.order != TS_ORDER_STRIDED_ROW_MAJOR &&
        st.order != TS_ORDER_BANDED_COLUMN_MAJOR)
      return fail(TS_ERR_TYPE, "stage %d: unknown order %d", s, st.order);
    if (st.order == TS_ORDER_STRIDED_ROW_MAJOR &&
        (st.order_stride < 1 || sp.grid_y % st.order_stride != 0))
      return fail(TS_ERR_CONFIG, "stage %d: order stride %d does not divide grid columns %d", s,
                  st.order_stride, sp.grid_y);
    if (st.order == TS_ORDER_BANDED_COLUMN_MAJOR && st.order_stride < 1)
      return fail(TS_ERR_CONFIG, "stage %d: band %d must be >= 1", s, st.order_stride);
    sp.order = st.order;
    sp.order_stride = st.order == TS_ORDER_ROW_MAJOR ? 1 : st.order_stride;
    sp.epilogue = st.epilogue;
    sp.k_blocks = st.k / ts::kBK;
    sp.tail_tiles = 0;
    sp.tail_splits = 1;
    if (st.tail_tiles > 0) {
      // last-wave balancing; consumers of this stage (checked below) must not exist
      if (swap || conv || splits > 1 || st.epilogue == TS_EPI_SWIGLU || st.out_sem ||
          (d->flags & TS_FLAG_ROW_INTERLEAVE))
        return fail(TS_ERR_CONFIG, "stage %d: tail splitting needs an unsplit normal-layout "
                                   "GeMM stage (no SwiGLU, row gates or row interleaving)", s);
      if (st.tail_tiles > sp.grid_x * sp.grid_y || st.tail_splits < 2 ||
          sp.k_blocks % st.tail_splits)
        return fail(TS_ERR_CONFIG, "stage %d: tail of %d tiles x %d slices invalid (%d tiles, "
                                   "%d K-blocks)", s, st.tail_tiles, st.tail_splits,
                    sp.grid_x * sp.grid_y, sp.k_blocks);
      if (!st.workspace || !st.counters)
        return fail(TS_ERR_VALUE, "stage %d: tail slices need workspace and counters", s);
      sp.tail_tiles = st.tail_tiles;
      sp.tail_splits = st.tail_splits;
    }
    sp.item_begin = items;
    items += sp.grid_x * sp.grid_y * splits + sp.tail_tiles * (sp.tail_splits - 1);
    sp.item_end = items;
    sp.in_dep = -1;
    sp.n_out_deps = 0;
    sp.dot_dep = -1;
    sp.last_arriver = 0;
    if (with_tmaps) {
      // activations: box rows = 128 per CTA (normal) or tile_n (swapped);
      // weights: box rows = tile_n / cta_group (normal) or 128 (swapped)
      if (sp.hmode) {
        int rr = make_tmap_window(&sp.tmap_win, st.a, st.conv_n, st.conv_h, st.conv_w, st.lda,
                                  st.dtype, sp.hs, sp.hrows);
        if (rr) return rr;
      }
      int r = conv ? make_tmap_im2col(&sp.tmap_a, st.a, st.conv_n, st.conv_h, st.conv_w, st.k / 9,
                                      st.lda, st.dtype, 128)
                   : make_tmap(&sp.tmap_a, st.a, st.m, st.k, st.lda, st.dtype, swap ? bn : 128);
      if (r) return r;
      r = make_tmap(&sp.tmap_b, st.b, st.n, st.k, st.ldb, st.dtype, swap ? 128 : half_n / cg);
      if (r) return r;
      if (np == 2) {  // 64-row activation boxes: each CTA multicasts half of its rows
        r = make_tmap(&sp.tmap_a_half, st.a, st.m, st.k, st.lda, st.dtype, 64);
        if (r) return r;
      }
      // split-K / tail slices of a CTA-pair 256-wide stage: the owner slice streams the
      // other slices' planes in by TMA (workspace: tiles x slices x 256 rows x tile width)
      const int zmax = sp.tail_tiles > 0 ? sp.tail_splits : sp.splits;
      // (flag bit 27: measured per plan — faster for some B=1024 plans, slower than the
      // register reductions at B=256/512 — so the planner tries it as a candidate)
      if (((d->flags >> 27) & 1) && cg == 2 && bn == 256 && !swap && np == 1 && !conv &&
          zmax > 1 && st.workspace != nullptr && sp.kind == ts::kStageGemm) {
        const long long rows = static_cast<long long>(sp.grid_x) * sp.grid_y * zmax * 256;
        r = make_tmap_ws(&sp.tmap_ws, st.workspace, rows, half_n << wide);
        if (r) return r;
        sp.red_mma = 1;
      }
    }
  }
  p->total_items = items;
  if (p->balanced) {
    // static stream-K assignment (see TS_FLAG_BALANCED): GeMM stages of CTA-pair 256-wide
    // chains whose partial planes are reduced into the head segment's TMEM accumulator
    if (d->mode != TS_MODE_FUSED)
      return fail(TS_ERR_CONFIG, "the balanced schedule runs in fused mode");
    if (cg != 2 || bn != 256 || swap || np != 1)
      return fail(TS_ERR_CONFIG, "the balanced schedule needs cta_group 2, tile_n 256, one CTA "
                                 "pair per cluster");
    if (d->flags & TS_FLAG_ROW_INTERLEAVE)
      return fail(TS_ERR_CONFIG, "row interleaving is a dynamic claim order");
    for (int s = 0; s < d->n_stages; ++s) {
      const ts_stage_desc& st = d->stages[s];
      const ts::StageParams& sp = p->st[s];
      if (sp.kind != ts::kStageGemm || sp.splits != 1 || sp.tail_tiles != 0 ||
          st.epilogue == TS_EPI_SWIGLU)
        return fail(TS_ERR_CONFIG, "stage %d: the balanced schedule takes unsplit GeMM stages "
                                   "(no conv / dot / all-reduce, tail or SwiGLU)", s);
      if (!st.workspace || !st.counters)
        return fail(TS_ERR_VALUE, "stage %d: the balanced schedule needs a workspace and counters", s);
      if (sp.k_blocks >= 65536)
        return fail(TS_ERR_CONFIG, "stage %d: k too large for the balanced schedule", s);
    }
  }
  for (int i = 0; i < d->n_deps; ++i) {
    const ts_dep_desc& dd = d->deps[i];
    if (dd.producer < 0 || dd.producer >= d->n_stages || dd.consumer < 0 ||
        dd.consumer >= d->n_stages)
      return fail(TS_ERR_CONFIG, "dependency %d names an unknown stage", i);
    if (dd.producer >= dd.consumer)
      return fail(TS_ERR_CONFIG,
                  "dependency %d: producer must be invoked before consumer (cycles are not allowed)", i);
    if (dd.operand != 0)
      return fail(TS_ERR_CONFIG, "dependency %d: GeMM stages only consume operand A", i);
    const ts::StageParams& ps = p->st[dd.producer];
    ts::StageParams& cs = p->st[dd.consumer];
    if (ps.tail_tiles > 0)
      return fail(TS_ERR_CONFIG, "dependency %d: a tail-split stage cannot be waited on", i);
    const ts::Grid3 pg{ps.grid_x, ps.grid_y, ps.splits};
    int r = ts::policy_check(dd.policy, dd.param, pg);
    if (r == ts::kType) return fail(TS_ERR_TYPE, "dependency %d: unknown policy %d", i, dd.policy);
    if (r) return fail(TS_ERR_CONFIG, "dependency %d: policy parameter %d invalid for producer grid %dx%d", i, dd.param, pg.x, pg.y);
    if (cs.grid_x > ps.grid_x)
      return fail(TS_ERR_CONFIG, "dependency %d: consumer rows %d exceed producer rows %d", i,
                  cs.grid_x, ps.grid_x);
    if (cs.in_dep >= 0)
      return fail(TS_ERR_CONFIG, "dependency %d: stage %d already has an operand-A dependency", i, dd.consumer);
    if (cs.kind == ts::kStageAllReduce) {
      if (dd.policy != ts::kTile)
        return fail(TS_ERR_CONFIG, "dependency %d: the allreduce stage waits tile by tile (TileSync)", i);
      if (ps.kind != ts::kStageGemm)
        return fail(TS_ERR_CONFIG, "dependency %d: the allreduce producer must be a GeMM", i);
      if (d->mode != TS_MODE_STREAM && dd.sem == nullptr)
        return fail(TS_ERR_VALUE, "dependency %d: null semaphore array", i);
      if (d->peers->sems[d->peers->rank] != dd.sem)
        return fail(TS_ERR_VALUE, "dependency %d: peers.sems[rank] must be this dependency's semaphores", i);
      ts::DepParams& dp = p->dep[i];
      dp.sem = dd.sem;
      dp.policy = dd.policy;
      dp.param = dd.param;
      dp.pgx = pg.x;
      dp.pgy = pg.y;
      dp.pgz = pg.z;
      dp.kb_per_kstep = 1;
      dp.sem_n = ts::sem_count(dd.policy, dd.param, pg);
      dp.consumer = dd.consumer;
      dp.producer = dd.producer;
      dp.posts = pg.x * pg.y * pg.z;
      cs.in_dep = i;
      ts::StageParams& pw = p->st[dd.producer];
      pw.out_deps[pw.n_out_deps++] = i;
      continue;
    }
    if (cs.kind == ts::kStageDot && ps.wide)
      return fail(TS_ERR_CONFIG, "dependency %d: a stage feeding the dot stage must use the chain's tile width", i);
    const int cols = ps.kind == ts::kStageDot ? bn : out_tile_cols(d->stages[dd.producer], bn, cg, swap);
    int kb_per_kstep = cols / ts::kBK;
    int k_steps = 0;
    if (cs.kind == ts::kStageDot) {
      // the dot reads [Q | K | V] = the producer's whole output row; one wait, k-step 0
      if (d->stages[dd.consumer].a != d->stages[dd.producer].c ||
          ps.grid_y * cols != 3 * cs.n)
        return fail(TS_ERR_CONFIG, "dependency %d: the dot stage must read its producer's [m, 3n] output", i);
      kb_per_kstep = 1;
      k_steps = 1;
    } else if (cs.kind == ts::kStageConv) {
      // a consumer k-step = (producer column tile, filter tap): Cin = producer columns
      if (d->stages[dd.consumer].k != 9 * ps.grid_y * cols || cols % ts::kBK)
        return fail(TS_ERR_CONFIG, "dependency %d: conv consumer k=%d must be 9 x producer output columns %d", i,
                    d->stages[dd.consumer].k, ps.grid_y * cols);
      if (dd.policy == ts::kConv2D && dd.param != 9)
        return fail(TS_ERR_CONFIG, "dependency %d: a 3x3 conv consumer needs Conv2DTileSync(9), got kk=%d", i, dd.param);
      if (dd.policy == ts::kStrided)
        return fail(TS_ERR_CONFIG, "dependency %d: StridedSync cannot feed a convolution", i);
      cs.conv_subs = cols / ts::kBK;
      k_steps = cs.k_blocks / kb_per_kstep;
    } else {
      if (d->stages[dd.consumer].k != ps.grid_y * cols)
        return fail(TS_ERR_CONFIG, "dependency %d: consumer k=%d must equal producer output columns %d", i,
                    d->stages[dd.consumer].k, ps.grid_y * cols);
      k_steps = cs.k_blocks / kb_per_kstep;
    }
    if (dd.policy == ts::kConv2D && cs.kind != ts::kStageConv) {
      if (kb_per_kstep % dd.param != 0)
        return fail(TS_ERR_CONFIG, "dependency %d: kk=%d does not divide the %d K-blocks of a producer tile", i, dd.param, kb_per_kstep);
      kb_per_kstep /= dd.param;
      k_steps *= dd.param;
    }
    if (dd.policy == ts::kTile && k_steps > ps.grid_y)
      return fail(TS_ERR_CONFIG, "dependency %d: tile sync needs one producer column per consumer k-step (%d > %d)", i, k_steps, ps.grid_y);
    if (d->mode != TS_MODE_STREAM && dd.sem == nullptr)
      return fail(TS_ERR_VALUE, "dependency %d: null semaphore array", i);
    ts::DepParams& dp = p->dep[i];
    dp.sem = dd.sem;
    dp.policy = dd.policy;
    dp.param = dd.param;
    dp.pgx = pg.x;
    dp.pgy = pg.y;
    dp.pgz = pg.z;
    dp.kb_per_kstep = kb_per_kstep;
    dp.sem_n = ts::sem_count(dd.policy, dd.param, pg);
    dp.consumer = dd.consumer;
    dp.producer = dd.producer;
    dp.posts = pg.x * pg.y * pg.z;
    cs.in_dep = i;
    ts::StageParams& pw = p->st[dd.producer];
    pw.out_deps[pw.n_out_deps++] = i;
  }
  if ((d->flags & TS_FLAG_ROW_INTERLEAVE) && d->mode == TS_MODE_FUSED) {
    const ts::StageParams& s0 = p->st[0];
    const ts::StageParams& s1 = p->st[1];
    if (d->n_stages != 2 || d->n_deps != 1 || d->deps[0].producer != 0 ||
        (d->deps[0].policy != ts::kRow && d->deps[0].policy != ts::kTile) ||
        s0.kind != ts::kStageGemm || s1.kind != ts::kStageGemm ||
        s0.order != TS_ORDER_ROW_MAJOR || s1.order != TS_ORDER_ROW_MAJOR ||
        s0.grid_x != s1.grid_x)
      return fail(TS_ERR_CONFIG, "row interleaving needs a two-GeMM Row/TileSync chain with "
                                 "RowMajor orders and equal row tiles");
    p->il_b1 = s0.grid_y * s0.splits;
    p->il_b2 = s1.grid_y * s1.splits;
  }
  // Fused launches run a GeMM-fed dot stage on the last-arriving producer CTA (its
  // tiles leave the claim list); diagnostic flag bit 16 keeps them as claimed items.
  if (d->mode == TS_MODE_FUSED && !((d->flags >> 16) & 1)) {
    bool changed = false;
    for (int i = 0; i < d->n_deps; ++i) {
      ts::StageParams& ps = p->st[d->deps[i].producer];
      ts::StageParams& cs = p->st[d->deps[i].consumer];
      if (cs.kind == ts::kStageDot && ps.kind == ts::kStageGemm && cs.grid_y <= 32 &&
          ps.dot_dep < 0 && cs.in_dep == i) {
        cs.last_arriver = 1;
        ps.dot_dep = i;
        changed = true;
      }
    }
    if (changed) {
      int next = 0;
      for (int s = 0; s < p->n_stages; ++s) {
        ts::StageParams& sp = p->st[s];
        const int n = sp.last_arriver ? 0 : sp.item_end - sp.item_begin;
        sp.item_begin = next;
        next += n;
        sp.item_end = next;
      }
      p->total_items = next;
    }
  }
  return TS_OK;
}

using StreamWriteFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

StreamWriteFn stream_write_fn() {
  static StreamWriteFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<StreamWriteFn>(p);
  });
  return fn;
}

using StreamWaitFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

StreamWaitFn stream_wait_fn() {
  static StreamWaitFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<StreamWaitFn>(p);
  });
  return fn;
}

__global__ void wait_kernel(const int* flags, int n) {
  for (int i = 0; i < n; ++i) {
    while (ts::ptx::ld_acquire_gpu(flags + i) == 0) __nanosleep(100);
  }
}

// one producer's started flag (co-resident launches): flags are scattered in scratch
__global__ void wait_kernel_one(const int* flag) {
  while (ts::ptx::ld_acquire_gpu(flag) == 0) __nanosleep(100);
}

}  // namespace

extern "C" {

int ts_abi_version(void) { return TS_ABI_VERSION; }

const char* ts_last_error(void) { return ts_host::g_err.c_str(); }

int ts_sem_count(int policy, int param, int gx, int gy, int gz, int* out) {
  if (gx < 1 || gy < 1 || gz < 1) return fail(TS_ERR_VALUE, "grid dimensions must be >= 1");
  const ts::Grid3 g{gx, gy, gz};
  int r = ts::policy_check(policy, param, g);
  if (r == ts::kType) return fail(TS_ERR_TYPE, "unknown policy %d", policy);
  if (r) {
    if (policy == ts::kStrided && param < 1) return fail(TS_ERR_CONFIG, "stride must be >= 1");
    if (policy == ts::kStrided)
      return fail(TS_ERR_CONFIG, "stride %d does not divide producer columns %d", param, gy);
    return fail(TS_ERR_CONFIG, "kk must be >= 1");
  }
  *out = ts::sem_count(policy, param, g);
  return TS_OK;
}

int ts_post_target(int policy, int param, int tx, int ty, int tz, int gx, int gy, int gz,
                   int* out) {
  const ts::Grid3 g{gx, gy, gz};
  if (!g.contains(tx, ty, tz))
    return fail(TS_ERR_VALUE, "tile (%d, %d, %d) outside producer grid %dx%dx%d", tx, ty, tz, gx,
                gy, gz);
  if (policy < ts::kTile || policy > ts::kConv2D) return fail(TS_ERR_TYPE, "unknown policy %d", policy);
  if (policy == ts::kStrided && param == 0) return fail(TS_ERR_VALUE, "stride must be nonzero");
  *out = ts::post_target(policy, param, tx, ty, g);
  return TS_OK;
}

int ts_consumer_wait(int policy, int param, int tx, int ty, int tz, int k_step, int pgx, int pgy,
                     int pgz, int producer_z, int* sem, int* expected) {
  (void)tz;
  (void)pgz;
  if (policy < ts::kTile || policy > ts::kConv2D) return fail(TS_ERR_TYPE, "unknown policy %d", policy);
  if ((policy == ts::kStrided || policy == ts::kConv2D) && param == 0)
    return fail(TS_ERR_VALUE, "policy parameter must be nonzero");
  ts::Wait w = ts::consumer_wait(policy, param, tx, ty, k_step, ts::Grid3{pgx, pgy, pgz}, producer_z);
  *sem = w.sem;
  *expected = w.expected;
  return TS_OK;
}

int ts_wait_steps(int policy, int param, int k_steps, int* out, int cap, int* n) {
  if (policy < ts::kTile || policy > ts::kConv2D) return fail(TS_ERR_TYPE, "unknown policy %d", policy);
  if (policy == ts::kConv2D && param < 1) return fail(TS_ERR_VALUE, "kk must be >= 1");
  int c = 0;
  if (policy == ts::kRow || policy == ts::kStrided) {
    // Row/Strided wait exactly once, at k-step 0 (policies.py:173-175), whatever k_steps is.
    if (cap > 0) out[0] = 0;
    c = 1;
  } else {
    for (int k = 0; k < k_steps; ++k) {
      if (ts::waits_at(policy, param, k)) {
        if (c < cap) out[c] = k;
        ++c;
      }
    }
  }
  *n = c;
  return c > cap ? fail(TS_ERR_VALUE, "output capacity %d too small (%d steps)", cap, c) : TS_OK;
}

int ts_order_tile(int order, int stride, int gx, int gy, int gz, int counter, int* x, int* y,
                  int* z) {
  const ts::Grid3 g{gx, gy, gz};
  if (counter < 0 || counter >= g.total())
    return fail(TS_ERR_VALUE, "counter %d outside grid %dx%dx%d", counter, gx, gy, gz);
  if (order != ts::kRowMajor && order != ts::kStridedRowMajor && order != ts::kBandedColumnMajor)
    return fail(TS_ERR_TYPE, "unknown order %d", order);
  if (order == ts::kStridedRowMajor && (stride < 1 || gy % stride != 0))
    return fail(TS_ERR_CONFIG, "stride %d does not divide grid columns %d", stride, gy);
  if (order == ts::kBandedColumnMajor && stride < 1)
    return fail(TS_ERR_CONFIG, "band %d must be >= 1", stride);
  ts::order_tile(order, stride, g, counter, x, y, z);
  return TS_OK;
}

int ts_avoid_wait_kernel(int prod_tiles, int prod_occ, int cons_tiles, int cons_occ, int num_sms,
                         int* out) {
  *out = ts::avoid_wait_kernel(prod_tiles, prod_occ, cons_tiles, cons_occ, num_sms) ? 1 : 0;
  return TS_OK;
}

int ts_chain_grid(const ts_chain_desc* desc, int s, int* gx, int* gy) {
  static thread_local ts::ChainParams p;
  int r = build_params(desc, &p, false);
  if (r) return r;
  if (s < 0 || s >= p.n_stages) return fail(TS_ERR_VALUE, "stage %d out of range", s);
  *gx = p.st[s].grid_x;
  *gy = p.st[s].grid_y;
  return TS_OK;
}

int ts_chain_launch(const ts_chain_desc* desc, void* stream) {
  static thread_local ts::ChainParams p;
  if (desc != nullptr && desc->mode == TS_MODE_CORESIDENT)
    return fail(TS_ERR_CONFIG, "co-resident chains launch through ts_chain_launch_coresident");
  int r = build_params(desc, &p, true);
  if (r) return r;
  if (desc->scratch == nullptr) return fail(TS_ERR_VALUE, "null scratch buffer");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int bn = tile_n_of(desc);
  const int cg = cta_group_of(desc);
  const int dtype = desc->stages[0].dtype;
  int ctas = desc->num_ctas > 0 ? desc->num_ctas : sm_count();
  if (ctas <= 0) return fail(TS_ERR_CUDA, "could not query the SM count");
  const int np = cluster_pairs_of(desc);
  ctas /= cg * np;  // items in flight: CTAs (cg = 1), CTA pairs (cg = 2) or 2-pair clusters
  if (ctas < 1) return fail(TS_ERR_VALUE, "num_ctas too small for cta_group %d x %d", cg, np);
  if (desc->mode == TS_MODE_FUSED) {
    p.item_lo = 0;
    p.item_hi = p.total_items;
    // balanced: every unit runs (the kernel derives the stream-K widths from its grid)
    int grid = p.balanced || ctas < p.total_items ? ctas : p.total_items;
    return launch_dispatch(bn, cg, desc->swap_ab, dtype, p, grid, s, np);
  }
  // Stream mode: the same kernel, one launch per stage, no semaphores — the
  // stream-synchronized baseline (reference Mode.STREAM engine.py:40-42).
  // An all-reduce stage keeps its dependency: its tiles still wait for the producer
  // tiles of every rank (peer ranks run their own launches).
  ts::ChainParams q = p;
  for (int i = 0; i < q.n_stages; ++i) {
    const bool ar = q.st[i].kind == ts::kStageAllReduce;
    if (!ar) q.st[i].in_dep = -1;
    q.st[i].n_out_deps = 0;
    q.st[i].dot_dep = -1;
    for (int j = 0; j < p.st[i].n_out_deps; ++j) {
      const int dd = p.st[i].out_deps[j];
      if (p.st[p.dep[dd].consumer].kind == ts::kStageAllReduce)
        q.st[i].out_deps[q.st[i].n_out_deps++] = dd;
    }
  }
  bool any_ar = false;
  for (int i = 0; i < q.n_stages; ++i) any_ar = any_ar || q.st[i].kind == ts::kStageAllReduce;
  if (!any_ar) q.n_deps = 0;
  for (int i = 0; i < q.n_stages; ++i) {
    q.item_lo = q.st[i].item_begin;
    q.item_hi = q.st[i].item_end;
    const int n = q.item_hi - q.item_lo;
    if (n <= 0) continue;  // e.g. a rank that owns no all-reduce tile
    r = launch_dispatch(bn, cg, desc->swap_ab, dtype, q, ctas < n ? ctas : n, s, np);
    if (r) return r;
  }
  return TS_OK;
}

int ts_wait_kernel_launch(const int* flags, int n, void* stream) {
  if (flags == nullptr || n < 1) return fail(TS_ERR_VALUE, "wait kernel needs >= 1 flag");
  wait_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(flags, n);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? TS_OK : cuda_fail(e, "wait_kernel launch");
}

int ts_chain_launch_coresident(const ts_chain_desc* desc, void* const* streams, int n_streams,
                               int wait_kernel, int launch_order, const int* grid) {
  static thread_local ts::ChainParams p;
  if (desc == nullptr || streams == nullptr) return fail(TS_ERR_VALUE, "null descriptor or streams");
  if (desc->mode != TS_MODE_CORESIDENT)
    return fail(TS_ERR_CONFIG, "ts_chain_launch_coresident needs mode TS_MODE_CORESIDENT");
  if (wait_kernel < 0 || wait_kernel > 2) return fail(TS_ERR_VALUE, "wait_kernel must be 0, 1 or 2");
  int r = build_params(desc, &p, true);
  if (r) return r;
  if (desc->scratch == nullptr) return fail(TS_ERR_VALUE, "null scratch buffer");
  if (n_streams != p.n_stages)
    return fail(TS_ERR_VALUE, "%d streams for %d stages", n_streams, p.n_stages);
  if (desc->flags & TS_FLAG_ROW_INTERLEAVE)
    return fail(TS_ERR_CONFIG, "row interleaving is a fused-mode claim order");
  for (int s = 0; s < p.n_stages; ++s) {
    if (p.st[s].kind == ts::kStageAllReduce)
      return fail(TS_ERR_CONFIG, "the all-reduce stage runs in fused or stream mode only");
    if (streams[s] == nullptr) return fail(TS_ERR_VALUE, "null stream for stage %d", s);
  }
  const int bn = tile_n_of(desc);
  const int cg = cta_group_of(desc);
  const int np = cluster_pairs_of(desc);
  const int dtype = desc->stages[0].dtype;
  int sms = sm_count();
  if (sms <= 0) return fail(TS_ERR_CUDA, "could not query the SM count");
  const int units = sms / (cg * np);  // one CTA (pair, cluster) per SM: occupancy 1
  int g[TS_MAX_STAGES];
  for (int s = 0; s < p.n_stages; ++s) {
    const int tiles = p.st[s].item_end - p.st[s].item_begin;
    g[s] = grid != nullptr && grid[s] > 0 ? (grid[s] < tiles ? grid[s] : tiles) : tiles;
  }
  for (int i = 0; i < p.n_stages; ++i) {
    const int s = launch_order ? p.n_stages - 1 - i : i;
    cudaStream_t st = static_cast<cudaStream_t>(streams[s]);
    // the reference's gate (engine.gated_producers): hold this stage back until every
    // producer it depends on has started, unless "auto" finds both grids fit one wave
    int flags_at[TS_MAX_DEPS], nf = 0;
    for (int d = 0; d < p.n_deps && wait_kernel != 0; ++d) {
      if (p.dep[d].consumer != s) continue;
      const int pr = p.dep[d].producer;
      if (wait_kernel == 2 && ts::avoid_wait_kernel(g[pr], 1, g[s], 1, units)) continue;
      flags_at[nf++] = ts::kCtlBase + ts::kCtlInts * pr + 2;
    }
    for (int f = 0; f < nf; ++f) {
      wait_kernel_one<<<1, 1, 0, st>>>(desc->scratch + flags_at[f]);
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return cuda_fail(e, "wait_kernel launch");
    }
    ts::ChainParams q = p;
    q.item_lo = q.st[s].item_begin;
    q.item_hi = q.st[s].item_end;
    q.ctl = desc->scratch + ts::kCtlBase + ts::kCtlInts * s;
    q.coresident = 1;
    r = launch_dispatch(bn, cg, desc->swap_ab, dtype, q, g[s], st, np);
    if (r) return r;
  }
  return TS_OK;
}

int ts_stream_signal(int* sem, int value, void* stream) {
  if (sem == nullptr) return fail(TS_ERR_VALUE, "null semaphore");
  StreamWriteFn fn = stream_write_fn();
  if (!fn) return fail(TS_ERR_CUDA, "cuStreamWriteValue32 unavailable");
  // default flags: the write is ordered after (and makes visible) the stream's prior work
  CUresult r = fn(static_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(sem),
                  static_cast<cuuint32_t>(value), CU_STREAM_WRITE_VALUE_DEFAULT);
  return r == CUDA_SUCCESS ? TS_OK : fail(TS_ERR_CUDA, "cuStreamWriteValue32 failed (%d)", (int)r);
}

int ts_stream_wait(const int* sem, int value, void* stream) {
  if (sem == nullptr) return fail(TS_ERR_VALUE, "null semaphore");
  StreamWaitFn fn = stream_wait_fn();
  if (!fn) return fail(TS_ERR_CUDA, "cuStreamWaitValue32 unavailable");
  CUresult r = fn(static_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(sem),
                  static_cast<cuuint32_t>(value), CU_STREAM_WAIT_VALUE_GEQ);
  return r == CUDA_SUCCESS ? TS_OK : fail(TS_ERR_CUDA, "cuStreamWaitValue32 failed (%d)", (int)r);
}

int ts_chain_units(int tile_n, int cta_group, int cluster_pairs, int swap_ab, int dtype,
                   int* out) {
  int sms = sm_count();
  if (sms <= 0) return fail(TS_ERR_CUDA, "could not query the SM count");
  const int cg = swap_ab ? 1 : (cta_group == 0 ? 2 : cta_group);
  const int np = cluster_pairs == 0 ? 1 : cluster_pairs;
  const int bn = tile_n == 0 ? 256 : tile_n;
  int mc = 0, r = TS_OK;
  const bool bf = dtype == TS_DTYPE_BF16;
  if (np == 2) {
    if (cg != 2 || bn != 256 || swap_ab)
      return fail(TS_ERR_CONFIG, "two-pair clusters need cta_group 2 and tile_n 256");
    r = bf ? prepare<256, 2, __nv_bfloat16, false, true>(&mc) : prepare<256, 2, __half, false, true>(&mc);
  } else if (cg == 2) {
    if (bn == 128) r = bf ? prepare<128, 2, __nv_bfloat16, false, false>(&mc) : prepare<128, 2, __half, false, false>(&mc);
    else if (bn == 256) r = bf ? prepare<256, 2, __nv_bfloat16, false, false>(&mc) : prepare<256, 2, __half, false, false>(&mc);
    else return fail(TS_ERR_VALUE, "cta_group 2 needs tile_n 128 or 256 (got %d)", bn);
  } else if (np != 1) {
    return fail(TS_ERR_VALUE, "cluster_pairs must be 0, 1 or 2 (got %d)", cluster_pairs);
  }
  if (r) return r;
  int units = sms / (cg * np);
  if (mc > 0 && mc < units) units = mc;
  *out = units;
  return TS_OK;
}

int ts_device_sm_count(int* out) {
  int n = sm_count();
  if (n <= 0) return fail(TS_ERR_CUDA, "no CUDA device");
  *out = n;
  return TS_OK;
}

}  // extern "C"
