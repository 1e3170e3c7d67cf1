// ts_policy.cuh — the synchronization-policy arithmetic shared by host and device.
//
// One copy of each rule, compiled for both sides: the kernels call these in the TMA
// producer warp (waits) and the epilogue (posts); the C ABI exports the same functions
// so the Python drop-in returns exactly what the device does.
//
// Semantics follow the reference policy layer, /root/reference/pkg/src/tilesync_sim/
// policies.py, with the paper's ambiguities resolved as SPEC.md:105-191 does:
//   * split-k: every z-slice posts +1 to one semaphore, expected values scale by z;
//   * StridedSync: rows*stride semaphores, index row*stride + col%stride;
//   * RowSync "col == 0" means "only at k-step 0".
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define TS_HD __host__ __device__ __forceinline__
#else
#define TS_HD inline
#endif

namespace ts {

enum PolicyKind : int { kTile = 0, kRow = 1, kStrided = 2, kConv2D = 3 };
enum OrderKind : int { kRowMajor = 0, kStridedRowMajor = 1, kBandedColumnMajor = 2 };
enum Status : int { kOk = 0, kConfig = 1, kValue = 2, kType = 3 };

struct Grid3 {
  int x, y, z;
  TS_HD int total() const { return x * y * z; }
  TS_HD bool contains(int tx, int ty, int tz) const {
    return tx >= 0 && tx < x && ty >= 0 && ty < y && tz >= 0 && tz < z;
  }
};

// A (semaphore, threshold) pair; sem < 0 means "no wait at this k-step".
struct Wait {
  int sem;
  int expected;
};

// check_policy — policies.py:102-112.
TS_HD int policy_check(int kind, int param, Grid3 prod) {
  if (kind == kStrided) {
    if (param < 1) return kConfig;
    if (prod.y % param != 0) return kConfig;
    return kOk;
  }
  if (kind == kConv2D) return param < 1 ? kConfig : kOk;
  if (kind == kTile || kind == kRow) return kOk;
  return kType;
}

// sem_count — policies.py:115-125.  Tile/Conv: one per producer tile (z shares);
// Row: one per producer row; Strided: `stride` per producer row.
TS_HD int sem_count(int kind, int param, Grid3 prod) {
  switch (kind) {
    case kTile:
    case kConv2D: return prod.x * prod.y;
    case kRow: return prod.x;
    case kStrided: return prod.x * param;
  }
  return -1;
}

// post_target — policies.py:128-142.  Where a finished producer tile (any z) adds 1.
TS_HD int post_target(int kind, int param, int tx, int ty, Grid3 prod) {
  switch (kind) {
    case kTile:
    case kConv2D: return tx * prod.y + ty;
    case kRow: return tx;
    case kStrided: return tx * param + ty % param;
  }
  return -1;
}

// consumer_wait — policies.py:145-166.  Which semaphore a consumer tile observes before
// reference k-step `k`, and the post count that makes the needed producer tiles whole.
TS_HD Wait consumer_wait(int kind, int param, int row, int col, int k, Grid3 prod,
                         int prod_z) {
  Wait w{-1, 0};
  switch (kind) {
    case kTile:
      w.sem = row * prod.y + k;
      w.expected = prod_z;
      break;
    case kRow:
      if (k == 0) {
        w.sem = row;
        w.expected = prod.y * prod_z;
      }
      break;
    case kStrided:
      if (k == 0) {
        w.sem = row * param + col % param;
        w.expected = (prod.y / param) * prod_z;
      }
      break;
    case kConv2D:
      if (k % param == 0) {
        w.sem = row * prod.y + k / param;
        w.expected = prod_z;
      }
      break;
  }
  return w;
}

// isSync: does `kind` wait at reference k-step `k`?  (wait_steps, policies.py:169-178)
TS_HD bool waits_at(int kind, int param, int k) {
  switch (kind) {
    case kTile: return true;
    case kRow:
    case kStrided: return k == 0;
    case kConv2D: return k % param == 0;
  }
  return false;
}

// order_tile — policies.py:181-205.  The tile of a stage's n-th counter draw.
// Lexicographic (x, y, z) with z fastest; StridedRowMajor regroups the column axis so
// that columns `stride` apart are drawn consecutively (group g = {g, g+s, g+2s, ...}).
//
// Extension (not in the reference simulator; the paper notes CuSync supports further
// orders): BandedColumnMajor(band) walks bands of `band` tile rows in
// order and, inside a band, goes column by column. Row-band tiles that read the same
// weight column block are then in flight together, so the block streams from HBM once
// per band instead of once per row; band = 1 is RowMajor.
TS_HD void order_tile(int kind, int stride, Grid3 g, int n, int* x, int* y, int* z) {
  int zz = n % g.z;
  int rest = n / g.z;
  *z = zz;
  if (kind == kBandedColumnMajor) {
    const int per_band = stride * g.y;
    const int b = rest / per_band;
    const int off = rest % per_band;
    const int rows = (g.x - b * stride) < stride ? (g.x - b * stride) : stride;
    *x = b * stride + off % rows;
    *y = off / rows;
    return;
  }
  int pos = rest % g.y;  // position along the (possibly regrouped) column walk
  *x = rest / g.y;
  if (kind == kStridedRowMajor) {
    int per_group = g.y / stride;
    *y = pos / per_group + (pos % per_group) * stride;
  } else {
    *y = pos;
  }
}

// avoid_wait_kernel — engine.py:173-180, SPEC.md:295 ("+W"): the wait kernel is not
// needed when both grids fit one combined wave at the smaller occupancy.
TS_HD bool avoid_wait_kernel(int prod_tiles, int prod_occ, int cons_tiles, int cons_occ,
                             int num_sms) {
  int occ = prod_occ < cons_occ ? prod_occ : cons_occ;
  return prod_tiles + cons_tiles <= occ * num_sms;
}

}  // namespace ts
