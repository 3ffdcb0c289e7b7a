// Per-level ranks of a hodlr_desc (SPEC.md:147-160 ragged panels, padded per
// level): column offsets of the level panels in the U / Y / V slabs and the
// offsets of the per-level K blocks, pivots and solve aids.  desc->ranks ==
// NULL is the uniform layout (rank r at every level).
#pragma once
#include "common.cuh"

namespace hodlr {

struct LevelRanks {
  int L = 0;
  bool uniform = true;
  int rmax = 0;
  int r[32] = {};         // r[l'] = rank of level l' (1..L)
  int64_t c[33] = {};     // c[l'] = first column of level l' (1..L+1; c[L+1] = total columns)
  int64_t koff[32] = {};  // K LU of parent level lv (0..L-1): (2 r[lv+1])^2 per parent
  int64_t kpoff[32] = {}; // kswaps / kperm: 2 r[lv+1] per parent
  int64_t kioff[32] = {}; // Kinv: inv_block_elems(2 r[lv+1]) per parent
  int64_t cols() const { return c[L + 1]; }
  int rank_below(int lv) const { return r[lv + 1]; }  // children of parent level lv
};

// false if desc->ranks is inconsistent (negative ranks, max != desc->r)
inline bool make_ranks(const hodlr_desc* d, LevelRanks& q) {
  q = LevelRanks{};
  if (!d || d->L < 0 || d->L > 30) return false;
  q.L = d->L;
  q.uniform = d->ranks == nullptr;
  int mx = 0;
  for (int l = 1; l <= d->L; ++l) {
    const int rl = q.uniform ? d->r : d->ranks[l - 1];
    if (rl < 0) return false;
    q.r[l] = rl;
    mx = rl > mx ? rl : mx;
  }
  q.rmax = d->L ? mx : d->r;
  if (!q.uniform && mx != d->r) return false;
  q.c[1] = 0;
  for (int l = 1; l <= d->L; ++l) q.c[l + 1] = q.c[l] + q.r[l];
  int64_t ko = 0, kp = 0, ki = 0;
  for (int lv = 0; lv < d->L; ++lv) {
    const int s = 2 * q.r[lv + 1];
    q.koff[lv] = ko;
    q.kpoff[lv] = kp;
    q.kioff[lv] = ki;
    ko += ((int64_t)1 << lv) * s * s;
    kp += ((int64_t)1 << lv) * s;
    ki += ((int64_t)1 << lv) * inv_block_elems(s);
  }
  return true;
}

}  // namespace hodlr
