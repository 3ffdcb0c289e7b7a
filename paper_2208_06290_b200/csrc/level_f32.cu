// FP32 level steps for rank 8 (the preconditioner configuration, cfg4):
//
//   C(I_c, :) -= Y_c^{l+1} W'_c            (update; skipped when W == null)
//   TW_q      += V_q^{(l)T} C(I_q, :)      (next level's [W|T] / w; skipped when V == null)
//
// The factorization runs level_f32_dmma_kernel (below): the fp64 DMMA chain
// on widened fp32 operands.  The solve runs the SIMT level_f32_kernel, whose
// per-column arithmetic does not depend on the number of right-hand sides.
// At rank 8 the step is HBM-bound (2 flops per byte).  SIMT kernel: one warp owns 8 columns of a row segment, each
// lane streams rows (coalesced column reads), keeps the 8 x 8 W' block of the
// current child and the 8 x 8 [W|T] partial in registers, and the warp's
// partials are combined with a fixed xor-butterfly.  Segment partials are
// summed in segment order.  The column split and the reduction order do not
// depend on the number of columns, so a column of a multi-RHS solve is
// bit-identical to the single-column solve.
#include "common.cuh"

namespace hodlr {

constexpr int F32_R = 8;
constexpr int F32_SEG = 1024;  // max rows per segment (the caller's seg_max, fixed per phase)

struct LevelF32Args {
  float* C;
  int64_t ldc;
  const float* A1;  // Y^{l+1} panel, ld lda
  const float* V;   // V^{(l)} panel (null: no reduction)
  int64_t lda;
  const float* W;   // paired W per parent (2R x ncols, ld 2R) at W + p * wstride (null: no update)
  int64_t wstride;
  int64_t n_c;
  int64_t node_rows;
  int ncols;
  int seg_rows;
  int chunks;       // ceil(ncols / 8) CTAs (one warp each) per segment (1 when ncols <= 4)
  float* TW;        // final: paired layout; partial: [seg][R x ncols] ld R
  int64_t tw_stride;
  int partial;
};

// one warp per CTA: work item = (segment, NCW-column chunk).  The W' blocks of
// all children in the segment are staged in shared memory up front; each lane
// then streams two rows per iteration (all loads issued before use).  NCW = 8
// for wide panels; 1 / 2 / 4 for few right-hand sides (same per-column
// operation sequence, so a column's result does not depend on NCW).
constexpr int F32_MAXCH = F32_SEG / 32;  // children per segment (n_c >= 32)

template <int NCW>
__global__ void __launch_bounds__(32, NCW == 8 ? 12 : (NCW == 4 ? 16 : 24)) level_f32_kernel(LevelF32Args g) {
  constexpr int R = F32_R;
  const int lane = threadIdx.x;
  const int seg = blockIdx.x / g.chunks, chunk = blockIdx.x % g.chunks;
  const int col0 = chunk * NCW;
  const int ncw = min(NCW, g.ncols - col0);  // columns of this warp (ragged last chunk)
  const int64_t seg0 = (int64_t)seg * g.seg_rows;
  const float* __restrict__ A1 = g.A1;
  const float* __restrict__ V = g.V;
  float* __restrict__ C = g.C;
  __shared__ __align__(16) float ws[F32_MAXCH][R][NCW];  // W' of the segment's children (broadcast reads)
  const int64_t ch0 = seg0 / g.n_c;
  const int nch = (int)ceil_div(g.seg_rows, g.n_c);
  if (g.W) {
    for (int e = lane; e < nch * R * NCW; e += 32) {
      const int cc = e / (R * NCW), k = e % R, j = (e / R) % NCW;
      const int64_t ch = ch0 + cc;
      const float* wp = g.W + (ch >> 1) * g.wstride + (ch & 1) * R;
      ws[cc][k][j] = (j < ncw) ? __ldg(wp + k + (int64_t)(col0 + j) * (2 * R)) : 0.f;
    }
    __syncwarp();
  }
  float tw[R][NCW];
#pragma unroll
  for (int k = 0; k < R; ++k)
#pragma unroll
    for (int j = 0; j < NCW; ++j) tw[k][j] = 0.f;
  const int ncr = (int)g.n_c;
#pragma unroll 1
  for (int i0 = 0; i0 < g.seg_rows; i0 += 64) {
    // lane owns rows i0 + 2 lane + {0, 1}: 8-byte loads of C, Y^{l+1} and V
    const int64_t row = seg0 + i0 + 2 * lane;
    float c[2][NCW], a[2][R], v[2][R];
#pragma unroll
    for (int j = 0; j < NCW; ++j) {
      const float2 t = (j < ncw) ? *reinterpret_cast<const float2*>(C + row + (int64_t)(col0 + j) * g.ldc)
                                 : make_float2(0.f, 0.f);
      c[0][j] = t.x, c[1][j] = t.y;
    }
    if (g.W) {
#pragma unroll
      for (int k = 0; k < R; ++k) {
        const float2 t = __ldg(reinterpret_cast<const float2*>(A1 + row + (int64_t)k * g.lda));
        a[0][k] = t.x, a[1][k] = t.y;
      }
    }
    if (V) {
#pragma unroll
      for (int k = 0; k < R; ++k) {
        const float2 t = __ldg(reinterpret_cast<const float2*>(V + row + (int64_t)k * g.lda));
        v[0][k] = t.x, v[1][k] = t.y;
      }
    }
    if (g.W) {
      const int cc = (i0 + 2 * lane) / ncr;  // child within the segment (rows 2 lane + {0,1} share it)
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        float t[NCW];
#pragma unroll
        for (int j = 0; j < NCW; ++j) t[j] = 0.f;
#pragma unroll
        for (int k = 0; k < R; ++k) {  // W' row k as two broadcast 16-byte loads
          float wk[NCW];
          if constexpr (NCW >= 4) {
#pragma unroll
            for (int j4 = 0; j4 < NCW; j4 += 4) {
              const float4 w4 = *reinterpret_cast<const float4*>(&ws[cc][k][j4]);
              wk[j4] = w4.x, wk[j4 + 1] = w4.y, wk[j4 + 2] = w4.z, wk[j4 + 3] = w4.w;
            }
          } else {
#pragma unroll
            for (int j = 0; j < NCW; ++j) wk[j] = ws[cc][k][j];
          }
#pragma unroll
          for (int j = 0; j < NCW; ++j) t[j] = fmaf(a[u][k], wk[j], t[j]);
        }
#pragma unroll
        for (int j = 0; j < NCW; ++j) c[u][j] = __fsub_rn(c[u][j], t[j]);
      }
#pragma unroll
      for (int j = 0; j < NCW; ++j)
        if (j < ncw) *reinterpret_cast<float2*>(C + row + (int64_t)(col0 + j) * g.ldc) = make_float2(c[0][j], c[1][j]);
    }
    if (V) {
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int k = 0; k < R; ++k)
#pragma unroll
          for (int j = 0; j < NCW; ++j) tw[k][j] = fmaf(v[u][k], c[u][j], tw[k][j]);
    }
  }
  if (!g.V) return;
#pragma unroll
  for (int k = 0; k < R; ++k)
#pragma unroll
    for (int j = 0; j < NCW; ++j) {
      float v = tw[k][j];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      tw[k][j] = v;
    }
  if (lane == 0) {
    if (g.partial) {
      float* out = g.TW + (int64_t)seg * R * g.ncols;
      for (int j = 0; j < ncw; ++j)
#pragma unroll
        for (int k = 0; k < R; ++k) out[k + (int64_t)(col0 + j) * R] = tw[k][j];
    } else {
      const int64_t q = seg0 / g.node_rows;
      float* out = g.TW + (q >> 1) * g.tw_stride + (q & 1) * R;
      for (int j = 0; j < ncw; ++j)
#pragma unroll
        for (int k = 0; k < R; ++k) out[k + (int64_t)(col0 + j) * 2 * R] = tw[k][j];
    }
  }
}

// TW_q = sum of the q's segment partials: warp per entry, lane l sums segments
// l, l + 32, ... in order, then a fixed xor butterfly (order depends only on the
// segment count, never on ncols); paired output
__global__ void level_reduce_f32_kernel(const float* part, float* TW, int ncols, int segs, int nnodes,
                                        int64_t tw_stride) {
  constexpr int R = F32_R;
  const int64_t per = (int64_t)R * ncols;
  const int64_t total = per * nnodes;
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; e < total; e += warps) {
    const int64_t q = e / per, mn = e % per;
    const int m = (int)(mn % R), n = (int)(mn / R);
    float s = 0.f;
    for (int k = lane; k < segs; k += 32) s += part[(q * segs + k) * per + mn];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) TW[(q >> 1) * tw_stride + (q & 1) * R + m + (int64_t)n * 2 * R] = s;
  }
}

// ---------------------------------------------------------------------------
// Factorization step on the fp64 DMMA chain (the same transposed scheme as
// level_update4_kernel, here at R = 8 with fp32 operands widened on load and
// results rounded on store):
//   C^T  = C^T + (-W'^T) A1^T      A: W' entries, B: A1 panel (LDS.128 pairs)
//   TW^T += C^T V                  A: the updated (rounded) C^T accumulators
// CTA = 8 warps over a row segment, panels of a 64-row chunk widened into
// shared memory (register prefetch of the next chunk, one barrier per chunk),
// warps stream their 8-column groups.  The fp32 solve keeps the SIMT kernel
// (its per-column arithmetic must not depend on nrhs).
// ---------------------------------------------------------------------------
constexpr int F32D_CH = 64, F32D_P = 66;

template <int GPW>
__global__ void __launch_bounds__(256, 3) level_f32_dmma_kernel(LevelF32Args g, int ncg, int tpc) {
  constexpr int R = F32_R, CH = F32D_CH, NI = CH / 16, P = F32D_P, PANEL = R * P;
  __shared__ __align__(16) double sm[2][2 * PANEL];  // [stage][A1 panel | V panel], [rank][row]
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int ar = lane >> 2, ac = lane & 3;
  const int seg = blockIdx.x / ncg, cg = blockIdx.x % ncg;
  const int64_t seg0 = (int64_t)seg * g.seg_rows;
  const int nch = g.seg_rows / CH;
  const int G = g.ncols >> 3;
  const int gb = cg * tpc, ge = min(G, gb + tpc);
  const bool upd = g.W != nullptr, red = g.V != nullptr;
  // staging share: rank sk, rows 2 (t % 32) + {0, 1}
  const int sk = t >> 5, sr = (t & 31) * 2;
  float2 pa = make_float2(0.f, 0.f), pv = make_float2(0.f, 0.f);
  auto fetch = [&](int ch) {
    const int64_t r0 = seg0 + (int64_t)ch * CH + sr + (int64_t)sk * g.lda;
    if (upd) pa = *reinterpret_cast<const float2*>(g.A1 + r0);
    if (red) pv = *reinterpret_cast<const float2*>(g.V + r0);
  };
  auto put = [&](int s) {
    *reinterpret_cast<double2*>(sm[s] + sk * P + sr) = make_double2(pa.x, pa.y);
    *reinterpret_cast<double2*>(sm[s] + PANEL + sk * P + sr) = make_double2(pv.x, pv.y);
  };
  double tw[GPW][2];
#pragma unroll
  for (int q = 0; q < GPW; ++q) tw[q][0] = tw[q][1] = 0.0;
  if (nch > 0) {
    fetch(0);
    put(0);
  }
  __syncthreads();
  for (int ch = 0; ch < nch; ++ch) {
    const int s = ch & 1;
    if (ch + 1 < nch) fetch(ch + 1);  // lands while this chunk is computed
    const double* As = sm[s];
    const double* Vs = sm[s] + PANEL;
    const int64_t row0 = seg0 + (int64_t)ch * CH;
    const int c = (int)(row0 / g.n_c);
    const float* Wp = upd ? g.W + (int64_t)(c >> 1) * g.wstride + (c & 1) * R : nullptr;
#pragma unroll
    for (int q = 0; q < GPW; ++q) {
      const int grp = gb + warp + 8 * q;
      if (grp < ge) {
        const int col = grp * 8 + ar;
        float* cptr = g.C + row0 + (int64_t)col * g.ldc + 4 * ac;
        float4 cin[NI];
#pragma unroll
        for (int i = 0; i < NI; ++i) cin[i] = *reinterpret_cast<const float4*>(cptr + 16 * i);
        double acc[2 * NI][2];
#pragma unroll
        for (int i = 0; i < 2 * NI; ++i) acc[i][0] = acc[i][1] = 0.0;
        if (upd) {
          const float2 w2 = __ldg(reinterpret_cast<const float2*>(Wp + (int64_t)col * (2 * R) + 2 * ac));
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const double a = -(double)(u ? w2.y : w2.x);
            const double* ak = As + (2 * ac + u) * P + 2 * ar;
#pragma unroll
            for (int i = 0; i < NI; ++i) {
              const double2 b2 = *reinterpret_cast<const double2*>(ak + 16 * i);
              dmma_8x8x4(acc[2 * i][0], acc[2 * i][1], a, b2.x);
              dmma_8x8x4(acc[2 * i + 1][0], acc[2 * i + 1][1], a, b2.y);
            }
          }
        }
        // C + (-(A1 W')), rounded to fp32; the rounded values feed the reduction
#pragma unroll
        for (int i = 0; i < NI; ++i) {
          const float x = (float)((double)cin[i].x + acc[2 * i][0]);
          const float y = (float)((double)cin[i].y + acc[2 * i + 1][0]);
          const float z = (float)((double)cin[i].z + acc[2 * i][1]);
          const float w = (float)((double)cin[i].w + acc[2 * i + 1][1]);
          if (upd) *reinterpret_cast<float4*>(cptr + 16 * i) = make_float4(x, y, z, w);
          acc[2 * i][0] = x, acc[2 * i + 1][0] = y, acc[2 * i][1] = z, acc[2 * i + 1][1] = w;
        }
        if (red) {
#pragma unroll
          for (int i = 0; i < NI; ++i)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const double2 v2 = *reinterpret_cast<const double2*>(Vs + ar * P + 16 * i + 4 * ac + 2 * h);
              dmma_8x8x4(tw[q][0], tw[q][1], acc[2 * i][h], v2.x);
              dmma_8x8x4(tw[q][0], tw[q][1], acc[2 * i + 1][h], v2.y);
            }
        }
      }
    }
    if (ch + 1 < nch) put(s ^ 1);  // stage s ^ 1 was last read before the previous barrier
    // a segment may hold several whole nodes: emit a node's [W|T] at its last chunk
    if (red && !g.partial && (row0 + CH) % g.node_rows == 0) {
      const int64_t qn = row0 / g.node_rows;
      float* out = g.TW + (qn >> 1) * g.tw_stride + (qn & 1) * R;
#pragma unroll
      for (int q = 0; q < GPW; ++q) {
        const int grp = gb + warp + 8 * q;
        if (grp < ge)
          *reinterpret_cast<float2*>(out + 2 * ac + (int64_t)(grp * 8 + ar) * (2 * R)) =
              make_float2((float)tw[q][0], (float)tw[q][1]);
        tw[q][0] = tw[q][1] = 0.0;
      }
    }
    __syncthreads();
  }
  if (!red || !g.partial) return;
  // tw[q][h] = TW^T[col][rank 2 ac + h], segment partial
  float* out = g.TW + (int64_t)seg * R * g.ncols;
#pragma unroll
  for (int q = 0; q < GPW; ++q) {
    const int grp = gb + warp + 8 * q;
    if (grp < ge)
      *reinterpret_cast<float2*>(out + 2 * ac + (int64_t)(grp * 8 + ar) * R) =
          make_float2((float)tw[q][0], (float)tw[q][1]);
  }
}

// One factorization level step (r = 8) on the DMMA chain.  ERR_ARG: shape or
// alignment not supported (the caller uses level_f32).
hodlr_status level_f32_dmma(int r, int64_t n, int64_t n_c, int64_t node_rows, float* C, int64_t ldc, const float* A1,
                            const float* V, int64_t lda, const float* W, int64_t wstride, int ncols, float* TW,
                            int64_t tw_stride, float* part, size_t part_bytes, cudaStream_t st) {
  if (ncols == 0) return HODLR_OK;
  if (r != F32_R || ncols % 8 || n_c % F32D_CH || n % F32D_CH || node_rows % F32D_CH) return HODLR_ERR_ARG;
  if ((ldc & 3) || (uintptr_t)C % 16 || (lda & 1) || (A1 && (uintptr_t)A1 % 8) || (V && (uintptr_t)V % 8) ||
      (W && ((wstride & 1) || (uintptr_t)W % 8)) || (TW && (tw_stride & 1)))
    return HODLR_ERR_ARG;
  // segments of up to F32_SEG rows: several whole nodes, or a node's slice (partials)
  const int64_t seg = std::min<int64_t>(n, F32_SEG);
  if (n % seg || (node_rows % seg && seg % node_rows)) return HODLR_ERR_ARG;
  const int64_t nseg = n / seg;
  const bool split = seg < node_rows && V != nullptr;
  if (split && (size_t)nseg * F32_R * ncols * sizeof(float) > part_bytes) return HODLR_ERR_ARG;
  LevelF32Args g{C, ldc, A1, V, lda, W, wstride, n_c, node_rows, ncols, (int)seg, 0, split ? part : TW, tw_stride,
                 split ? 1 : 0};
  const int G = ncols / 8;
  const int gpw = G <= 8 ? 1 : 2;
  const int tpc = std::min(G, 8 * gpw);
  const int ncg = (G + tpc - 1) / tpc;
  const int64_t grid = nseg * ncg;
  if (grid > 2147483647LL) return HODLR_ERR_ARG;
  if (gpw == 1)
    level_f32_dmma_kernel<1><<<(unsigned)grid, 256, 0, st>>>(g, ncg, tpc);
  else
    level_f32_dmma_kernel<2><<<(unsigned)grid, 256, 0, st>>>(g, ncg, tpc);
  HODLR_CHECK_LAUNCH();
  if (!split) return HODLR_OK;
  const int nnodes = (int)(n / node_rows);
  const int64_t total = (int64_t)F32_R * ncols * nnodes;
  level_reduce_f32_kernel<<<(unsigned)std::min<int64_t>(ceil_div(total, 8), 4736), 256, 0, st>>>(
      part, TW, ncols, (int)(node_rows / seg), nnodes, tw_stride);
  HODLR_CHECK_LAUNCH();
  return HODLR_OK;
}

size_t level_f32_partial_bytes(int64_t n, int ncols) { return (size_t)(n / 64 + 1) * F32_R * ncols * sizeof(float); }

// One fp32 level step over n rows (r = 8, n_c >= 32).  ERR_ARG: unsupported shape.
hodlr_status level_f32(int r, int64_t n, int64_t n_c, int64_t node_rows, float* C, int64_t ldc, const float* A1,
                       const float* V, int64_t lda, const float* W, int64_t wstride, int ncols, float* TW,
                       int64_t tw_stride, float* part, size_t part_bytes, cudaStream_t st, int seg_max) {
  if (ncols == 0) return HODLR_OK;
  if (r != F32_R || n_c < 32 || n_c % 32 || n % 64 || node_rows % 64) return HODLR_ERR_ARG;
  const int64_t seg = std::min<int64_t>(node_rows, std::min(seg_max, F32_SEG));
  if (n % seg || (node_rows % seg) || seg % 64) return HODLR_ERR_ARG;
  // 8-byte row-pair accesses
  if ((ldc | lda) & 1 || (uintptr_t)C % 8 || (uintptr_t)A1 % 8 || (uintptr_t)V % 8) return HODLR_ERR_ARG;
  const int64_t nseg = n / seg;
  const bool split = seg < node_rows && V != nullptr;
  if (split && (size_t)nseg * F32_R * ncols * sizeof(float) > part_bytes) return HODLR_ERR_ARG;
  LevelF32Args g{C, ldc, A1, V, lda, W, wstride, n_c, node_rows, ncols, (int)seg, (int)ceil_div(ncols, 8),
                 split ? part : TW, tw_stride, split ? 1 : 0};
  const int64_t grid = nseg * g.chunks;
  if (grid > 2147483647LL) return HODLR_ERR_ARG;
  if (g.ncols > 4) {  // chunks of 8 columns (ceil(ncols / 8) warps per segment)
    level_f32_kernel<8><<<(unsigned)grid, 32, 0, st>>>(g);
  } else if (g.ncols > 2) {
    level_f32_kernel<4><<<(unsigned)grid, 32, 0, st>>>(g);
  } else if (g.ncols == 2) {
    level_f32_kernel<2><<<(unsigned)grid, 32, 0, st>>>(g);
  } else {
    level_f32_kernel<1><<<(unsigned)grid, 32, 0, st>>>(g);
  }
  HODLR_CHECK_LAUNCH();
  if (!split) return HODLR_OK;
  const int nnodes = (int)(n / node_rows);
  const int64_t total = (int64_t)F32_R * ncols * nnodes;
  level_reduce_f32_kernel<<<(unsigned)std::min<int64_t>(ceil_div(total, 8), 4736), 256, 0, st>>>(
      part, TW, ncols, (int)(node_rows / seg), nnodes, tw_stride);
  HODLR_CHECK_LAUNCH();
  return HODLR_OK;
}

}  // namespace hodlr
