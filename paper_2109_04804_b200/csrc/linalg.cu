// linalg.cu -- BJ_ext block inversion and application, GMRES/Newton vector ops.
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include "launch.h"
#include "tma.cuh"

long long g_hbpdc_launches = 0;

// ============================================================================
// Batched Gauss-Jordan inversion with partial pivoting ("we calculate
// those inverses via LU-decomposition"; any pivoted elimination gives the same
// inverse up to rounding).  One CTA per m x m matrix (m <= 256), matrix in
// global memory (L2-resident while its CTA runs).
//
// Blocked in-place GJ with implicit pivoting: panel of NB columns is
// eliminated in shared memory (pivot search over rows not yet used), which
// yields U = E_panel[:, P] - I[:, P]; every other column j then receives the
// rank-NB update A[:, j] += U A[P, j].  The stored matrix Z satisfies
// A^-1[a][b] = Z[p_a][q_b] with p_a the pivot row of column a and q_b the
// column whose pivot row is b; the final pass writes that into S.
// ============================================================================
namespace {
__device__ __forceinline__ void gj_dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}
#ifndef GJ_PIPE
#define GJ_PIPE 1
#endif
#ifndef GJ_ROT
#define GJ_ROT 1
#endif
#ifndef GJ_REDUX
#define GJ_REDUX 1
#endif
#ifndef GJ_ROTG
#define GJ_ROTG 8
#endif
constexpr int GJ_TW = 32;    // column tile of the rank-NB update
constexpr int GJ_APS = GJ_TW + 4;  // pivot-row tile stride (conflict-free B fragments)
#ifndef GJ_MINB
#define GJ_MINB 2
#endif
}

// GJ_NB: panel width.  Each panel step streams the whole matrix through L2 (DRAM once the
// in-flight matrices overflow L2), so a wider panel means proportionally fewer passes.
// GJ_T threads (= the largest m: thread r owns row r): 256 for the 2D configs, 384 for the
// 3D hexahedra (m = 5 * 4^3 = 320, NEXT-4).
// MC: the block size as a compile-time constant (0: runtime m).  MC == GJ_T with MC a multiple
// of GJ_NB (the 2D N = 7 blocks, m = 256) drops every bounds guard of the panel and the trailing
// update (ncu r02o: 16 % ISETP, 10 % IMAD of the executed instructions; the DMMAs were 7 %).
template <int GJ_NB, int GJ_T, int MC = 0>
__global__ void __launch_bounds__(GJ_T, GJ_T > 256 ? 1 : GJ_MINB) gj_kernel(double* __restrict__ Zall,
                                                                          double* __restrict__ Sall, int m_in,
                                                                          int* __restrict__ info) {
  constexpr bool FULL = MC == GJ_T && MC % GJ_NB == 0;
  const int m = MC ? MC : m_in;
  constexpr int GJ_MMAX = GJ_T;
  constexpr int GJ_PS = GJ_NB + 4;   // panel row stride (== 4 mod 16: conflict-free DMMA A fragments)
  extern __shared__ __align__(16) double gj_dyn[];
  double* Pn = gj_dyn;                       // panel [GJ_MMAX][GJ_PS]
  double* AP = gj_dyn + GJ_MMAX * GJ_PS;     // pivot rows of a column tile [GJ_NB][GJ_APS]
  __shared__ int piv[GJ_MMAX];      // pivot row of column c
  __shared__ int colof[GJ_MMAX];    // column whose pivot row is r (-1: unused)
#if GJ_REDUX
  __shared__ unsigned long long redk[GJ_T / 32];
#else
  __shared__ double redv[GJ_T / 32];
#endif
  __shared__ int redi[GJ_T / 32];
  __shared__ double prb[GJ_NB];      // pivot row / pivot of the current column
  __shared__ double s_pval;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  double* A = Zall + (size_t)blockIdx.x * m * m;
  double* S = Sall + (size_t)blockIdx.x * m * m;
  for (int q = tid; q < m; q += GJ_T) colof[q] = -1;
  int singular = 0;
  __syncthreads();

  // thread r owns panel row r in registers (m <= GJ_T): two barriers per column
  const int r = tid;
  bool used = false;
  for (int c0 = 0; c0 < m; c0 += GJ_NB) {
    const int nb = FULL ? GJ_NB : min(GJ_NB, m - c0);
    {
    double row[GJ_NB];
#pragma unroll
    for (int j = 0; j < GJ_NB; ++j) row[j] = (FULL || (r < m && j < nb)) ? A[(size_t)r * m + c0 + j] : 0.0;
    int mycol = -1;                                  // panel column this row pivoted
    // one pivot step: ks = the register slot holding the pivot column (compile-time after
    // unrolling), kc = the panel column it stands for
    auto pivot_step = [&](const int ks, const int kc) {
      // ---- pivot search: max |row[ks]| over unused rows (ties: smallest r)
      // a NaN entry ranks as +inf so that some row is always chosen (a NaN pivot must not leave
      // the column without a pivot row); non-finite pivots are reported as singular below
#if GJ_REDUX
      // 64-bit key = bits(|x|) + 1 for a candidate row (monotone in |x| >= 0, NaN ranked as +inf),
      // 0 otherwise; the maximum by three 32-bit warp reductions (high word, low word among the
      // lanes that hold the high maximum, smallest row among the lanes that hold both) instead of
      // five shuffle rounds of (value, index) pairs -- the same pivot row as before, bit for bit.
      const bool cand = (FULL || r < m) && !used;
      const double ax = isnan(row[ks]) ? INFINITY : fabs(row[ks]);
      const unsigned long long key = cand ? (unsigned long long)__double_as_longlong(ax) + 1ull : 0ull;
      auto kmax3 = [](unsigned long long kk, unsigned ri, unsigned long long& ko, unsigned& ro) {
        const unsigned hi = (unsigned)(kk >> 32), lo = (unsigned)kk;
        const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
        const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
        ro = __reduce_min_sync(0xffffffffu, (kk != 0ull && hi == mh && lo == ml) ? ri : 0x7fffffffu);
        ko = ((unsigned long long)mh << 32) | ml;
      };
      unsigned long long wk;
      unsigned wr;
      kmax3(key, (unsigned)r, wk, wr);
      if (lane == 0) { redk[wid] = wk; redi[wid] = (int)wr; }
      __syncthreads();
      unsigned long long bk;
      unsigned bu;
      kmax3(lane < GJ_T / 32 ? redk[lane] : 0ull, lane < GJ_T / 32 ? (unsigned)redi[lane] : 0x7fffffffu, bk, bu);
      const int bi = (int)bu;
      const double best = bk ? __longlong_as_double((long long)(bk - 1ull)) : -1.0;
#else
      const bool cand = (FULL || r < m) && !used;
      double best = cand ? (isnan(row[ks]) ? INFINITY : fabs(row[ks])) : -1.0;
      int bi = cand ? r : 0x7fffffff;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      if (lane == 0) { redv[wid] = best; redi[wid] = bi; }
      __syncthreads();
      best = redv[0]; bi = redi[0];
#pragma unroll
      for (int w = 1; w < GJ_T / 32; ++w)
        if (redv[w] > best || (redv[w] == best && redi[w] < bi)) { best = redv[w]; bi = redi[w]; }
#endif
      const bool sing = !(best > 0.0) || !(best < INFINITY);
      if (r == bi) {                                 // the pivot row: broadcast it scaled by 1/pivot
        const double pinv = 1.0 / (sing ? 1.0 : row[ks]);
#pragma unroll
        for (int j = 0; j < GJ_NB; ++j) prb[j] = row[j] * pinv;
        s_pval = pinv;
        used = true;
        mycol = kc;
        colof[r] = c0 + kc;
        piv[c0 + kc] = r;
      }
      __syncthreads();
      if (sing) singular = 1;
      const double pinv = s_pval;
      // ---- in-place GJ step on the panel columns
      if (FULL || r < m) {
        if (r == bi) {
#pragma unroll
          for (int j = 0; j < GJ_NB; ++j) row[j] = j == ks ? pinv : prb[j];
        } else {
          const double fr = row[ks];
#pragma unroll
          for (int j = 0; j < GJ_NB; ++j) row[j] = j == ks ? -fr * pinv : fma(-fr, prb[j], row[j]);
        }
      }
        };
    constexpr bool PFULL = MC != 0 && MC % GJ_NB == 0;     // every panel has GJ_NB columns
    if constexpr ((GJ_ROT == 2 ? PFULL : (GJ_ROT == 1 && FULL)) && GJ_NB % GJ_ROTG == 0) {
      // The fully unrolled panel (GJ_NB pivot steps) is ~9k instructions, more than the
      // instruction cache keeps for 16 warps at different places in it (ncu r02y: 14 % of the
      // stall samples "no instruction").  Unroll GJ_ROTG steps only and rotate the row registers
      // (and with them the order of the broadcast pivot row) by GJ_ROTG slots after each group:
      // the pivot column is always in slots 0 .. GJ_ROTG-1, and after GJ_NB / GJ_ROTG rotations
      // the columns are back in place.
#pragma unroll 1
      for (int kg = 0; kg < GJ_NB; kg += GJ_ROTG) {
#pragma unroll
        for (int kk = 0; kk < GJ_ROTG; ++kk) pivot_step(kk, kg + kk);
        double tmp[GJ_ROTG];
#pragma unroll
        for (int j = 0; j < GJ_ROTG; ++j) tmp[j] = row[j];
#pragma unroll
        for (int j = 0; j + GJ_ROTG < GJ_NB; ++j) row[j] = row[j + GJ_ROTG];
#pragma unroll
        for (int j = 0; j < GJ_ROTG; ++j) row[GJ_NB - GJ_ROTG + j] = tmp[j];
      }
    } else {
#pragma unroll
      for (int k = 0; k < GJ_NB; ++k) {
        if (!FULL && k >= nb) break;
        pivot_step(k, k);
      }
    }
    // ---- store the panel (augmented columns E[:, P]); U = panel - I[:, P] to shared memory
    if (FULL || r < m) {
#pragma unroll
      for (int j = 0; j < GJ_NB; ++j)
        if (FULL || j < nb) {
          A[(size_t)r * m + c0 + j] = row[j];
          Pn[r * GJ_PS + j] = j == mycol ? row[j] - 1.0 : row[j];
        }
    }
    }
    __syncthreads();
    // ---- rank-nb update of every other column: A[:, j] += U A[P, j], on the fp64
    //      tensor cores: per 32-column tile warp w owns rows 32w .. 32w + 31 as
    //      4 x 4 DMMA tiles (8 x 8), k = the panel's 16 columns in 4 k-steps;
    //      A fragments (U) from the panel, B fragments (pivot rows) from AP
    const int g = lane >> 2, t4 = lane & 3;
#if GJ_PIPE
    // Software pipeline over the column tiles (r02zg): the tile's accumulators are loaded
    // BEFORE the barrier that publishes its pivot rows, and the next tile's pivot rows are
    // gathered into registers while this tile's DMMAs run (AP double-buffered), so a tile
    // exposes one global round trip instead of two dependent ones and one barrier instead
    // of two.  The tile made of the panel's own columns is skipped (its result was discarded).
    constexpr int NAPL = (GJ_NB * GJ_TW + GJ_T - 1) / GJ_T;
    constexpr bool SKIP_OWN = GJ_NB == GJ_TW;
    auto ap_load = [&](int t0, double (&v)[NAPL]) {
#pragma unroll
      for (int q = 0; q < NAPL; ++q) {
        const int idx = tid + q * GJ_T;
        const int k = idx / GJ_TW, jj = idx % GJ_TW;
        const int col = t0 + jj;
        const bool in = (GJ_NB * GJ_TW) % GJ_T == 0 || idx < GJ_NB * GJ_TW;
        v[q] = (in && (FULL || (k < nb && col < m))) ? A[(size_t)piv[c0 + k] * m + col] : 0.0;
      }
    };
    auto next_tile = [&](int t0) {
      t0 += GJ_TW;
      if (SKIP_OWN && t0 == c0) t0 += GJ_TW;
      return t0;
    };
    int t0 = (SKIP_OWN && c0 == 0) ? GJ_TW : 0;
    double apv[NAPL];
    if (t0 < m) ap_load(t0, apv);
    for (int it = 0; t0 < m; t0 = next_tile(t0), ++it) {
      double* APb = AP + (it & 1) * (GJ_NB * GJ_APS);
      const bool mine = FULL || 32 * wid < m;
      double acc[4][4][2];
      if (mine) {
#pragma unroll
        for (int rb = 0; rb < 4; ++rb) {
          const int r = 32 * wid + 8 * rb + g;
#pragma unroll
          for (int cb = 0; cb < 4; ++cb) {
            const int col = t0 + 8 * cb + 2 * t4;
            if (FULL) {
              const double2 v = *reinterpret_cast<const double2*>(A + (size_t)r * m + col);
              acc[rb][cb][0] = v.x;
              acc[rb][cb][1] = v.y;
            } else {
              acc[rb][cb][0] = (r < m && col < m) ? A[(size_t)r * m + col] : 0.0;
              acc[rb][cb][1] = (r < m && col + 1 < m) ? A[(size_t)r * m + col + 1] : 0.0;
            }
          }
        }
      }
#pragma unroll
      for (int q = 0; q < NAPL; ++q) {
        const int idx = tid + q * GJ_T;
        if ((GJ_NB * GJ_TW) % GJ_T == 0 || idx < GJ_NB * GJ_TW) APb[(idx / GJ_TW) * GJ_APS + idx % GJ_TW] = apv[q];
      }
      __syncthreads();
      const int tn = next_tile(t0);
      if (tn < m) ap_load(tn, apv);
      if (mine) {
#pragma unroll
        for (int ks = 0; ks < GJ_NB / 4; ++ks) {
          const int kk = 4 * ks + t4;
          double av[4], bv[4];
#pragma unroll
          for (int rb = 0; rb < 4; ++rb) {
            const int r = 32 * wid + 8 * rb + g;
            av[rb] = (FULL || (r < m && kk < nb)) ? Pn[r * GJ_PS + kk] : 0.0;
          }
#pragma unroll
          for (int cb = 0; cb < 4; ++cb) bv[cb] = APb[kk * GJ_APS + 8 * cb + g];
#pragma unroll
          for (int rb = 0; rb < 4; ++rb)
#pragma unroll
            for (int cb = 0; cb < 4; ++cb) gj_dmma(acc[rb][cb], av[rb], bv[cb]);
        }
#pragma unroll
        for (int rb = 0; rb < 4; ++rb) {
          const int r = 32 * wid + 8 * rb + g;
          if (!FULL && r >= m) continue;
#pragma unroll
          for (int cb = 0; cb < 4; ++cb) {
            const int col = t0 + 8 * cb + 2 * t4;
            if (FULL && SKIP_OWN) {
              *reinterpret_cast<double2*>(A + (size_t)r * m + col) = make_double2(acc[rb][cb][0], acc[rb][cb][1]);
            } else {
#pragma unroll
              for (int h = 0; h < 2; ++h)
                if ((FULL || col + h < m) && (col + h < c0 || col + h >= c0 + nb)) A[(size_t)r * m + col + h] = acc[rb][cb][h];
            }
          }
        }
      }
    }
    __syncthreads();     // every tile is stored before the next panel (or the unpermute) reads A
#else
    for (int t0 = 0; t0 < m; t0 += GJ_TW) {
      for (int idx = tid; idx < GJ_NB * GJ_TW; idx += GJ_T) {
        const int k = idx / GJ_TW, jj = idx % GJ_TW;
        const int col = t0 + jj;
        AP[k * GJ_APS + jj] = (FULL || (k < nb && col < m)) ? A[(size_t)piv[c0 + k] * m + col] : 0.0;
      }
      __syncthreads();
      if (FULL || 32 * wid < m) {
        double acc[4][4][2];
#pragma unroll
        for (int rb = 0; rb < 4; ++rb) {
          const int r = 32 * wid + 8 * rb + g;
#pragma unroll
          for (int cb = 0; cb < 4; ++cb) {
            const int col = t0 + 8 * cb + 2 * t4;
            acc[rb][cb][0] = (FULL || (r < m && col < m)) ? A[(size_t)r * m + col] : 0.0;
            acc[rb][cb][1] = (FULL || (r < m && col + 1 < m)) ? A[(size_t)r * m + col + 1] : 0.0;
          }
        }
#pragma unroll
        for (int ks = 0; ks < GJ_NB / 4; ++ks) {
          const int kk = 4 * ks + t4;
          double av[4], bv[4];
#pragma unroll
          for (int rb = 0; rb < 4; ++rb) {
            const int r = 32 * wid + 8 * rb + g;
            av[rb] = (FULL || (r < m && kk < nb)) ? Pn[r * GJ_PS + kk] : 0.0;
          }
#pragma unroll
          for (int cb = 0; cb < 4; ++cb) bv[cb] = AP[kk * GJ_APS + 8 * cb + g];
#pragma unroll
          for (int rb = 0; rb < 4; ++rb)
#pragma unroll
            for (int cb = 0; cb < 4; ++cb) gj_dmma(acc[rb][cb], av[rb], bv[cb]);
        }
#pragma unroll
        for (int rb = 0; rb < 4; ++rb) {
          const int r = 32 * wid + 8 * rb + g;
          if (!FULL && r >= m) continue;
#pragma unroll
          for (int cb = 0; cb < 4; ++cb)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int col = t0 + 8 * cb + 2 * t4 + h;
              if ((FULL || col < m) && (col < c0 || col >= c0 + nb)) A[(size_t)r * m + col] = acc[rb][cb][h];
            }
        }
      }
      __syncthreads();
    }
#endif
  }
  // ---- unpermute: S[a][b] = Z[piv[a]][colof[b]]
  for (int a = wid; a < m; a += GJ_T / 32) {
    const double* zr = A + (size_t)piv[a] * m;
    for (int b = lane; b < m; b += 32) S[(size_t)a * m + b] = zr[colof[b]];
  }
  if (singular && tid == 0) info[blockIdx.x] = 1;
}

cudaError_t launch_gj_invert(double* Z, double* S, int m, int nmat, int* info, cudaStream_t st) {
  if (m > 384 || m < 1) return cudaErrorInvalidValue;
  if (nmat <= 0) return cudaSuccess;
  // Panel width: 16 (r01) or 32 (default, HBPDC_GJ_NB).  Occupancy: every resident CTA streams its
  // whole m x m matrix through L2 on each of the m / NB panel updates; 2 CTAs/SM x 148 SMs x
  // 512 KB (m = 256) overflow the 126 MB L2.  One CTA per SM (HBPDC_GJ_OCC=1, 76 MB in flight)
  // was measured slower (C3 build 116 -> 141 ms, r02b): the pivot-search latency is no longer
  // hidden.  Default 2.
  static const int nb = [] {
    const char* e = getenv("HBPDC_GJ_NB");
    return e && atoi(e) == 16 ? 16 : 32;
  }();
  static const int occ = [] {
    const char* e = getenv("HBPDC_GJ_OCC");
    return e ? atoi(e) : 2;
  }();
  auto go = [&](auto kern, int NB, int T) {
    size_t smem = (size_t)(T * (NB + 4) + (GJ_PIPE ? 2 : 1) * NB * GJ_APS) * sizeof(double);
    if (occ == 1 && m > 128) smem = std::max<size_t>(smem, 120 * 1024);   // one CTA per SM
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<nmat, T, smem, st>>>(Z, S, m, info);
  };
#ifndef GJ_T320
#define GJ_T320 1
#endif
  if (m == 320 && GJ_T320) go(gj_kernel<32, 320, 320>, 32, 320);     // 3D N = 3 (T3): 10 warps, guard-free
  else if (m == 320) go(gj_kernel<32, 384, 320>, 32, 384);            // 3D N = 3 (T3)
  else if (m > 256) go(gj_kernel<32, 384>, 32, 384);
  else if (m == 144 && !getenv("HBPDC_GJ_T256")) go(gj_kernel<32, 160, 144>, 32, 160);   // C5: N = 5
  else if (m <= 160 && !getenv("HBPDC_GJ_T256")) go(gj_kernel<32, 160>, 32, 160);
  else if (nb == 16) go(gj_kernel<16, 256>, 16, 256);
  else if (m == 256) go(gj_kernel<32, 256, 256>, 32, 256);     // the 2D N = 7 blocks (C3, C4)
  else go(gj_kernel<32, 256>, 32, 256);
  hbpdc_count_launch();
  return cudaGetLastError();
}

// ============================================================================
// BJ_ext application, streaming half: U_e = S_e W_e, V_e = S_e sigma_e.
// One CTA (8 warps) per element; each warp takes 4 rows at a time, lane l
// reads columns l, l+32, ... (coalesced 256-B segments of a row), keeps the
// matching W/sigma entries in registers, and reduces 8 partial sums across
// the warp with a butterfly that halves the payload at each stage.
// S is read exactly once: this is the HBM-bound kernel (8 m^2 B / element).
// ============================================================================
template <int CPL>
__global__ void __launch_bounds__(256) gemv2_kernel(const double* __restrict__ S, int shared,
                                                    const double* __restrict__ W, const double* __restrict__ sg,
                                                    double* __restrict__ U, double* __restrict__ V, int m, int nE) {
  const int e = blockIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const double* Se = S + (shared ? 0 : (size_t)e * m * m);
  const double* we = W + (size_t)e * m;
  const double* se = sg + (size_t)e * m;
  double wr[CPL], sr[CPL];
#pragma unroll
  for (int q = 0; q < CPL; ++q) {
    const int c = lane + 32 * q;
    wr[q] = c < m ? we[c] : 0.0;
    sr[q] = c < m ? se[c] : 0.0;
  }
  for (int r0 = wid * 4; r0 < m; r0 += 32) {
    double p[8];
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) {
      const int r = r0 + rr;
      double a = 0.0, b = 0.0;
      if (r < m) {
        const double* row = Se + (size_t)r * m;
#pragma unroll
        for (int q = 0; q < CPL; ++q) {
          const int c = lane + 32 * q;
          const double s = c < m ? __ldg(row + c) : 0.0;
          a = fma(s, wr[q], a);
          b = fma(s, sr[q], b);
        }
      }
      p[2 * rr] = a;
      p[2 * rr + 1] = b;
    }
    // butterfly: 8 values over 32 lanes -> value (lane >> 2) & 7 complete in lanes
    {
      const bool hi = lane & 16;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const double send = hi ? p[t] : p[t + 4];
        const double recv = __shfl_xor_sync(0xffffffffu, send, 16);
        p[t] = (hi ? p[t + 4] : p[t]) + recv;
      }
    }
    {
      const bool hi = lane & 8;
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const double send = hi ? p[t] : p[t + 2];
        const double recv = __shfl_xor_sync(0xffffffffu, send, 8);
        p[t] = (hi ? p[t + 2] : p[t]) + recv;
      }
    }
    {
      const bool hi = lane & 4;
      const double send = hi ? p[0] : p[1];
      const double recv = __shfl_xor_sync(0xffffffffu, send, 4);
      p[0] = (hi ? p[1] : p[0]) + recv;
    }
    p[0] += __shfl_xor_sync(0xffffffffu, p[0], 2);
    p[0] += __shfl_xor_sync(0xffffffffu, p[0], 1);
    // lane bits (4,3,2) select the value index: idx = 4*b4 + 2*b3 + b2
    if ((lane & 3) == 0) {
      const int idx = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
      const int r = r0 + (idx >> 1);
      if (r < m) {
        if (idx & 1) V[(size_t)e * m + r] = p[0];
        else U[(size_t)e * m + r] = p[0];
      }
    }
  }
}

// ---- TMA-streamed variant (per-element S): persistent CTAs walk their
// elements' S blocks in chunks of GT_R rows; thread 0 keeps GT_NST chunks in
// flight with cp.async.bulk (completion on an mbarrier), the 8 warps reduce
// one row each per chunk from shared memory.

// NR right-hand sides (NR = 2: u = S W, v = S sigma of one system; NR = 2B: the
// B corrector-stage systems of a sweep solved in lock step share ONE pass over
// S).  Every output row is accumulated in the same order for
// any NR, so batched and single-system results are bitwise identical.
struct GemvRHS {
  const double* in[GEMV_MAX_RHS];
  double* out[GEMV_MAX_RHS];
};


// Warp-specialised pipeline: warp 8 (one lane) is the producer, warps 0-7
// consume.  Per element the producer bulk-copies the NR right-hand-side
// vectors into one of two RHS buffers, then streams the element's S in chunks
// of ROWS rows through a GT_NST-deep ring; "full" mbarriers carry the
// transaction bytes, "empty" mbarriers collect one arrival per consumer warp,
// so warps drift independently through the ring (no CTA-wide barrier per chunk).
// Up to 4 right-hand sides live in one warp's registers; NR = 6 splits them
// over 2 warps per row (each reads the full row, 3 RHS, 2 rows per chunk to
// keep two independent FMA chains).  Each output is one warp's full-row dot
// product, reduced over the same lane tree for every NR (bitwise equal).
// Measured at C3 size (scripts/bench_gemv.cu): NR = 2, 4: 6.8-6.9 TB/s
// (104-105% of the measured copy bandwidth), NR = 6: 5.8 TB/s.
// consumer warps (one CTA per SM)
template <int NR> struct GwCons { static constexpr int value = 16; };
#ifndef GW_WPR_MAXK
#define GW_WPR_MAXK 4                            // right-hand sides one warp keeps in registers
#endif
constexpr int GW_NST_MAX = 16;                   // ring stages (runtime nst <= this)
constexpr size_t GW_RING_BYTES = 160 * 1024;     // S bytes in flight per CTA (one CTA per SM)

template <int CPL, int NR>
__global__ void __launch_bounds__(32 * (GwCons<NR>::value + 1)) gemvN_tma_kernel(const double* __restrict__ S,
                                                                       const GemvRHS io, int m, int nE,
                                                                       int GW_NST) {
  constexpr int GW_CONS = GwCons<NR>::value;
  constexpr int WPR = NR > GW_WPR_MAXK ? 2 : 1;  // warps per row
  constexpr int KPW = NR / WPR;                  // right-hand sides per warp
  constexpr int ROWS = GW_CONS;                  // rows per chunk
  constexpr int RPW = WPR;                       // rows per warp per chunk (interleaved chains)
  extern __shared__ __align__(128) unsigned char smraw[];
  double* ring = reinterpret_cast<double*>(smraw);                     // GW_NST x ROWS x m
  double* rhs = ring + (size_t)GW_NST * ROWS * m;                      // 2 x NR x m
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(rhs + (size_t)2 * NR * m);
  unsigned long long *fullS = bars, *emptyS = bars + GW_NST_MAX, *fullR = bars + 2 * GW_NST_MAX, *emptyR = fullR + 2;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int cpe = (m + ROWS - 1) / ROWS;                               // chunks per element
  const int nmy = blockIdx.x < nE ? (nE - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  if (threadIdx.x == 0) {
    for (int q = 0; q < GW_NST; ++q) { mbar_init(&fullS[q], 1); mbar_init(&emptyS[q], GW_CONS); }
    for (int q = 0; q < 2; ++q) { mbar_init(&fullR[q], 1); mbar_init(&emptyR[q], GW_CONS); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (wid == GW_CONS) {                                                // ---- producer
    if (lane == 0) {
      int c = 0;                                                       // chunk counter
      for (int it = 0; it < nmy; ++it) {
        const int e = blockIdx.x + it * gridDim.x;
        const int rb = it & 1;
        if (it >= 2) mbar_wait(&emptyR[rb], (unsigned)(((it >> 1) - 1) & 1));
        mbar_expect_tx(&fullR[rb], (unsigned)(NR * m * sizeof(double)));
        for (int k = 0; k < NR; ++k)
          tma_load_1d(rhs + ((size_t)rb * NR + k) * m, io.in[k] + (size_t)e * m, (unsigned)(m * sizeof(double)),
                      &fullR[rb]);
        for (int ch = 0; ch < cpe; ++ch, ++c) {
          const int st = c % GW_NST;
          if (c >= GW_NST) mbar_wait(&emptyS[st], (unsigned)(((c / GW_NST) - 1) & 1));
          const int r0 = ch * ROWS;
          const int rows = min(ROWS, m - r0);
          const unsigned bytes = (unsigned)(rows * m * sizeof(double));
          mbar_expect_tx(&fullS[st], bytes);
          tma_load_1d(ring + (size_t)st * ROWS * m, S + ((size_t)e * m + r0) * m, bytes, &fullS[st]);
        }
      }
    }
    return;
  }
  // ---- consumers: warp wid takes rows wid / WPR + i ROWS / RPW (i < RPW) of
  //      every chunk, for right-hand sides k0 .. k0 + KPW - 1, k0 = (wid % WPR) KPW
  const int rslot = wid / WPR, k0 = (wid % WPR) * KPW;
  double xr[KPW][CPL];
  int c = 0;
  for (int it = 0; it < nmy; ++it) {
    const int e = blockIdx.x + it * gridDim.x;
    const int rb = it & 1;
    mbar_wait(&fullR[rb], (unsigned)((it >> 1) & 1));
#pragma unroll
    for (int k = 0; k < KPW; ++k)
#pragma unroll
      for (int q = 0; q < CPL; ++q) {
        const int col = lane + 32 * q;
        xr[k][q] = col < m ? rhs[((size_t)rb * NR + k0 + k) * m + col] : 0.0;
      }
    fence_proxy_async_smem();            // order this lane's reads before the buffer's next bulk copy
    __syncwarp();
    if (lane == 0) mbar_arrive(&emptyR[rb]);
    for (int ch = 0; ch < cpe; ++ch, ++c) {
      const int st = c % GW_NST;
      mbar_wait(&fullS[st], (unsigned)((c / GW_NST) & 1));
      double acc[RPW][KPW];
#pragma unroll
      for (int i = 0; i < RPW; ++i)
#pragma unroll
        for (int k = 0; k < KPW; ++k) acc[i][k] = 0.0;
#pragma unroll
      for (int q = 0; q < CPL; ++q) {
        const int col = lane + 32 * q;
#pragma unroll
        for (int i = 0; i < RPW; ++i) {
          const double* row = ring + ((size_t)st * ROWS + rslot + i * (ROWS / RPW)) * m;
          const double sv = col < m ? row[col] : 0.0;
#pragma unroll
          for (int k = 0; k < KPW; ++k) acc[i][k] = fma(sv, xr[k][q], acc[i][k]);
        }
      }
#pragma unroll
      for (int i = 0; i < RPW; ++i) {
        const int r = ch * ROWS + rslot + i * (ROWS / RPW);
        if constexpr (KPW <= 2) {
#pragma unroll
          for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int k = 0; k < KPW; ++k) acc[i][k] += __shfl_xor_sync(0xffffffffu, acc[i][k], o);
          if (r < m && lane < KPW) io.out[k0 + lane][(size_t)e * m + r] = lane == 0 ? acc[i][0] : acc[i][KPW - 1];
        } else {
          // KPW > 2: transposed butterfly over V = 4 or 8 (padded) values: step
          // jj halves the live values across lane bit 16 >> jj, the remaining
          // low lane bits are a plain reduction; lane bits 4 .. 5 - LV then
          // index the value.  Each value is summed over the same lane tree
          // (bits 16, 8, 4, 2, 1) as the plain butterfly (operands swapped at
          // most: a + b == b + a), so results are bitwise equal to KPW <= 2.
          constexpr int V = KPW <= 4 ? 4 : 8;
          constexpr int LV = V == 4 ? 2 : 3;
          double p[V];
#pragma unroll
          for (int k = 0; k < V; ++k) p[k] = k < KPW ? acc[i][k] : 0.0;
#pragma unroll
          for (int jj = 0; jj < LV; ++jj) {
            const int h = V >> (jj + 1), mask = 16 >> jj;
            const bool hi = lane & mask;
#pragma unroll
            for (int q = 0; q < h; ++q) {
              const double send = hi ? p[q] : p[q + h];
              const double recv = __shfl_xor_sync(0xffffffffu, send, mask);
              p[q] = (hi ? p[q + h] : p[q]) + recv;
            }
          }
#pragma unroll
          for (int mask = 16 >> LV; mask >= 1; mask >>= 1) p[0] += __shfl_xor_sync(0xffffffffu, p[0], mask);
          int idx = 0;
#pragma unroll
          for (int jj = 0; jj < LV; ++jj)
            if (lane & (16 >> jj)) idx |= V >> (jj + 1);
          if (r < m && (lane & ((32 >> LV) - 1)) == 0 && idx < KPW) io.out[k0 + idx][(size_t)e * m + r] = p[0];
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&emptyS[st]);
    }
  }
}

// ---- fp64 tensor-core variant (all NR through the same kernel, so batched and
// single-system outputs stay bitwise equal): per element, out (m x 8, NR used
// columns) = S_e (m x m) X (m x 8) with mma.sync m8n8k4 f64.  Same producer /
// ring as gemvN_tma_kernel (chunks of GD_ROWS rows).  Consumer warp w takes row
// block w & 1 (8 rows) of each chunk and k-range w >> 1 (kw k-steps, two per
// 16-byte shared load: column 4 kr kw + 8 p + 2 t + (ks & 1)), with its B
// fragments (the right-hand sides) in registers for the whole element.  The 8
// k-range partials of a row block are summed in warp order through shared
// memory (one named barrier per chunk, double-buffered), so every output has a
// fixed summation order independent of NR.  Why: the FMA kernel reads each S value once per
// 3 right-hand sides and is issue-bound at 6 (5.6 TB/s); here one 16-byte
// load feeds two DMMAs of all 8 columns.
constexpr int GD_CONS = 16;                       // consumer warps
constexpr int GD_KWMAX = 8;                       // k-steps per warp (m <= 256)

// RB row blocks of 8 rows per chunk x (GD_CONS / RB) k-ranges: RB = 2 (m = 256: every k-range full)
// or RB = 4 (m = 144: 4 k-ranges of 40 columns keep 90 % of the consumer warps busy instead of 75 %
// with 8 k-ranges of 24 -- the chunk's makespan is the busiest warp's).
template <int NR, int RB = 2, int KWMAX = GD_KWMAX>
__global__ void __launch_bounds__(32 * (GD_CONS + 1), 1) gemv_dmma_kernel(const double* __restrict__ S,
                                                                         const GemvRHS io, int m, int nE,
                                                                         int GW_NST, int kw) {
  constexpr int GD_ROWS = 8 * RB;                                      // rows per chunk
  constexpr int KR = GD_CONS / RB;                                     // k-ranges
  extern __shared__ __align__(128) unsigned char smraw[];
  double* ring = reinterpret_cast<double*>(smraw);                     // GW_NST x GD_ROWS x m
  double* rhs = ring + (size_t)GW_NST * GD_ROWS * m;                   // 2 x NR x m
  double* red = rhs + (size_t)2 * NR * m;                              // 2 x GD_CONS x 64
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(red + 2 * GD_CONS * 64);
  unsigned long long *fullS = bars, *emptyS = bars + GW_NST_MAX, *fullR = bars + 2 * GW_NST_MAX, *emptyR = fullR + 2;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int cpe = (m + GD_ROWS - 1) / GD_ROWS;
  __shared__ double* sOut[NR];                                         // output pointers (indexed per thread)
  if (threadIdx.x < NR) sOut[threadIdx.x] = io.out[threadIdx.x];
  const int nmy = blockIdx.x < nE ? (nE - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  if (threadIdx.x == 0) {
    for (int q = 0; q < GW_NST; ++q) { mbar_init(&fullS[q], 1); mbar_init(&emptyS[q], GD_CONS); }
    for (int q = 0; q < 2; ++q) { mbar_init(&fullR[q], 1); mbar_init(&emptyR[q], GD_CONS); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (wid == GD_CONS) {                                                // ---- producer
    if (lane == 0) {
      int c = 0;
      for (int it = 0; it < nmy; ++it) {
        const int e = blockIdx.x + it * gridDim.x;
        const int rb = it & 1;
        if (it >= 2) mbar_wait(&emptyR[rb], (unsigned)(((it >> 1) - 1) & 1));
        mbar_expect_tx(&fullR[rb], (unsigned)(NR * m * sizeof(double)));
        for (int k = 0; k < NR; ++k)
          tma_load_1d(rhs + ((size_t)rb * NR + k) * m, io.in[k] + (size_t)e * m, (unsigned)(m * sizeof(double)),
                      &fullR[rb]);
        for (int ch = 0; ch < cpe; ++ch, ++c) {
          const int st = c % GW_NST;
          if (c >= GW_NST) mbar_wait(&emptyS[st], (unsigned)(((c / GW_NST) - 1) & 1));
          const int r0 = ch * GD_ROWS;
          const int rows = min(GD_ROWS, m - r0);
          const unsigned bytes = (unsigned)(rows * m * sizeof(double));
          mbar_expect_tx(&fullS[st], bytes);
          tma_load_1d(ring + (size_t)st * GD_ROWS * m, S + ((size_t)e * m + r0) * m, bytes, &fullS[st]);
        }
      }
    }
    return;
  }
  const int g = lane >> 2, t = lane & 3;
  const int rbk = wid % RB, kr = wid / RB;
  const int cbase = 4 * kr * kw + 2 * t;          // + 8 p + (ks & 1)
  int c = 0;
  for (int it = 0; it < nmy; ++it) {
    const int e = blockIdx.x + it * gridDim.x;
    const int rb = it & 1;
    mbar_wait(&fullR[rb], (unsigned)((it >> 1) & 1));
    double b[KWMAX];
#pragma unroll
    for (int ks = 0; ks < KWMAX; ++ks) {
      const int col = cbase + 8 * (ks >> 1) + (ks & 1);
      b[ks] = (ks < kw && g < NR && col < m) ? rhs[((size_t)rb * NR + g) * m + col] : 0.0;
    }
    fence_proxy_async_smem();            // order this lane's reads before the buffer's next bulk copy
    __syncwarp();
    if (lane == 0) mbar_arrive(&emptyR[rb]);
    for (int ch = 0; ch < cpe; ++ch, ++c) {
      const int st = c % GW_NST;
      const int buf = c & 1;
      mbar_wait(&fullS[st], (unsigned)((c / GW_NST) & 1));
      const double* ar = ring + ((size_t)st * GD_ROWS + 8 * rbk + g) * m;
      double ae[2] = {0.0, 0.0}, ao[2] = {0.0, 0.0};
#pragma unroll
      for (int p = 0; p < KWMAX / 2; ++p) {
        if (2 * p < kw) {
          const int col = cbase + 8 * p;
          double2 a2 = make_double2(0.0, 0.0);
          if (col < m) a2 = *reinterpret_cast<const double2*>(ar + col);
          gj_dmma(ae, a2.x, b[2 * p]);
          gj_dmma(ao, a2.y, b[2 * p + 1]);
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&emptyS[st]);
      double* rw = red + ((size_t)buf * GD_CONS + wid) * 64 + g * 8 + 2 * t;
      rw[0] = ae[0] + ao[0];
      rw[1] = ae[1] + ao[1];
      asm volatile("bar.sync 1, %0;" ::"n"(32 * GD_CONS) : "memory");
      if (threadIdx.x < GD_ROWS * NR) {
        const int r = threadIdx.x / NR, j = threadIdx.x % NR;
        const double* rr = red + (size_t)buf * GD_CONS * 64 + (r >> 3) * 64 + (r & 7) * 8 + j;
        double s0 = 0.0, s1 = 0.0;                  // two chains, fixed order (warp kr RB + rb)
#pragma unroll
        for (int q = 0; q < KR; q += 2) {
          s0 += rr[(size_t)RB * q * 64];
          s1 += rr[(size_t)RB * (q + 1) * 64];
        }
        const int row = ch * GD_ROWS + r;
        if (row < m) sOut[j][(size_t)e * m + row] = s0 + s1;
      }
    }
  }
}

template <int NR, int RB = 2, int KWMAX = GD_KWMAX>
static cudaError_t launch_gemv_dmma_rb(const double* S, const GemvRHS& io, int m, int nE, cudaStream_t st) {
  constexpr int GD_ROWS = 8 * RB;
  constexpr int KR = GD_CONS / RB;
  static int nsm = 0;
  if (!nsm) {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    nsm = v;
  }
  if (m > 4 * KWMAX * KR || (m & 1)) return cudaErrorInvalidValue;
  int kw = ((m + 3) / 4 + KR - 1) / KR;
  kw += kw & 1;                                   // k-steps in pairs (16-byte loads)
  const size_t chunk = (size_t)GD_ROWS * m * sizeof(double);
  const size_t fixed = (size_t)2 * NR * m * sizeof(double) + (size_t)2 * GD_CONS * 64 * sizeof(double) +
                       (2 * GW_NST_MAX + 4) * sizeof(unsigned long long);
  const int nst = (int)std::max<size_t>(2, std::min<size_t>(GW_NST_MAX, GW_RING_BYTES / chunk));
  const size_t smem = (size_t)nst * chunk + fixed;
  constexpr int threads = 32 * (GD_CONS + 1);
  cudaFuncSetAttribute(gemv_dmma_kernel<NR, RB, KWMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gemv_dmma_kernel<NR, RB, KWMAX>, threads, smem);
  const int grid = std::min(nE, nsm * std::max(occ, 1));
  gemv_dmma_kernel<NR, RB, KWMAX><<<grid, threads, smem, st>>>(S, io, m, nE, nst, kw);
  hbpdc_count_launch();
  return cudaGetLastError();
}

// row-block layout with the better consumer utilisation for this m (ties: RB = 2)
inline double gemv_util(int m, int RB) {
  const int KR = GD_CONS / RB;
  int kw = ((m + 3) / 4 + KR - 1) / KR;
  kw += kw & 1;
  return (double)m / (4.0 * KR * kw);
}

template <int NR>
static cudaError_t launch_gemv_dmma(const double* S, const GemvRHS& io, int m, int nE, cudaStream_t st) {
  static const bool off = getenv("HBPDC_GEMV_RB2") != nullptr;
  if (m > 256) return launch_gemv_dmma_rb<NR, 2, 10>(S, io, m, nE, st);     // 3D: m = 320, 8 k-ranges of 40
  if (!off && gemv_util(m, 4) > gemv_util(m, 2) + 1e-12) return launch_gemv_dmma_rb<NR, 4, 16>(S, io, m, nE, st);
  return launch_gemv_dmma_rb<NR, 2, GD_KWMAX>(S, io, m, nE, st);
}

template <int NR>
static cudaError_t launch_gemvN(const double* S, const GemvRHS& io, int m, int nE, cudaStream_t st) {
  static int nsm = 0;
  if (!nsm) {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    nsm = v;
  }
  constexpr int GW_CONS = GwCons<NR>::value;
  constexpr int ROWS = GW_CONS;                  // rows per chunk (as in the kernel)
  const size_t chunk = (size_t)ROWS * m * sizeof(double);
  const int nst = (int)std::max<size_t>(2, std::min<size_t>(GW_NST_MAX, GW_RING_BYTES / chunk));
  const size_t smem = (size_t)nst * chunk + (size_t)2 * NR * m * sizeof(double) +
                      (2 * GW_NST_MAX + 4) * sizeof(unsigned long long);
  const int cpl = (m + 31) / 32;
  constexpr int threads = 32 * (GW_CONS + 1);
  // persistent grid: exactly the resident CTAs
#define GT(C)                                                                                   \
  case C: {                                                                                     \
    cudaFuncSetAttribute(gemvN_tma_kernel<C, NR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    int occ = 0;                                                                                \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gemvN_tma_kernel<C, NR>, threads, smem); \
    const int grid = std::min(nE, nsm * std::max(occ, 1));                                      \
    gemvN_tma_kernel<C, NR><<<grid, threads, smem, st>>>(S, io, m, nE, nst);                     \
  } break;
  switch (cpl) {
    GT(1) GT(2) GT(3) GT(4) GT(5) GT(6) GT(7) GT(8) GT(9) GT(10)     // m <= 320 (3D: 5 * 4^3)
    default: return cudaErrorInvalidValue;
  }
#undef GT
  hbpdc_count_launch();
  return cudaGetLastError();
}

cudaError_t launch_block_gemv_multi(const double* S, int nr, const double* const* in, double* const* out, int m,
                                    int nE, cudaStream_t st) {
  if (nE <= 0) return cudaSuccess;
  if (nr < 1 || nr > GEMV_MAX_RHS || (m * sizeof(double)) % 16 != 0) return cudaErrorInvalidValue;
  GemvRHS io{};
  for (int k = 0; k < nr; ++k) { io.in[k] = in[k]; io.out[k] = out[k]; }
#ifndef GEMV_USE_DMMA
#define GEMV_USE_DMMA 1
#endif
  if (GEMV_USE_DMMA && m <= 320) {
    switch (nr) {
      case 1: return launch_gemv_dmma<1>(S, io, m, nE, st);     // BJ^H_ext: one RHS per system
      case 2: return launch_gemv_dmma<2>(S, io, m, nE, st);
      case 3: return launch_gemv_dmma<3>(S, io, m, nE, st);
      case 4: return launch_gemv_dmma<4>(S, io, m, nE, st);
      case 6: return launch_gemv_dmma<6>(S, io, m, nE, st);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (nr) {
    case 2: return launch_gemvN<2>(S, io, m, nE, st);
    case 4: return launch_gemvN<4>(S, io, m, nE, st);
    case 6: return launch_gemvN<6>(S, io, m, nE, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_block_gemv2(const double* S, int shared, const double* W, const double* sig, double* U,
                               double* V, int m, int nE, cudaStream_t st) {
  if (nE <= 0) return cudaSuccess;
  const int cpl = (m + 31) / 32;
  if (!shared && (m * sizeof(double)) % 16 == 0) {
    const double* in[2] = {W, sig};
    double* out[2] = {U, V};
    return launch_block_gemv_multi(S, 2, in, out, m, nE, st);
  }
#define G(C) case C: gemv2_kernel<C><<<nE, 256, 0, st>>>(S, shared, W, sig, U, V, m, nE); break;
  switch (cpl) {
    G(1) G(2) G(3) G(4) G(5) G(6) G(7) G(8) G(9) G(10)
    default: return cudaErrorInvalidValue;
  }
#undef G
  hbpdc_count_launch();
  return cudaGetLastError();
}

// ============================================================================
// Vector kernels (deterministic two-level reductions: RED_BLOCKS x RED_THREADS)
// ============================================================================
__device__ __forceinline__ double block_sum(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0) {
    for (int w = 0; w < RED_THREADS / 32; ++w) s += sh[w];
  }
  __syncthreads();
  return s;   // valid in thread 0
}

// ---- Arnoldi multi-dot: h_k = V_k . w for k < nk, plus w . w (k = nk) -------------
// Each CTA owns a chunk of 256 x DOT_T elements of w in registers (w is read
// once), streams V_k over that chunk for every k, and reduces DOT_KB dot
// products at a time (warp butterfly + one shared-memory pass).  Partials
// go to part[k * gridDim.x + block]; launch_reduce_partials_n finishes them.
constexpr int DOT_T = 4;    // doubles per thread per vector (measured best on B200: 6.5 TB/s at nk >= 32)
constexpr int DOT_KB = 8;

__global__ void __launch_bounds__(256) arnoldi_dots_kernel(const double* __restrict__ V, size_t ldx, int nk,
                                                           const double* __restrict__ w, size_t L,
                                                           double* __restrict__ part) {
  __shared__ double red[8][DOT_KB];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const size_t base = (size_t)blockIdx.x * (256 * DOT_T) + threadIdx.x;
  double wr[DOT_T];
#pragma unroll
  for (int t = 0; t < DOT_T; ++t) {
    const size_t i = base + (size_t)t * 256;
    wr[t] = i < L ? w[i] : 0.0;
  }
  for (int k0 = 0; k0 <= nk; k0 += DOT_KB) {
    double acc[DOT_KB];
#pragma unroll
    for (int q = 0; q < DOT_KB; ++q) {
      const int k = k0 + q;
      double a = 0.0;
      if (k < nk) {
        const double* vk = V + (size_t)k * ldx;
#pragma unroll
        for (int t = 0; t < DOT_T; ++t) {
          const size_t i = base + (size_t)t * 256;
          if (i < L) a = fma(__ldg(vk + i), wr[t], a);
        }
      } else if (k == nk) {
#pragma unroll
        for (int t = 0; t < DOT_T; ++t) a = fma(wr[t], wr[t], a);
      }
      acc[q] = a;
    }
#pragma unroll
    for (int q = 0; q < DOT_KB; ++q)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], o);
    if (lane == 0)
#pragma unroll
      for (int q = 0; q < DOT_KB; ++q) red[wid][q] = acc[q];
    __syncthreads();
    if (threadIdx.x < DOT_KB && k0 + (int)threadIdx.x <= nk) {
      double s = 0.0;
#pragma unroll
      for (int ww = 0; ww < 8; ++ww) s += red[ww][threadIdx.x];
      part[(size_t)(k0 + threadIdx.x) * gridDim.x + blockIdx.x] = s;
    }
    __syncthreads();
  }
}

int arnoldi_dot_blocks(size_t L) { return (int)((L + 256 * DOT_T - 1) / (256 * DOT_T)); }

// ---- DCGS2 (delayed reorthogonalisation) reduction: one pass over Q_0..Q_{nk-1}
// with two right-hand sides u, w (w may be NULL):
//   rows 2k, 2k+1: Q_k.u, Q_k.w  (k < nk);  rows 2nk, 2nk+1, 2nk+2: u.u, u.w, w.w
__global__ void __launch_bounds__(256) dcgs2_dots_kernel(const double* __restrict__ Q, size_t ldx, int nk,
                                                         const double* __restrict__ u,
                                                         const double* __restrict__ w, size_t L,
                                                         double* __restrict__ part) {
  constexpr int KB = 8;                    // basis vectors per reduction round (2 KB results)
  __shared__ double red[8][2 * KB];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const size_t base = (size_t)blockIdx.x * (256 * DOT_T) + threadIdx.x;
  double ur[DOT_T], wr[DOT_T];
#pragma unroll
  for (int t = 0; t < DOT_T; ++t) {
    const size_t i = base + (size_t)t * 256;
    ur[t] = i < L ? u[i] : 0.0;
    wr[t] = (w && i < L) ? w[i] : 0.0;
  }
  const int nrows = 2 * nk + 3;
  const bool full = (size_t)blockIdx.x * (256 * DOT_T) + 256 * DOT_T <= L;
  for (int k0 = 0; k0 < nk + 2; k0 += KB) {
    double acc[2 * KB];
    if (full && k0 + KB <= nk) {
      // full round: all KB x DOT_T loads in flight before the FMAs (streaming, evict-first)
      double x[KB][DOT_T];
#pragma unroll
      for (int q = 0; q < KB; ++q)
#pragma unroll
        for (int t = 0; t < DOT_T; ++t) x[q][t] = __ldcs(Q + (size_t)(k0 + q) * ldx + base + (size_t)t * 256);
#pragma unroll
      for (int q = 0; q < KB; ++q) {
        double a = 0.0, b = 0.0;
#pragma unroll
        for (int t = 0; t < DOT_T; ++t) { a = fma(x[q][t], ur[t], a); b = fma(x[q][t], wr[t], b); }
        acc[2 * q] = a;
        acc[2 * q + 1] = b;
      }
    } else {
#pragma unroll
    for (int q = 0; q < KB; ++q) {
      const int k = k0 + q;
      double a = 0.0, b = 0.0;
      if (k < nk) {
        const double* qk = Q + (size_t)k * ldx;
#pragma unroll
        for (int t = 0; t < DOT_T; ++t) {
          const size_t i = base + (size_t)t * 256;
          if (i < L) {
            const double x = __ldg(qk + i);
            a = fma(x, ur[t], a);
            b = fma(x, wr[t], b);
          }
        }
      } else if (k == nk) {              // u.u, u.w
#pragma unroll
        for (int t = 0; t < DOT_T; ++t) { a = fma(ur[t], ur[t], a); b = fma(ur[t], wr[t], b); }
      } else if (k == nk + 1) {          // w.w
#pragma unroll
        for (int t = 0; t < DOT_T; ++t) a = fma(wr[t], wr[t], a);
      }
      acc[2 * q] = a;
      acc[2 * q + 1] = b;
    }
    }
    // transpose reduction: 16 values over 32 lanes in 16 shuffles; afterwards
    // lanes with bit 0 clear hold value (lane >> 1) & 15 summed over the warp
#pragma unroll
    for (int s = 8; s >= 1; s >>= 1) {
      const bool hi = lane & (2 * s);
#pragma unroll
      for (int q = 0; q < s; ++q) {
        const double send = hi ? acc[q] : acc[q + s];
        const double recv = __shfl_xor_sync(0xffffffffu, send, 2 * s);
        acc[q] = (hi ? acc[q + s] : acc[q]) + recv;
      }
    }
    acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], 1);
    if ((lane & 1) == 0) {
      // index bits: lane bit 4 -> 8, bit 3 -> 4, bit 2 -> 2, bit 1 -> 1
      const int idx = ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 + ((lane >> 1) & 1);
      red[wid][idx] = acc[0];
    }
    __syncthreads();
    if (threadIdx.x < 2 * KB) {
      const int row = 2 * k0 + threadIdx.x;   // rows 2k, 2k+1 for k = k0 + threadIdx.x/2
      if (row < nrows) {
        double s = 0.0;
#pragma unroll
        for (int ww = 0; ww < 8; ++ww) s += red[ww][threadIdx.x];
        part[(size_t)row * gridDim.x + blockIdx.x] = s;
      }
    }
    __syncthreads();
  }
}

cudaError_t launch_dcgs2_dots(const double* Q, size_t ldx, int nk, const double* u, const double* w, size_t L,
                              double* part, cudaStream_t st) {
  dcgs2_dots_kernel<<<arnoldi_dot_blocks(L), 256, 0, st>>>(Q, ldx, nk, u, w, L, part);
  hbpdc_count_launch();
  return cudaGetLastError();
}

// ---- DCGS2 update: one pass over Q_0..Q_{nk-1} producing
//   q_j     = (u - sum a_k Q_k) * ib                 (written over u)
//   u_{j+1} =  w * ib - sum d_k Q_k - u * cb         (written over w)
__global__ void __launch_bounds__(256) dcgs2_update_kernel(const double* __restrict__ Q, size_t ldx, int nk,
                                                           const double* __restrict__ a,
                                                           const double* __restrict__ d, double* __restrict__ u,
                                                           double* __restrict__ w, double ib, double cb, size_t L) {
  __shared__ double as[1024], ds[1024];
  for (int k = threadIdx.x; k < nk && k < 1024; k += 256) { as[k] = a[k]; ds[k] = d[k]; }
  __syncthreads();
  const size_t base = (size_t)blockIdx.x * (256 * DOT_T) + threadIdx.x;
  double qa[DOT_T], qd[DOT_T];
#pragma unroll
  for (int t = 0; t < DOT_T; ++t) { qa[t] = 0.0; qd[t] = 0.0; }
  const bool full = (size_t)blockIdx.x * (256 * DOT_T) + 256 * DOT_T <= L;
  int k = 0;
  if (full) {
    constexpr int U = 8;                       // basis vectors per batch of hoisted loads
    for (; k + U <= nk; k += U) {
      double x[U][DOT_T];
#pragma unroll
      for (int q = 0; q < U; ++q)
#pragma unroll
        for (int t = 0; t < DOT_T; ++t) x[q][t] = __ldcs(Q + (size_t)(k + q) * ldx + base + (size_t)t * 256);
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const double ak = (k + q) < 1024 ? as[k + q] : a[k + q];
        const double dk = (k + q) < 1024 ? ds[k + q] : d[k + q];
#pragma unroll
        for (int t = 0; t < DOT_T; ++t) { qa[t] = fma(ak, x[q][t], qa[t]); qd[t] = fma(dk, x[q][t], qd[t]); }
      }
    }
  }
  for (; k < nk; ++k) {
    const double ak = k < 1024 ? as[k] : a[k];
    const double dk = k < 1024 ? ds[k] : d[k];
    const double* qk = Q + (size_t)k * ldx;
#pragma unroll
    for (int t = 0; t < DOT_T; ++t) {
      const size_t i = base + (size_t)t * 256;
      if (i < L) {
        const double x = __ldg(qk + i);
        qa[t] = fma(ak, x, qa[t]);
        qd[t] = fma(dk, x, qd[t]);
      }
    }
  }
#pragma unroll
  for (int t = 0; t < DOT_T; ++t) {
    const size_t i = base + (size_t)t * 256;
    if (i < L) {
      const double ui = u[i], wi = w[i];
      u[i] = (ui - qa[t]) * ib;
      w[i] = fma(wi, ib, -qd[t]) - ui * cb;
    }
  }
}

cudaError_t launch_dcgs2_update(const double* Q, size_t ldx, int nk, const double* a, const double* d, double* u,
                                double* w, double ib, double cb, size_t L, cudaStream_t st) {
  dcgs2_update_kernel<<<arnoldi_dot_blocks(L), 256, 0, st>>>(Q, ldx, nk, a, d, u, w, ib, cb, L);
  hbpdc_count_launch();
  return cudaGetLastError();
}

cudaError_t launch_arnoldi_dots(const double* V, size_t ldx, int nk, const double* w, size_t L, double* part,
                                cudaStream_t st) {
  arnoldi_dots_kernel<<<arnoldi_dot_blocks(L), 256, 0, st>>>(V, ldx, nk, w, L, part);
  hbpdc_count_launch();
  return cudaGetLastError();
}

// out[k] = sum_b part[k * nb + b], k < nk (deterministic order)
__global__ void reduce_partials_n_kernel(const double* __restrict__ part, int nb, double* out) {
  __shared__ double sh[8];
  const int k = blockIdx.x;
  double v = 0.0;
  for (int b = threadIdx.x; b < nb; b += 256) v += part[(size_t)k * nb + b];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int q = 0; q < 8; ++q) s += sh[q];
    out[k] = s;
  }
}

cudaError_t launch_reduce_partials_n(const double* part, int nk, int nb, double* out, cudaStream_t st) {
  if (nk <= 0) return cudaSuccess;
  reduce_partials_n_kernel<<<nk, 256, 0, st>>>(part, nb, out);
  hbpdc_count_launch();
  return cudaGetLastError();
}

// ---- Arnoldi update: w -= sum_k h_k V_k, and partial sums of the new w . w ---------
__global__ void __launch_bounds__(256) arnoldi_axpy_kernel(const double* __restrict__ V, size_t ldx, int nk,
                                                           const double* __restrict__ h, double* __restrict__ w,
                                                           size_t L, double* __restrict__ sq) {
  __shared__ double hs[1024];
  __shared__ double red[8];
  for (int k = threadIdx.x; k < nk && k < 1024; k += 256) hs[k] = h[k];
  __syncthreads();
  const size_t base = (size_t)blockIdx.x * (256 * DOT_T) + threadIdx.x;
  double acc[DOT_T];
#pragma unroll
  for (int t = 0; t < DOT_T; ++t) {
    const size_t i = base + (size_t)t * 256;
    acc[t] = i < L ? w[i] : 0.0;
  }
  for (int k = 0; k < nk; ++k) {
    const double hk = k < 1024 ? hs[k] : h[k];
    const double* vk = V + (size_t)k * ldx;
#pragma unroll
    for (int t = 0; t < DOT_T; ++t) {
      const size_t i = base + (size_t)t * 256;
      if (i < L) acc[t] = fma(-hk, __ldg(vk + i), acc[t]);
    }
  }
  double ss = 0.0;
#pragma unroll
  for (int t = 0; t < DOT_T; ++t) {
    const size_t i = base + (size_t)t * 256;
    if (i < L) { w[i] = acc[t]; ss = fma(acc[t], acc[t], ss); }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int q = 0; q < 8; ++q) s += red[q];
    sq[blockIdx.x] = s;
  }
}

cudaError_t launch_arnoldi_axpy(const double* V, size_t ldx, int nk, const double* h, double* w, size_t L,
                                double* sq_part, cudaStream_t st) {
  arnoldi_axpy_kernel<<<arnoldi_dot_blocks(L), 256, 0, st>>>(V, ldx, nk, h, w, L, sq_part);
  hbpdc_count_launch();
  return cudaGetLastError();
}

// out = sqrt(sum part[0..nb))  (and c / that, if c_fd > 0, into out_fd)
__global__ void finish_sqrt_kernel(const double* __restrict__ part, int nb, double* out) {
  __shared__ double sh[8];
  double v = 0.0;
  for (int b = threadIdx.x; b < nb; b += 256) v += part[b];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int q = 0; q < 8; ++q) s += sh[q];
    *out = sqrt(s);
  }
}

cudaError_t launch_finish_sqrt(const double* part, int nb, double* out, cudaStream_t st) {
  finish_sqrt_kernel<<<1, 256, 0, st>>>(part, nb, out);
  hbpdc_count_launch();
  return cudaGetLastError();
}

// partial[k][b] for k in [k0, k0 + KB)
template <int KB>
__global__ void __launch_bounds__(RED_THREADS) multidot_kernel(const double* __restrict__ X, size_t ldx, int k0,
                                                               int nk, const double* __restrict__ y, size_t L,
                                                               double* __restrict__ partial) {
  __shared__ double sh[RED_THREADS / 32];
  double acc[KB];
#pragma unroll
  for (int q = 0; q < KB; ++q) acc[q] = 0.0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < L; i += stride) {
    const double yi = y[i];
#pragma unroll
    for (int q = 0; q < KB; ++q)
      if (k0 + q < nk) acc[q] = fma(X[(size_t)(k0 + q) * ldx + i], yi, acc[q]);
  }
#pragma unroll
  for (int q = 0; q < KB; ++q) {
    if (k0 + q >= nk) break;
    const double s = block_sum(acc[q], sh);
    if (threadIdx.x == 0) partial[(size_t)(k0 + q) * RED_BLOCKS + blockIdx.x] = s;
  }
}

cudaError_t launch_multidot(const double* X, size_t ldx, int nk, const double* y, size_t L, double* partial,
                            cudaStream_t st) {
  for (int k0 = 0; k0 < nk; k0 += 8) {
    multidot_kernel<8><<<RED_BLOCKS, RED_THREADS, 0, st>>>(X, ldx, k0, nk, y, L, partial);
    if (k0 > 0) hbpdc_count_launch();
  }
  hbpdc_count_launch();
  return cudaGetLastError();
}

__global__ void reduce_partials_kernel(const double* __restrict__ partial, int nk, double* out, int accumulate) {
  __shared__ double sh[RED_THREADS / 32];
  const int k = blockIdx.x;
  double v = 0.0;
  for (int b = threadIdx.x; b < RED_BLOCKS; b += RED_THREADS) v += partial[(size_t)k * RED_BLOCKS + b];
  const double s = block_sum(v, sh);
  if (threadIdx.x == 0) out[k] = accumulate ? out[k] + s : s;
}

cudaError_t launch_reduce_partials(const double* partial, int nk, double* out, int accumulate, cudaStream_t st) {
  if (nk <= 0) return cudaSuccess;
  reduce_partials_kernel<<<nk, RED_THREADS, 0, st>>>(partial, nk, out, accumulate);
  hbpdc_count_launch();
  return cudaGetLastError();
}

// y -= sum_k h[k] X_k, optionally with partial sums of y^2
__global__ void __launch_bounds__(RED_THREADS) multiaxpy_kernel(const double* __restrict__ X, size_t ldx, int nk,
                                                                const double* __restrict__ h, double* __restrict__ y,
                                                                size_t L, double* __restrict__ sq) {
  __shared__ double sh[RED_THREADS / 32];
  __shared__ double hs[1024];
  for (int k = threadIdx.x; k < nk && k < 1024; k += blockDim.x) hs[k] = h[k];
  __syncthreads();
  double ss = 0.0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < L; i += stride) {
    double v = y[i];
    for (int k = 0; k < nk; ++k) v = fma(-(k < 1024 ? hs[k] : h[k]), X[(size_t)k * ldx + i], v);
    y[i] = v;
    ss = fma(v, v, ss);
  }
  if (sq) {
    const double s = block_sum(ss, sh);
    if (threadIdx.x == 0) sq[blockIdx.x] = s;
  }
}

cudaError_t launch_multiaxpy(const double* X, size_t ldx, int nk, const double* h, double* y, size_t L,
                             double* sq_partial, cudaStream_t st) {
  multiaxpy_kernel<<<RED_BLOCKS, RED_THREADS, 0, st>>>(X, ldx, nk, h, y, L, sq_partial);
  hbpdc_count_launch();
  return cudaGetLastError();
}

__global__ void lincomb_kernel(const double* __restrict__ X, size_t ldx, int nk, const double* __restrict__ c,
                               double* __restrict__ y, size_t L) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < L; i += stride) {
    double v = 0.0;
    for (int k = 0; k < nk; ++k) v = fma(c[k], X[(size_t)k * ldx + i], v);
    y[i] = v;
  }
}

cudaError_t launch_lincomb(const double* X, size_t ldx, int nk, const double* c, double* y, size_t L,
                           cudaStream_t st) {
  lincomb_kernel<<<RED_BLOCKS, RED_THREADS, 0, st>>>(X, ldx, nk, c, y, L);
  hbpdc_count_launch();
  return cudaGetLastError();
}

__global__ void scale_inv_kernel(const double* __restrict__ x, const double* __restrict__ nrm, double* __restrict__ y,
                                 size_t L) {
  const double n = *nrm;
  const double s = n > 0.0 ? 1.0 / n : 0.0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < L; i += stride) y[i] = x[i] * s;
}

cudaError_t launch_scale_by_inv(const double* x, const double* nrm, double* y, size_t L, cudaStream_t st) {
  scale_inv_kernel<<<RED_BLOCKS, RED_THREADS, 0, st>>>(x, nrm, y, L);
  hbpdc_count_launch();
  return cudaGetLastError();
}

__global__ void axpby_kernel(double a, const double* __restrict__ x, double b, double* __restrict__ y, size_t L) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < L; i += stride) y[i] = a * x[i] + b * y[i];
}

cudaError_t launch_axpby(double a, const double* x, double b, double* y, size_t L, cudaStream_t st) {
  axpby_kernel<<<RED_BLOCKS, RED_THREADS, 0, st>>>(a, x, b, y, L);
  hbpdc_count_launch();
  return cudaGetLastError();
}

__global__ void waxpby_kernel(double a, const double* __restrict__ x, double b, const double* __restrict__ z,
                              double* __restrict__ y, size_t L) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < L; i += stride) y[i] = a * x[i] + b * z[i];
}

// y = a x + b y (z aliases y: same expression as waxpby_kernel, without the restrict on z / y)
__global__ void waxpby_ip_kernel(double a, const double* __restrict__ x, double b, double* y, size_t L) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < L; i += stride) y[i] = a * x[i] + b * y[i];
}

cudaError_t launch_waxpby(double a, const double* x, double b, const double* z, double* y, size_t L,
                          cudaStream_t st) {
  if (z == y) {
    waxpby_ip_kernel<<<RED_BLOCKS, RED_THREADS, 0, st>>>(a, x, b, y, L);
    hbpdc_count_launch();
    return cudaGetLastError();
  }
  waxpby_kernel<<<RED_BLOCKS, RED_THREADS, 0, st>>>(a, x, b, z, y, L);
  hbpdc_count_launch();
  return cudaGetLastError();
}

__global__ void __launch_bounds__(RED_THREADS) sumsq_kernel(const double* __restrict__ x, size_t L,
                                                            double* __restrict__ partial) {
  __shared__ double sh[RED_THREADS / 32];
  double ss = 0.0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < L; i += stride) ss = fma(x[i], x[i], ss);
  const double s = block_sum(ss, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

cudaError_t launch_sumsq(const double* x, size_t L, double* partial, cudaStream_t st) {
  sumsq_kernel<<<RED_BLOCKS, RED_THREADS, 0, st>>>(x, L, partial);
  hbpdc_count_launch();
  return cudaGetLastError();
}

__global__ void finish_norm_kernel(const double* __restrict__ partial, double* out) {
  __shared__ double sh[RED_THREADS / 32];
  double v = 0.0;
  for (int b = threadIdx.x; b < RED_BLOCKS; b += RED_THREADS) v += partial[b];
  const double s = block_sum(v, sh);
  if (threadIdx.x == 0) *out = sqrt(s);
}

cudaError_t launch_finish_norm(const double* partial, double* out, cudaStream_t st) {
  finish_norm_kernel<<<1, RED_THREADS, 0, st>>>(partial, out);
  hbpdc_count_launch();
  return cudaGetLastError();
}

// eps_FD = c / ||x||_2 with c = sqrt(eps_machine)/eps; 0 if ||x|| = 0
__global__ void finish_fd_eps_kernel(const double* __restrict__ partial, int np, double c, double* out) {
  __shared__ double sh[RED_THREADS / 32];
  double v = 0.0;
  for (int b = threadIdx.x; b < np; b += RED_THREADS) v += partial[b];
  const double s = block_sum(v, sh);
  if (threadIdx.x == 0) *out = s > 0.0 ? c / sqrt(s) : 0.0;
}

cudaError_t launch_finish_fd_eps(const double* partial, double c, double* out, cudaStream_t st, int np) {
  finish_fd_eps_kernel<<<1, RED_THREADS, 0, st>>>(partial, np > 0 ? np : RED_BLOCKS, c, out);
  hbpdc_count_launch();
  return cudaGetLastError();
}

// order-independent 64-bit fingerprint of x: sum_i bits(x_i) * (2 i + 1) mod 2^64
// (integer addition is associative: deterministic for any launch shape)
__global__ void fingerprint_kernel(const double* __restrict__ x, size_t L, unsigned long long* out) {
  unsigned long long h = 0ull;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < L; i += stride)
    h += (unsigned long long)__double_as_longlong(x[i]) * (2ull * i + 1ull);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, h);
}

cudaError_t launch_fingerprint(const double* x, size_t L, unsigned long long* out, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(unsigned long long), st);
  if (e != cudaSuccess) return e;
  fingerprint_kernel<<<RED_BLOCKS, RED_THREADS, 0, st>>>(x, L, out);
  hbpdc_count_launch();
  return cudaGetLastError();
}

// admissibility of an Euler / NS state (negative pressure is an error):
// flag[0] = smallest inadmissible node index e * nodes + k (0x7f7f7f7f if none),
// flag[1] |= 1 for a non-finite value, 2 for rho <= 0 or p <= 0
__global__ void admissible_kernel(const double* __restrict__ W, int nE, int nodes, int nv, double gm1, double eps2,
                                  int* flag) {
  const int stride = gridDim.x * blockDim.x;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nE * nodes; t += stride) {
    const int e = t / nodes, k = t % nodes;
    const double* w = W + (size_t)e * nv * nodes + k;
    const double rho = w[0], E = w[(size_t)(nv - 1) * nodes];
    bool fin = isfinite(rho) && isfinite(E);
    double ke = 0.0;
    for (int v = 1; v < nv - 1; ++v) {          // 2 (2D) or 3 (3D) momentum components
      const double mv = w[(size_t)v * nodes];
      fin = fin && isfinite(mv);
      ke = fma(mv, mv, ke);
    }
    const double p = gm1 * (E - 0.5 * eps2 * ke / rho);
    if (!fin || !(rho > 0.0) || !(p > 0.0)) {
      atomicMin(flag, t);
      atomicOr(flag + 1, fin ? 2 : 1);
    }
  }
}

cudaError_t launch_admissible(const double* W, int nE, int nodes, int nv, double gamma, double eps2, int* flag,
                              cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(flag, 0x7f, sizeof(int), st);      // 0x7f7f7f7f: no bad node
  if (e == cudaSuccess) e = cudaMemsetAsync(flag + 1, 0, sizeof(int), st);
  if (e != cudaSuccess) return e;
  admissible_kernel<<<RED_BLOCKS, RED_THREADS, 0, st>>>(W, nE, nodes, nv, gamma - 1.0, eps2, flag);
  hbpdc_count_launch();
  return cudaGetLastError();
}

struct ComboArgs {
  const double* base;
  const double* X[8];
  const double* Y[8];
  double a[8], b[8];
  int nx, ny;
};

__global__ void stage_combo_kernel(ComboArgs A, double* __restrict__ y, size_t L) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < L; i += stride) {
    double v = A.base ? A.base[i] : 0.0;
    for (int k = 0; k < A.nx; ++k) v = fma(A.a[k], A.X[k][i], v);
    for (int k = 0; k < A.ny; ++k) v = fma(A.b[k], A.Y[k][i], v);
    y[i] = v;
  }
}

cudaError_t launch_stage_combo(const double* base, int nx, const double* const* X, const double* a, int ny,
                               const double* const* Y, const double* b, double* y, size_t L, cudaStream_t st) {
  if (nx > 8 || ny > 8) return cudaErrorInvalidValue;
  ComboArgs A{};
  A.base = base;
  A.nx = nx;
  A.ny = ny;
  for (int k = 0; k < nx; ++k) { A.X[k] = X[k]; A.a[k] = a[k]; }
  for (int k = 0; k < ny; ++k) { A.Y[k] = Y[k]; A.b[k] = b[k]; }
  stage_combo_kernel<<<RED_BLOCKS, RED_THREADS, 0, st>>>(A, y, L);
  hbpdc_count_launch();
  return cudaGetLastError();
}
