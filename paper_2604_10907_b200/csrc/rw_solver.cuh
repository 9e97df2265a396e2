// rw_solver.cuh — the B200-native per-setup solver (device code).
//
// One CTA owns one retained setup at a time and runs the whole reference state machine
// for it on device — optimize_beta (routing_opt.cpp:138-173) -> optimize_fractions
// (:70-136) -> solve_dual (score_dual.cpp:232-327) -> eval_dual passes (:25-49), polish
// (:54-76), repair (:81-185) — with no host round trip.  A persistent grid pulls setups
// from an atomic queue (setup_search.cpp:213-236's thread pool, on 148 SMs).
//
// Bit-exactness: eval_dual accumulates sum += best_j left to right in FP64.
// A tile's b_j values are reduced in parallel with *binade quanta*: while the running sum
// S stays inside one binade [2^e, 2^(e+1)) every add lands on the grid u = 2^(e-52), so
// S_{j+1} = S_j + u*q_j with q_j = round(b_j/u) — an integer that does not depend on S_j
// except at exact half-ulp ties, where RNE picks the even neighbour (a function of S_j's
// last mantissa bit only).  A chunk of consecutive elements therefore maps S to
// S + u*Q_p with p = parity(S/u): two int64 numbers (Q0, Q1) per chunk, composable
// associatively (warp tree).  Which binade S is in is decided from an approximate prefix
// sum with a rigorous error margin; elements near a binade crossing (or S <= tiny) are
// replayed with true IEEE adds by the walker thread.  Result: the exact bits of the
// reference's sequential sum.
#pragma once

#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include "rw_job.h"

namespace rw {

constexpr unsigned FULL = 0xffffffffu;

// ---------------------------------------------------------------------------------------
// scalar helpers mirroring libstdc++ semantics
__device__ __forceinline__ double smax(double a, double b) { return (a < b) ? b : a; }  // std::max

// Order-preserving 64-bit key of a double; -0.0 canonicalised to +0.0 so equal values
// (as `>` sees them, score_dual.cpp:71) get equal keys.
__device__ __forceinline__ unsigned long long dkey(double x) {
  if (x == 0.0) x = 0.0;
  unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double dkey_inv(unsigned long long k) {
  unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)b);
}

// S -> S + u*Q_p for S in the binade the quanta were computed for (p = mantissa LSB).
__device__ __forceinline__ double apply_quanta(double S, long long q0, long long q1) {
  long long bits = __double_as_longlong(S);
  long long q = (bits & 1) ? q1 : q0;
  bits = (bits >= 0) ? bits + q : bits - q;
  return __longlong_as_double(bits);
}

// Is |P| safely (margin E) inside one normal binade?  Writes its exponent and sign.
__device__ __forceinline__ bool in_binade(double P, double E, int& e, int& neg) {
  double ap = fabs(P);
  if (!(ap >= 0x1p-900) || !(ap < 0x1p+1000)) return false;
  long long bits = __double_as_longlong(ap);
  int ex = (int)(bits >> 52) - 1023;
  double lo = __longlong_as_double((long long)(ex + 1023) << 52);
  double hi = lo * 2.0;
  e = ex;
  neg = P < 0.0;
  return (ap >= lo + E) && (ap < hi - E);
}

// ---------------------------------------------------------------------------------------
// shared memory
template <int MM, int L, int T>
struct Smem {
  static constexpr int R = L * T;       // rows per tile
  static constexpr int W = T / 32;      // warps
  static constexpr int BPAD = L * T + (L * T) / 8 + 1;
  double b[BPAD];                       // tile's b_j at k + k/8 (conflict-free both ways)
  long long q0[T], q1[T];               // pieces: SAFE -> (Q0, Q1); RAW -> (start, count)
  double scan_x[W], scan_y[W];
  unsigned hist[256];
  unsigned char pkind[T];             // piece kind per slot (SAFE / RAW)
  int wcnt[W];                         // pieces per warp
  // reduction scratch
  double red_d[W];
  int red_j[W];
  int red_v[W];
  // pass outputs / carries
  double S, P, A, tileP, tileA;
  int counts[MM];
  // solve_dual state
  double alpha[MM], best_alpha[MM], polished[MM], zero[MM], c[MM], init[MM];
  double alpha_star[MM], resid[MM];
  double best_g, score, dual_bound, gap, max_delta;
  int iterations, converged, flag, status;
  int target[MM], delta[MM];
  double gain[MM * MM];
  int witness[MM * MM];
  // radix select
  unsigned long long sel_prefix;
  int sel_k;
  int cand_n, above_n;
  double pol_delta;
  // optimize_fractions state
  double w[MM], best_w[MM], warm[MM], grad[MM], step[MM], nextw[MM], tmp[MM];
  double best_obj;
  int have_warm;
  double fr_w[MM], fr_score, fr_lat, fr_obj;
  int fr_iters, fr_conv;
  unsigned fr_oor;
  // optimize_beta state
  double lo, hi, eps;
  int b_feasible, b_has, n_trace;
  double beta_star, w_star[MM];
  double bst_w[MM], bst_score, bst_lat, bst_obj;
  int bst_iters, bst_conv;
  unsigned bst_oor;
  double tr_best_lat, tr_best_score;
  // counters
  long long eval_passes, polish_passes, repair_calls;
  long long prof[8];  // cycle counters (debug: Job.prof_out)
  long long cur_item;
};

// ---------------------------------------------------------------------------------------
// latency model (latency.cpp:15-26, 140-204) — executed by one thread
__device__ __forceinline__ long long upper_knot(const Job& jb, int p, double load) {
  long long a = jb.koff[p], lo = a, hi = jb.koff[p + 1];
  while (lo < hi) {  // first knot with load < x
    long long mid = lo + (hi - lo) / 2;
    if (load < __ldg(jb.kx + mid)) hi = mid;
    else lo = mid + 1;
  }
  return lo - a;
}
__device__ __forceinline__ double segment_slope(const Job& jb, int p, long long hi) {
  long long base = jb.koff[p];
  double x1 = __ldg(jb.kx + base + hi - 1), y1 = __ldg(jb.ky + base + hi - 1);
  double x2 = __ldg(jb.kx + base + hi), y2 = __ldg(jb.ky + base + hi);
  return __ddiv_rn(__dsub_rn(y2, y1), __dsub_rn(x2, x1));
}
__device__ inline double latency_at(const Job& jb, int p, double load) {
  long long nk = jb.koff[p + 1] - jb.koff[p];
  long long hi = upper_knot(jb, p, load);
  long long base = jb.koff[p];
  if (hi == 0) return __ldg(jb.ky + base);
  if (hi == nk) hi = nk - 1;
  double x1 = __ldg(jb.kx + base + hi - 1), y1 = __ldg(jb.ky + base + hi - 1);
  return __dadd_rn(y1, __dmul_rn(__dsub_rn(load, x1), segment_slope(jb, p, hi)));
}
__device__ inline double latency_slope(const Job& jb, int p, double load) {
  long long nk = jb.koff[p + 1] - jb.koff[p];
  long long hi = upper_knot(jb, p, load);
  if (hi == 0) return 0.0;
  if (hi == nk) hi = nk - 1;
  return segment_slope(jb, p, hi);
}
// system_latency_eval (latency.cpp:443-461): returns latency, sets oor mask.
__device__ inline double system_latency(const Job& jb, const int32_t* pidx, int m, const double* w,
                                 double lambda, double kappa, unsigned* oor, double* loads,
                                 double* lats) {
  double total = 0.0;
  unsigned mask = 0;
  for (int i = 0; i < m; ++i) {
    int p = pidx[i];
    double load = __dmul_rn(lambda, w[i]);
    double lat = latency_at(jb, p, load);
    double max_load = __ldg(jb.kx + jb.koff[p + 1] - 1);
    if (load > __dmul_rn(kappa, max_load)) mask |= 1u << i;
    if (loads) loads[i] = load;
    if (lats) lats[i] = lat;
    if (w[i] != 0.0) total = __dadd_rn(total, __dmul_rn(w[i], lat));
  }
  if (oor) *oor = mask;
  return total;
}
// system_latency_grad (latency.cpp:429-441)
__device__ inline void system_latency_grad(const Job& jb, const int32_t* pidx, int m, const double* w,
                                    double lambda, double* grad) {
  for (int i = 0; i < m; ++i) {
    double load = __dmul_rn(lambda, w[i]);
    grad[i] = __dadd_rn(latency_at(jb, pidx[i], load),
                        __dmul_rn(load, latency_slope(jb, pidx[i], load)));
  }
}
// project_simplex (routing_opt.cpp:37-68); returns false on non-finite input.
__device__ inline bool project_simplex(int m, const double* v, double* w, double* u) {
  for (int i = 0; i < m; ++i) {
    if (!isfinite(v[i])) return false;
    u[i] = v[i];
  }
  for (int i = 1; i < m; ++i) {  // descending (only the sorted values matter)
    double x = u[i];
    int k = i - 1;
    while (k >= 0 && u[k] < x) {
      u[k + 1] = u[k];
      --k;
    }
    u[k + 1] = x;
  }
  double css = 0.0, theta = 0.0;
  for (int k = 0; k < m; ++k) {
    css = __dadd_rn(css, u[k]);
    double t = __ddiv_rn(__dsub_rn(css, 1.0), (double)(k + 1));
    if (u[k] > t) theta = t;
  }
  double sum = 0.0;
  for (int i = 0; i < m; ++i) {
    w[i] = smax(__dsub_rn(v[i], theta), 0.0);
    sum = __dadd_rn(sum, w[i]);
  }
  for (int i = 0; i < m; ++i) w[i] = __ddiv_rn(w[i], sum);
  return true;
}

// ---------------------------------------------------------------------------------------
// The solver: all threads of the CTA execute every member function (uniform control
// flow); scalar state lives in shared memory and is updated by thread 0 between barriers.
enum PassMode { PASS_EVAL = 0, PASS_FIXED = 1 };
enum PieceKind { PIECE_NONE = 0, PIECE_SAFE = 1, PIECE_RAW = 2 };

// Shared memory is always reached through the extern __shared__ symbol so every access
// compiles to LDS/STS (a reference member would decay to generic LD/ST).
template <class SMT>
__device__ __forceinline__ SMT& smem() {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  return *reinterpret_cast<SMT*>(smem_raw);
}
#define SMX (smem<SM>())

template <int MM, int L, int T>
struct Solver {
  using SM = Smem<MM, L, T>;
  static constexpr int R = SM::R;
  static constexpr int W = SM::W;
  static constexpr int NPK = (MM + 3) / 4;  // packed 16-bit count words

  const Job& jb;
  const int n, m;
  const int tid, lane, wid;
  uint8_t* mo;               // this CTA's model_of workspace [n]
  unsigned long long* keys;  // this CTA's radix-select workspace [n]
  const int32_t* pidx;       // current setup's profile indices [m]

  __device__ Solver(const Job& j, uint8_t* mo_, unsigned long long* keys_)
      : jb(j), n(j.n), m(j.m), tid(threadIdx.x), lane(threadIdx.x & 31),
        wid(threadIdx.x >> 5), mo(mo_), keys(keys_), pidx(nullptr) {}

  
  __device__ void fail(int code) {
    if (tid == 0 && SMX.status == 0) SMX.status = code;
  }

  // ---- one pass over the N x M matrix (score_dual.cpp:25-49) ------------------------
  // PASS_EVAL : b_j = max_i (s_ji - alpha_i), arg = first max; counts; optional model_of.
  // PASS_FIXED: b_j = s_j,mo[j] (mo == null -> column 0).
  // Result: SMX.S = the reference's sequential FP64 sum of b_j, bit for bit.
  //
  // Per tile of R = L*T rows:
  //  phase 1 (coalesced, all threads): rows -> b_j into smem, argmax, packed counts.
  //  phase 2 (all threads): thread t owns the contiguous chunk [t*L, t*L+L).  An
  //    approximate block scan of (sum b, sum |b|) locates the binade of the running sum at
  //    both chunk ends; a monotone chunk (all b >= 0 or all <= 0) whose two ends sit in
  //    the same binade with margin E is SAFE and maps S -> S + u*Q_p (integer quanta,
  //    two tracks for half-ulp ties).  Otherwise the chunk is RAW (exact IEEE adds).
  //    A segmented warp scan composes runs of SAFE chunks of one binade into a single
  //    piece, so each warp publishes ~1 piece (a few around binade crossings).
  //  phase 3 (thread 0): apply the pieces in order to the exact running sum S.
  // b_j of tile row k lives at k + k/8: coalesced writes in phase 1 and, for L = 24, the
  // chunk reads of phase 2 (lane t at 27t + r) are bank-conflict free.
  __device__ __forceinline__ static int bpos(int k) { return k + (k >> 3); }

  // quanta of one |b| for u = 2^(base_sh - 1023 - 52): floor and half-way flag (exact, INT)
  __device__ __forceinline__ static long long quanta_floor(double ab, int base_sh, bool& tie,
                                                           bool& above) {
    const unsigned long long B =
        (unsigned long long)__double_as_longlong(ab) & 0x7fffffffffffffffull;
    const int ebits = (int)(B >> 52);
    const unsigned long long Mb =
        (B & 0x000fffffffffffffull) | (ebits ? 0x0010000000000000ull : 0ull);
    const int sh = base_sh - max(ebits, 1);
    tie = false;
    above = false;
    if (sh <= 0) return (long long)(Mb << (-sh));
    if (sh >= 54) return 0;
    const unsigned long long rem = Mb & ((1ull << sh) - 1ull);
    const unsigned long long half = 1ull << (sh - 1);
    tie = (rem == half);
    above = (rem > half);
    return (long long)(Mb >> sh);
  }

  __device__ void pass(int mode, const double* alpha_s, bool want_counts, uint8_t* mo_out,
                       const uint8_t* mo_in) {
    if (mode == PASS_EVAL) {
      if (m == MM) {
        if (mo_out) pass_t<PASS_EVAL, true, true>(n, alpha_s, want_counts, mo_out, mo_in);
        else pass_t<PASS_EVAL, true, false>(n, alpha_s, want_counts, mo_out, mo_in);
      } else {
        if (mo_out) pass_t<PASS_EVAL, false, true>(n, alpha_s, want_counts, mo_out, mo_in);
        else pass_t<PASS_EVAL, false, false>(n, alpha_s, want_counts, mo_out, mo_in);
      }
    } else {
      pass_t<PASS_FIXED, false, false>(n, alpha_s, want_counts, mo_out, mo_in);
    }
  }

  // Rows per load group in phase 1 (all loads of a group are in flight together).
  static constexpr int G = (MM <= 4) ? 8 : ((MM <= 8) ? 4 : 2);
  static_assert(L % G == 0, "L must be a multiple of the load group");

  template <int MODE, bool FULLM, bool WMO>
  __device__ __noinline__ void pass_t(const int n_, const double* alpha_s, const bool want_counts,
                                      uint8_t* mo_out, const uint8_t* mo_in) {
    const int tid_ = threadIdx.x, lane_ = tid_ & 31, wid_ = tid_ >> 5;
    const int m_ = FULLM ? MM : jb.m;
    const double* __restrict__ sc = jb.scores;
    __syncthreads();  // callers may still be reading the previous pass's S / counts
    double a[MM];
#pragma unroll
    for (int i = 0; i < MM; ++i) a[i] = (FULLM || i < m_) ? alpha_s[i] : 0.0;
    if (tid_ == 0) {
      SMX.S = 0.0;
      SMX.P = 0.0;
      SMX.A = 0.0;
      if (MODE == PASS_EVAL) SMX.eval_passes++;
    }
    if (tid_ < MM) SMX.counts[tid_] = 0;
    __syncthreads();
    const bool vec2 = FULLM ? (MM % 2 == 0) : ((m_ & 1) == 0);
    for (int base = 0; base < n_; base += R) {
      const int len = min(R, n_ - base);
      // -- phase 1 ----------------------------------------------------------------------
      long long t_p1 = clock64();
      unsigned long long pk[NPK];
#pragma unroll
      for (int q = 0; q < NPK; ++q) pk[q] = 0ull;
      for (int r0 = 0; r0 < L; r0 += G) {
        if (r0 * T >= len) break;  // block-uniform
        double v[G][MODE == PASS_EVAL ? MM : 1];
        int ag[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const int kk = min((r0 + g) * T + tid_, len - 1);
          const double* row = sc + (size_t)(base + kk) * m_;
          if (MODE == PASS_EVAL) {
            if (vec2) {
              const double2* r2 = reinterpret_cast<const double2*>(row);
#pragma unroll
              for (int i = 0; i < MM / 2; ++i) {
                if (FULLM || 2 * i < m_) {
                  const double2 x = __ldg(r2 + i);
                  v[g][2 * i] = x.x;
                  v[g][2 * i + 1] = x.y;
                } else {
                  v[g][2 * i] = 0.0;
                  v[g][2 * i + 1] = 0.0;
                }
              }
            } else {
#pragma unroll
              for (int i = 0; i < MM; ++i) v[g][i] = (FULLM || i < m_) ? __ldg(row + i) : 0.0;
            }
          } else {
            ag[g] = mo_in ? (int)mo_in[base + kk] : 0;
            v[g][0] = __ldg(row + ag[g]);
          }
        }
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const int k = (r0 + g) * T + tid_;
          double bj;
          int arg;
          if (MODE == PASS_EVAL) {
            bj = __dsub_rn(v[g][0], a[0]);
            arg = 0;
#pragma unroll
            for (int i = 1; i < MM; ++i) {
              if (FULLM || i < m_) {
                const double x = __dsub_rn(v[g][i], a[i]);
                if (x > bj) {
                  bj = x;
                  arg = i;
                }
              }
            }
          } else {
            bj = v[g][0];
            arg = ag[g];
          }
          if (k < len) {
            SMX.b[bpos(k)] = bj;
            if (want_counts) {
              if (NPK == 1) {
                pk[0] += 1ull << (arg * 16);
              } else {
#pragma unroll
                for (int q = 0; q < NPK; ++q)
                  pk[q] += ((arg >> 2) == q) ? (1ull << ((arg & 3) * 16)) : 0ull;
              }
            }
            if (WMO) mo_out[base + k] = (uint8_t)arg;
          }
        }
      }
      if (want_counts) {
#pragma unroll
        for (int q = 0; q < NPK; ++q) {
          unsigned long long x = pk[q];
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) x += __shfl_down_sync(FULL, x, off);
          if (lane_ == 0) {
#pragma unroll
            for (int f = 0; f < 4; ++f) {
              const int i = 4 * q + f;
              const unsigned cnt = (unsigned)((x >> (16 * f)) & 0xffffull);
              if (i < m_ && cnt) atomicAdd(&SMX.counts[i], (int)cnt);
            }
          }
        }
      }
      __syncthreads();
      long long t_p2 = clock64();
      if (tid_ == 0) SMX.prof[0] += t_p2 - t_p1;
      // -- phase 2 ----------------------------------------------------------------------
      static_assert(L % 8 == 0, "chunk addressing assumes L % 8 == 0");
      const int c0 = tid_ * L;
      const int cnt = max(0, min(L, len - c0));
      const double* bch = SMX.b + bpos(c0);
      double bl[L];
      double ps = 0.0;
      unsigned orhi = 0u, andhi = 0xffffffffu;
#pragma unroll
      for (int r = 0; r < L; ++r) {
        bl[r] = 0.0;
        if (r < cnt) {
          bl[r] = bch[r + (r >> 3)];
          ps += bl[r];
          const unsigned hi = (unsigned)__double2hiint(bl[r]);
          orhi |= hi;
          andhi &= hi;
        }
      }
      const bool allpos = (orhi >> 31) == 0u;   // every b has its sign bit clear (incl. +0)
      const bool allneg = (andhi >> 31) != 0u;  // every b has its sign bit set
      double pa;
      if (allpos) pa = ps;
      else if (allneg) pa = -ps;
      else {
        pa = 0.0;
#pragma unroll
        for (int r = 0; r < L; ++r) pa += fabs(bl[r]);
      }
      // block exclusive scan of (ps, pa) — approximate; used only behind a margin
      double ix = ps, iy = pa;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        double tx = __shfl_up_sync(FULL, ix, off), ty = __shfl_up_sync(FULL, iy, off);
        if (lane_ >= off) {
          ix += tx;
          iy += ty;
        }
      }
      if (lane_ == 31) {
        SMX.scan_x[wid_] = ix;
        SMX.scan_y[wid_] = iy;
      }
      __syncthreads();
      if (wid_ == 0) {  // exclusive scan of the W warp totals (+ the tile carry)
        double wx = (lane_ < W) ? SMX.scan_x[lane_] : 0.0;
        double wy = (lane_ < W) ? SMX.scan_y[lane_] : 0.0;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          double tx = __shfl_up_sync(FULL, wx, off), ty = __shfl_up_sync(FULL, wy, off);
          if (lane_ >= off) {
            wx += tx;
            wy += ty;
          }
        }
        const double ox = __shfl_up_sync(FULL, wx, 1), oy = __shfl_up_sync(FULL, wy, 1);
        const double cp = SMX.P, ca = SMX.A;
        if (lane_ < W) {
          SMX.scan_x[lane_] = cp + (lane_ ? ox : 0.0);
          SMX.scan_y[lane_] = ca + (lane_ ? oy : 0.0);
        }
        if (lane_ == W - 1) {
          SMX.tileP = wx;
          SMX.tileA = wy;
        }
      }
      double ex = __shfl_up_sync(FULL, ix, 1), ey = __shfl_up_sync(FULL, iy, 1);
      if (lane_ == 0) {
        ex = 0.0;
        ey = 0.0;
      }
      __syncthreads();
      const double P0 = SMX.scan_x[wid_] + ex;
      const double A0 = SMX.scan_y[wid_] + ey;
      const long long jg = (long long)base + c0;
      int kind = (cnt > 0) ? PIECE_RAW : PIECE_NONE;
      int e_ref = 0, neg_ref = 0;
      if (cnt > 0) {
        if (allpos || allneg) {
          // S_j is monotone across the chunk: both ends in one binade => all inside.
          const double P1 = P0 + ps, A1 = A0 + pa;
          const double E = (double)(jg + cnt + 64) * 0x1p-51 * A1;
          int e1, n1;
          if (in_binade(P0, E, e_ref, neg_ref) && in_binade(P1, E, e1, n1) && e1 == e_ref &&
              n1 == neg_ref)
            kind = PIECE_SAFE;
        } else {
          double P = P0, A = A0;
          bool ok = true;
#pragma unroll
          for (int r = 0; r <= L; ++r) {
            if (r <= cnt && ok) {
              const double x = (r < cnt) ? bl[r] : 0.0;
              const double E = (double)(jg + r + 64) * 0x1p-51 * (A + fabs(x));
              int e, ng;
              if (!in_binade(P, E, e, ng)) ok = false;
              else if (r == 0) {
                e_ref = e;
                neg_ref = ng;
              } else if (e != e_ref || ng != neg_ref) ok = false;
              P += x;
              A += fabs(x);
            }
          }
          if (ok) kind = PIECE_SAFE;
        }
      }
      long long Q0 = 0, Q1 = 0;
      if (kind == PIECE_SAFE) {
        // q_j = round(b_j / u), u = 2^(e-52).  Monotone fast path in FP64: y = |b| * 2^(52-e)
        // is exact and < 2^52 (S and S + b share the binade), so t = y + 2^52 rounds y to
        // the integer grid (RNE) and bits(t) - bits(2^52) is that integer; a half-way
        // y (|t - 2^52 - y| == 1/2) is a tie whose rounding depends on S — slow path.
        bool tie_any = false;
        if (allpos || allneg) {
          const double scale = __longlong_as_double((long long)(52 - e_ref + 1023) << 52);
          unsigned long long acc = 0ull;
#pragma unroll
          for (int r = 0; r < L; ++r) {
            if (r < cnt) {
              const double y = fabs(bl[r]) * scale;
              const double t = y + 0x1p52;
              acc += (unsigned long long)__double_as_longlong(t) - 0x4330000000000000ull;
              tie_any |= (fabs((t - 0x1p52) - y) == 0.5);
            }
          }
          Q0 = allpos ? (long long)acc : -(long long)acc;
          Q1 = Q0;
        }
        if (!(allpos || allneg) || tie_any) {  // general: signed b, two parity tracks
          const int base_sh = 1023 + e_ref;
          Q0 = 0;
          Q1 = 0;
          for (int r = 0; r < cnt; ++r) {
            const double x = bch[r + (r >> 3)];
            bool tie, above;
            const long long q = quanta_floor(x, base_sh, tie, above);
            const bool negb = x < 0.0;
            if (tie) {  // |x|/u = q + 1/2; RNE picks the neighbour leaving S/u even
              const long long lo = negb ? -q - 1 : q;
              Q0 += ((Q0 + lo) & 1) ? lo + 1 : lo;
              Q1 += ((1 + Q1 + lo) & 1) ? lo + 1 : lo;
            } else {
              const long long qq = q + (above ? 1 : 0);
              Q0 += negb ? -qq : qq;
              Q1 += negb ? -qq : qq;
            }
          }
        }
      }
      // segmented warp scan: compose consecutive SAFE chunks of one binade
      const int key = (kind == PIECE_SAFE) ? (e_ref * 2 + neg_ref) : -100000 - lane_;
      const int pkey = __shfl_up_sync(FULL, key, 1);
      const bool head = (lane_ == 0) || kind != PIECE_SAFE || pkey != key;
      {
        bool f = head;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          long long o0 = __shfl_up_sync(FULL, Q0, d), o1 = __shfl_up_sync(FULL, Q1, d);
          bool of = __shfl_up_sync(FULL, f, d);
          if (lane_ >= d && !f) {
            long long n0 = o0 + ((o0 & 1) ? Q1 : Q0);
            long long n1 = o1 + (((1 + o1) & 1) ? Q1 : Q0);
            Q0 = n0;
            Q1 = n1;
            f = of;
          }
        }
      }
      const bool nhead = __shfl_down_sync(FULL, head, 1);
      const bool tail = (kind != PIECE_NONE) && (lane_ == 31 || nhead);
      const unsigned tmask = __ballot_sync(FULL, tail);
      if (tail) {
        const int slot = wid_ * 32 + __popc(tmask & ((1u << lane_) - 1u));
        SMX.pkind[slot] = (unsigned char)kind;
        SMX.q0[slot] = (kind == PIECE_SAFE) ? Q0 : (long long)c0;
        SMX.q1[slot] = (kind == PIECE_SAFE) ? Q1 : (long long)cnt;
      }
      if (lane_ == 0) SMX.wcnt[wid_] = __popc(tmask);
      __syncthreads();
      long long t_p3 = clock64();
      if (tid_ == 0) SMX.prof[1] += t_p3 - t_p2;
      // -- phase 3: ordered walk over the pieces (one thread) ----------------------------
      if (tid_ == 0) {
        double S = SMX.S;
        for (int w = 0; w < W; ++w) {
          const int np = SMX.wcnt[w];
          for (int p = 0; p < np; ++p) {
            const int slot = w * 32 + p;
            const long long x0 = SMX.q0[slot], x1 = SMX.q1[slot];
            if (SMX.pkind[slot] == PIECE_SAFE) {
              S = apply_quanta(S, x0, x1);
            } else {
              const int k0 = (int)x0, rc = (int)x1;
              for (int r = 0; r < rc; ++r) S = __dadd_rn(S, SMX.b[bpos(k0 + r)]);
            }
          }
        }
        SMX.S = S;
        SMX.P += SMX.tileP;
        SMX.A += SMX.tileA;
      }
      __syncthreads();
      if (tid_ == 0) SMX.prof[2] += clock64() - t_p3;
    }
  }

  // g(alpha) = (sum_j best_j + sum_i alpha_i c_i) / N   (score_dual.cpp:47-48)
  __device__ double eval_dual(const double* alpha_s, bool want_counts, uint8_t* mo_out) {
    pass(PASS_EVAL, alpha_s, want_counts, mo_out, nullptr);
    double g = SMX.S;
    for (int i = 0; i < m; ++i) g = __dadd_rn(g, __dmul_rn(alpha_s[i], SMX.c[i]));
    return __ddiv_rn(g, (double)n);  // every thread computes the same value
  }

  // ---- radix select: k-th largest key among keys[0..n) (nth_element, :71-72) ----------
  __device__ __forceinline__ void hist_add(bool ok, unsigned d) {
    unsigned act = __activemask();
    unsigned key = ok ? d : 0xffffffffu;
    unsigned peers = __match_any_sync(act, key);
    if (ok && lane == __ffs(peers) - 1) atomicAdd(&SMX.hist[d], __popc(peers));
  }
  // Picks the digit holding the sel_k-th largest among counted candidates (warp 0).
  __device__ void select_digit(int shift) {
    if (wid == 0) {
      // lane l covers bins [248 - 8l, 255 - 8l], top bins first
      const int top = 255 - 8 * lane;
      int local = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) local += (int)SMX.hist[top - q];
      int incl = local;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        int t = __shfl_up_sync(FULL, incl, off);
        if (lane >= off) incl += t;
      }
      const int excl = incl - local;
      const int k = SMX.sel_k;
      if (excl < k && k <= incl) {
        int above = excl;
        for (int q = 0; q < 8; ++q) {
          int h = (int)SMX.hist[top - q];
          if (above + h >= k) {
            SMX.sel_prefix |= (unsigned long long)(top - q) << shift;
            SMX.sel_k = k - above;
            break;
          }
          above += h;
        }
      }
    }
  }

  // ---- polish_pass (score_dual.cpp:54-76) on SMX.polished --------------------------------
  // For coordinate i the new price is the k-th largest b_j = s_ji - max_{k!=i}(s_jk - a_k),
  // k = ceil(c_i - 1e-9) (nth_element, :69-72).  Near the optimum that value sits close to
  // the current a_i, so one sweep counts the keys above a window [a_i - d, a_i + d] and
  // gathers the keys inside it into shared memory; the k-th largest is then selected among
  // the few candidates (radix select in smem).  If the window misses or overflows, an exact
  // 8-digit radix select over all N keys (written during the same sweep) is the fallback.
  // d adapts per CTA; the result is exact either way.
  __device__ __noinline__ void polish_pass() {
    constexpr int CAP = SM::BPAD;
    const long long t_pol = clock64();
    if (tid == 0) {
      SMX.max_delta = 0.0;
      SMX.polish_passes++;
    }
    unsigned long long* cand = reinterpret_cast<unsigned long long*>(SMX.b);
    for (int i = 0; i < m; ++i) {
      __syncthreads();
      double a[MM];
#pragma unroll
      for (int q = 0; q < MM; ++q) a[q] = (q < m) ? SMX.polished[q] : 0.0;
      const double ci = SMX.c[i];
      int k = ci > 1e-12 ? (int)ceil(__dsub_rn(ci, 1e-9)) : 1;
      k = max(1, min(k, n));
      const double ai = SMX.polished[i], dl = SMX.pol_delta;
      const unsigned long long klo = dkey(ai - dl), khi = dkey(ai + dl);
      if (tid < 256) SMX.hist[tid] = 0u;
      if (tid == 0) {
        SMX.sel_prefix = 0ull;
        SMX.sel_k = k;
        SMX.cand_n = 0;
        SMX.above_n = 0;
      }
      __syncthreads();
      int my_above = 0;
      for (int j = tid; j < n; j += T) {
        const double* row = jb.scores + (size_t)j * m;
        double rest = -CUDART_INF;
        double vi = 0.0;
#pragma unroll
        for (int q = 0; q < MM; ++q) {
          if (q < m) {
            double v = __ldg(row + q);
            if (q == i) vi = v;
            else rest = smax(rest, __dsub_rn(v, a[q]));
          }
        }
        const unsigned long long key = dkey(__dsub_rn(vi, rest));
        keys[j] = key;
        my_above += (key > khi) ? 1 : 0;
        const bool in = (key >= klo) && (key <= khi);
        const unsigned act = __activemask();
        const unsigned inm = __ballot_sync(act, in);
        if (inm) {
          const int leader = __ffs(inm) - 1;
          int basepos = 0;
          if (lane == leader) basepos = atomicAdd(&SMX.cand_n, __popc(inm));
          basepos = __shfl_sync(act, basepos, leader);
          if (in) {
            const int pos = basepos + __popc(inm & ((1u << lane) - 1u));
            if (pos < CAP) cand[pos] = key;
          }
        }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) my_above += __shfl_down_sync(FULL, my_above, off);
      if (lane == 0 && my_above) atomicAdd(&SMX.above_n, my_above);
      __syncthreads();
      const int nc = SMX.cand_n, na = SMX.above_n;
      const bool win = (nc <= CAP) && (na < k) && (k <= na + nc);
      if (win) {
        if (tid == 0) SMX.sel_k = k - na;
        for (int shift = 56; shift >= 0; shift -= 8) {
          __syncthreads();
          if (tid < 256) SMX.hist[tid] = 0u;
          __syncthreads();
          const unsigned long long hi = (shift == 56) ? 0ull : (SMX.sel_prefix >> (shift + 8));
          for (int q = tid; q < nc; q += T) {
            const unsigned long long key = cand[q];
            hist_add(shift == 56 || (key >> (shift + 8)) == hi,
                     (unsigned)((key >> shift) & 0xffull));
          }
          __syncthreads();
          select_digit(shift);
        }
      } else {
        for (int shift = 56; shift >= 0; shift -= 8) {
          __syncthreads();
          if (tid < 256) SMX.hist[tid] = 0u;
          __syncthreads();
          const unsigned long long hi = (shift == 56) ? 0ull : (SMX.sel_prefix >> (shift + 8));
          for (int j = tid; j < n; j += T) {
            const unsigned long long key = keys[j];
            hist_add(shift == 56 || (key >> (shift + 8)) == hi,
                     (unsigned)((key >> shift) & 0xffull));
          }
          __syncthreads();
          select_digit(shift);
        }
      }
      __syncthreads();
      if (tid == 0) {
        const double next = dkey_inv(SMX.sel_prefix);
        SMX.max_delta = smax(SMX.max_delta, fabs(__dsub_rn(next, SMX.polished[i])));
        SMX.polished[i] = next;
        if (nc > CAP) SMX.pol_delta *= 0.125;
        else if (!win) SMX.pol_delta = fmin(SMX.pol_delta * 8.0, 4.0);
        else if (nc > CAP / 4) SMX.pol_delta *= 0.5;
        if (!win) SMX.prof[4]++;
      }
    }
    __syncthreads();
    if (tid == 0) SMX.prof[3] += clock64() - t_pol;
  }

  // ---- block argmin / argmax helpers (lexicographic with index tie-break) ------------
  // returns winner to all threads via smem: (val, j, v)
  __device__ void block_argmin(double& val, int& j, int& v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      double ov = __shfl_down_sync(FULL, val, off);
      int oj = __shfl_down_sync(FULL, j, off), ovv = __shfl_down_sync(FULL, v, off);
      bool take = (oj >= 0) && (j < 0 || ov < val || (ov == val && oj < j));
      if (take) {
        val = ov;
        j = oj;
        v = ovv;
      }
    }
    if (lane == 0) {
      SMX.red_d[wid] = val;
      SMX.red_j[wid] = j;
      SMX.red_v[wid] = v;
    }
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < W; ++w) {
        double ov = SMX.red_d[w];
        int oj = SMX.red_j[w];
        if (oj >= 0 && (SMX.red_j[0] < 0 || ov < SMX.red_d[0] ||
                        (ov == SMX.red_d[0] && oj < SMX.red_j[0]))) {
          SMX.red_d[0] = ov;
          SMX.red_j[0] = oj;
          SMX.red_v[0] = SMX.red_v[w];
        }
      }
    }
    __syncthreads();
    val = SMX.red_d[0];
    j = SMX.red_j[0];
    v = SMX.red_v[0];
    __syncthreads();
  }
  __device__ void block_argmax(double& val, int& j) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      double ov = __shfl_down_sync(FULL, val, off);
      int oj = __shfl_down_sync(FULL, j, off);
      bool take = (oj >= 0) && (j < 0 || ov > val || (ov == val && oj < j));
      if (take) {
        val = ov;
        j = oj;
      }
    }
    if (lane == 0) {
      SMX.red_d[wid] = val;
      SMX.red_j[wid] = j;
    }
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < W; ++w) {
        double ov = SMX.red_d[w];
        int oj = SMX.red_j[w];
        if (oj >= 0 && (SMX.red_j[0] < 0 || ov > SMX.red_d[0] ||
                        (ov == SMX.red_d[0] && oj < SMX.red_j[0]))) {
          SMX.red_d[0] = ov;
          SMX.red_j[0] = oj;
        }
      }
    }
    __syncthreads();
    val = SMX.red_d[0];
    j = SMX.red_j[0];
    __syncthreads();
  }

  // ---- repair_counts (score_dual.cpp:81-185); counts in SMX.counts, targets in SMX.target
  __device__ double repair() {
    if (tid == 0) {
      SMX.repair_calls++;
      for (int i = 0; i < m; ++i) SMX.delta[i] = SMX.counts[i] - SMX.target[i];
    }
    __syncthreads();
    // Phase 1: min-loss single moves while any surplus remains (:96-118)
    for (;;) {
      bool over = false;
      for (int i = 0; i < m; ++i) over = over || SMX.delta[i] > 0;
      if (!over) break;
      double bl = CUDART_INF;
      int bj = -1, bv = -1;
      for (int j = tid; j < n; j += T) {
        int u = mo[j];
        if (SMX.delta[u] <= 0) continue;
        const double* row = jb.scores + (size_t)j * m;
        double su = __ldg(row + u);
        for (int v = 0; v < m; ++v) {
          if (SMX.delta[v] >= 0) continue;
          double loss = __dsub_rn(su, __ldg(row + v));
          if (bj < 0 || loss < bl) {
            bl = loss;
            bj = j;
            bv = v;
          }
        }
      }
      block_argmin(bl, bj, bv);
      if (tid == 0) {
        int u = mo[bj];
        mo[bj] = (uint8_t)bv;
        SMX.counts[u]--;
        SMX.counts[bv]++;
        SMX.delta[u]--;
        SMX.delta[bv]++;
      }
      __syncthreads();
    }
    // Phase 2: profitable 2- and 3-cycles (:120-180)
    if (m >= 2) {
      for (int pass_i = 0; pass_i < 10000; ++pass_i) {
        for (int u = 0; u < m; ++u) {
          double bg[MM];
          int bjv[MM];
#pragma unroll
          for (int v = 0; v < MM; ++v) {
            bg[v] = -CUDART_INF;
            bjv[v] = -1;
          }
          for (int j = tid; j < n; j += T) {
            if (mo[j] != u) continue;
            const double* row = jb.scores + (size_t)j * m;
            double su = __ldg(row + u);
#pragma unroll
            for (int v = 0; v < MM; ++v) {
              if (v < m && v != u) {
                double g = __dsub_rn(__ldg(row + v), su);
                if (bjv[v] < 0 || g > bg[v]) {
                  bg[v] = g;
                  bjv[v] = j;
                }
              }
            }
          }
          for (int v = 0; v < m; ++v) {
            double g = bg[v];
            int j = bjv[v];
            block_argmax(g, j);
            if (tid == 0) {
              SMX.gain[u * m + v] = (j >= 0) ? g : -CUDART_INF;
              SMX.witness[u * m + v] = j;
            }
          }
        }
        __syncthreads();
        if (tid == 0) {
          double best = 1e-15;
          int cu = -1, cv = -1, cw = -1;
          for (int u = 0; u < m; ++u)
            for (int v = u + 1; v < m; ++v) {
              double g = __dadd_rn(SMX.gain[u * m + v], SMX.gain[v * m + u]);
              if (g > best) {
                best = g;
                cu = u;
                cv = v;
                cw = -1;
              }
            }
          for (int u = 0; u < m; ++u)
            for (int v = 0; v < m; ++v) {
              if (v == u) continue;
              for (int w = 0; w < m; ++w) {
                if (w == u || w == v) continue;
                double g = __dadd_rn(__dadd_rn(SMX.gain[u * m + v], SMX.gain[v * m + w]),
                                     SMX.gain[w * m + u]);
                if (g > best) {
                  best = g;
                  cu = u;
                  cv = v;
                  cw = w;
                }
              }
            }
          SMX.flag = (cu < 0);
          if (cu >= 0) {
            auto move = [&](int j, int v) {
              int uu = mo[j];
              mo[j] = (uint8_t)v;
              SMX.counts[uu]--;
              SMX.counts[v]++;
              SMX.delta[uu]--;
              SMX.delta[v]++;
            };
            if (cw < 0) {
              int j1 = SMX.witness[cu * m + cv], j2 = SMX.witness[cv * m + cu];
              move(j1, cv);
              move(j2, cu);
            } else {
              int j1 = SMX.witness[cu * m + cv], j2 = SMX.witness[cv * m + cw],
                  j3 = SMX.witness[cw * m + cu];
              move(j1, cv);
              move(j2, cw);
              move(j3, cu);
            }
          }
        }
        __syncthreads();
        if (SMX.flag) break;
        __syncthreads();
      }
    }
    __syncthreads();
    // exact sequential mean of the repaired assignment (:182-184)
    pass(PASS_FIXED, SMX.zero, false, nullptr, mo);
    return __ddiv_rn(SMX.S, (double)n);
  }

  // ---- solve_dual (score_dual.cpp:232-327) ---------------------------------------------
  // in: SMX.c (targets), SMX.init (when has_init); out: SMX.alpha_star, score, dual_bound, gap,
  // resid, iterations, converged, SMX.counts (realised), mo (assignment)
  __device__ void solve_dual(const rw_subgradient_params& p, bool has_init) {
    if (tid == 0) {  // TargetCounts::validate (:195-205)
      double t = 0.0;
      bool ok = true;
      for (int i = 0; i < m; ++i) {
        if (!isfinite(SMX.c[i]) || SMX.c[i] < -1e-9) ok = false;
        t = __dadd_rn(t, SMX.c[i]);
      }
      double scale = (double)n > 1.0 ? (double)n : 1.0;
      if (!(fabs(__dsub_rn(t, (double)n)) <= __dmul_rn(1e-6, scale))) ok = false;
      if (!ok && SMX.status == 0) SMX.status = RW_ERR_VALIDATION;
    }
    __syncthreads();
    if (SMX.status) return;
    if (m == 1) {  // :239-249
      pass(PASS_FIXED, SMX.zero, false, nullptr, nullptr);
      for (int j = tid; j < n; j += T) mo[j] = 0;
      if (tid == 0) {
        SMX.alpha_star[0] = 0.0;
        SMX.score = SMX.dual_bound = __ddiv_rn(SMX.S, (double)n);
        SMX.gap = 0.0;
        SMX.resid[0] = __ddiv_rn(__dsub_rn((double)n, SMX.c[0]), (double)n);
        SMX.counts[0] = n;
        SMX.iterations = 0;
        SMX.converged = 1;
      }
      __syncthreads();
      return;
    }
    if (tid == 0) {
      for (int i = 0; i < m; ++i) {
        SMX.alpha[i] = has_init ? SMX.init[i] : 0.0;
        SMX.best_alpha[i] = SMX.alpha[i];
        SMX.zero[i] = 0.0;
      }
      SMX.best_g = CUDART_INF;
      SMX.converged = 0;
      SMX.iterations = 0;
    }
    __syncthreads();
    {  // consider(0, g(0))  (:271-274)
      double g = eval_dual(SMX.zero, false, nullptr);
      if (tid == 0 && g < SMX.best_g) {
        SMX.best_g = g;
        for (int i = 0; i < m; ++i) SMX.best_alpha[i] = 0.0;
      }
    }
    for (int t = 0; t < p.max_iters; ++t) {  // :279-292
      double g = eval_dual(SMX.alpha, true, nullptr);
      if (tid == 0) {
        if (g < SMX.best_g) {
          SMX.best_g = g;
          for (int i = 0; i < m; ++i) SMX.best_alpha[i] = SMX.alpha[i];
        }
        SMX.iterations = t + 1;
        double resid = 0.0;
        for (int i = 0; i < m; ++i)
          resid = smax(resid, fabs(__dsub_rn((double)SMX.counts[i], SMX.c[i])));
        resid = __ddiv_rn(resid, (double)n);
        if (resid <= p.residual_tol) {
          SMX.converged = 1;
          SMX.flag = 1;
        } else {
          SMX.flag = 0;
          double eta = __ddiv_rn(p.eta0, sqrt(__dadd_rn((double)t, 1.0)));
          for (int i = 0; i < m; ++i)
            SMX.alpha[i] = __dadd_rn(
                SMX.alpha[i],
                __ddiv_rn(__dmul_rn(eta, __dsub_rn((double)SMX.counts[i], SMX.c[i])), (double)n));
        }
      }
      __syncthreads();
      if (SMX.flag) break;
    }
    if (tid == 0)
      for (int i = 0; i < m; ++i) SMX.polished[i] = SMX.best_alpha[i];
    for (int ps = 0; ps < p.polish_passes; ++ps) {  // :297-306
      polish_pass();
      double g = eval_dual(SMX.polished, false, nullptr);
      if (tid == 0) {
        if (g < SMX.best_g) {
          SMX.best_g = g;
          for (int i = 0; i < m; ++i) SMX.best_alpha[i] = SMX.polished[i];
        }
        SMX.flag = (SMX.max_delta <= 1e-15);
        if (SMX.flag) SMX.converged = 1;
      }
      __syncthreads();
      if (SMX.flag) break;
    }
    if (tid == 0) {  // gauge (:309-310)
      double lo = SMX.best_alpha[0];
      for (int i = 1; i < m; ++i)
        if (SMX.best_alpha[i] < lo) lo = SMX.best_alpha[i];
      for (int i = 0; i < m; ++i) {
        SMX.best_alpha[i] = __dsub_rn(SMX.best_alpha[i], lo);
        SMX.alpha_star[i] = SMX.best_alpha[i];
      }
    }
    __syncthreads();
    double db = eval_dual(SMX.best_alpha, true, mo);  // :313
    bool integral = true;
    for (int i = 0; i < m; ++i)
      if (fabs(__dsub_rn(SMX.c[i], round(SMX.c[i]))) > 1e-9) integral = false;
    if (tid == 0) {
      SMX.dual_bound = db;
      for (int i = 0; i < m; ++i)
        SMX.resid[i] = __ddiv_rn(__dsub_rn((double)SMX.counts[i], SMX.c[i]), (double)n);
      if (integral)
        for (int i = 0; i < m; ++i) SMX.target[i] = (int)llround(SMX.c[i]);
    }
    __syncthreads();
    if (integral) {  // :317-321
      double sc = repair();
      if (tid == 0) {
        SMX.score = sc;
        SMX.gap = __dsub_rn(SMX.dual_bound, sc);
      }
    } else if (tid == 0) {
      SMX.score = SMX.dual_bound;
      SMX.gap = 0.0;
    }
    __syncthreads();
  }

  // ---- optimize_fractions (routing_opt.cpp:70-136) -------------------------------------
  // out: SMX.fr_w, fr_score, fr_lat, fr_obj, fr_iters, fr_conv, fr_oor
  __device__ void optimize_fractions(double beta, const rw_opt_context& opt,
                                     const rw_pga_params& p) {
    if (tid == 0) {
      for (int i = 0; i < m; ++i) {
        SMX.w[i] = __ddiv_rn(1.0, (double)m);
        SMX.best_w[i] = SMX.w[i];
      }
      SMX.best_obj = -CUDART_INF;
      SMX.have_warm = 0;
      SMX.fr_iters = 0;
      SMX.fr_conv = 0;
    }
    __syncthreads();
    for (int t = 0; t < p.max_iters; ++t) {
      if (tid == 0)
        for (int i = 0; i < m; ++i) {
          SMX.c[i] = __dmul_rn((double)n, SMX.w[i]);
          SMX.init[i] = SMX.warm[i];
        }
      __syncthreads();
      solve_dual(p.dual, SMX.have_warm != 0);
      if (SMX.status) return;
      if (tid == 0) {
        for (int i = 0; i < m; ++i) SMX.warm[i] = SMX.alpha_star[i];
        SMX.have_warm = 1;
        double lat = system_latency(jb, pidx, m, SMX.w, opt.lambda_rps, opt.kappa, nullptr,
                                    nullptr, nullptr);
        double obj = __dsub_rn(SMX.dual_bound, __dmul_rn(beta, __dsub_rn(lat, opt.tau_ms)));
        if (obj > SMX.best_obj) {
          SMX.best_obj = obj;
          for (int i = 0; i < m; ++i) SMX.best_w[i] = SMX.w[i];
        }
        SMX.fr_iters = t + 1;
        system_latency_grad(jb, pidx, m, SMX.w, opt.lambda_rps, SMX.grad);
        for (int i = 0; i < m; ++i)
          SMX.step[i] = __dadd_rn(
              SMX.w[i], __dmul_rn(p.eta, __dsub_rn(SMX.alpha_star[i], __dmul_rn(beta, SMX.grad[i]))));
        if (!project_simplex(m, SMX.step, SMX.nextw, SMX.tmp)) {
          if (SMX.status == 0) SMX.status = RW_ERR_VALIDATION;
          SMX.flag = 1;
        } else {
          double moved = 0.0;
          for (int i = 0; i < m; ++i) moved = smax(moved, fabs(__dsub_rn(SMX.nextw[i], SMX.w[i])));
          for (int i = 0; i < m; ++i) SMX.w[i] = SMX.nextw[i];
          SMX.flag = (moved <= p.w_tol);
          if (SMX.flag) SMX.fr_conv = 1;
        }
      }
      __syncthreads();
      if (SMX.status) return;
      if (SMX.flag) break;
    }
    if (tid == 0)
      for (int i = 0; i < m; ++i) SMX.c[i] = __dmul_rn((double)n, SMX.best_w[i]);
    __syncthreads();
    solve_dual(p.dual, false);  // canonical cold re-solve (:121-123)
    if (SMX.status) return;
    if (tid == 0) {
      unsigned oor = 0;
      double lat = system_latency(jb, pidx, m, SMX.best_w, opt.lambda_rps, opt.kappa, &oor,
                                  nullptr, nullptr);
      for (int i = 0; i < m; ++i) SMX.fr_w[i] = SMX.best_w[i];
      SMX.fr_score = SMX.score;
      SMX.fr_lat = lat;
      SMX.fr_obj = __dsub_rn(SMX.score, __dmul_rn(beta, __dsub_rn(lat, opt.tau_ms)));
      SMX.fr_oor = oor;
    }
    __syncthreads();
  }

  // ---- optimize_beta (routing_opt.cpp:138-173) ------------------------------------------
  __device__ void optimize_beta(const rw_opt_context& opt, const rw_beta_params& bp,
                                rw_beta_step* trace, int trace_cap) {
    if (tid == 0) {
      double lo = bp.beta_min, hi = bp.beta_max;
      if (hi < 0.0) {
        if (!(opt.tau_ms > 0.0)) SMX.status = RW_ERR_VALIDATION;
        hi = __ddiv_rn(10.0, opt.tau_ms);
      }
      double eps = bp.epsilon;
      if (eps < 0.0) eps = __ddiv_rn(__dsub_rn(hi, lo), 1024.0);
      if (!(lo >= 0.0) || !(lo < hi)) SMX.status = RW_ERR_VALIDATION;
      if (!(eps > 0.0)) SMX.status = RW_ERR_VALIDATION;
      SMX.lo = lo;
      SMX.hi = hi;
      SMX.eps = eps;
      SMX.b_feasible = 0;
      SMX.b_has = 0;
      SMX.n_trace = 0;
      SMX.beta_star = 0.0;
      SMX.bst_score = SMX.bst_lat = SMX.bst_obj = 0.0;
      SMX.bst_iters = SMX.bst_conv = 0;
      SMX.bst_oor = 0;
      for (int i = 0; i < m; ++i) {
        SMX.w_star[i] = 0.0;
        SMX.bst_w[i] = 0.0;
      }
      SMX.tr_best_lat = 0.0;
      SMX.tr_best_score = 0.0;
    }
    __syncthreads();
    if (SMX.status) return;
    while (__dsub_rn(SMX.hi, SMX.lo) > SMX.eps) {
      const double mid = __dmul_rn(0.5, __dadd_rn(SMX.lo, SMX.hi));
      optimize_fractions(mid, opt, bp.pga);
      if (SMX.status) return;
      if (tid == 0) {
        bool ok = SMX.fr_lat <= opt.tau_ms && SMX.fr_oor == 0u;
        if (trace && SMX.n_trace < trace_cap) {
          trace[SMX.n_trace].beta = mid;
          trace[SMX.n_trace].score = SMX.fr_score;
          trace[SMX.n_trace].latency_ms = SMX.fr_lat;
          trace[SMX.n_trace].feasible = ok ? 1 : 0;
          trace[SMX.n_trace].pad_ = 0;
        }
        if (SMX.n_trace == 0 || SMX.fr_lat < SMX.tr_best_lat) {  // setup_search.cpp:200-202
          SMX.tr_best_lat = SMX.fr_lat;
          SMX.tr_best_score = SMX.fr_score;
        }
        SMX.n_trace++;
        if (ok) {
          SMX.b_feasible = 1;
          SMX.b_has = 1;
          SMX.beta_star = mid;
          for (int i = 0; i < m; ++i) {
            SMX.w_star[i] = SMX.fr_w[i];
            SMX.bst_w[i] = SMX.fr_w[i];
          }
          SMX.bst_score = SMX.fr_score;
          SMX.bst_lat = SMX.fr_lat;
          SMX.bst_obj = SMX.fr_obj;
          SMX.bst_iters = SMX.fr_iters;
          SMX.bst_conv = SMX.fr_conv;
          SMX.bst_oor = SMX.fr_oor;
          SMX.hi = mid;
        } else {
          SMX.lo = mid;
        }
      }
      __syncthreads();
    }
  }

  __device__ void reset_counters() {
    if (tid == 0) {
      SMX.status = 0;
      SMX.eval_passes = 0;
      SMX.polish_passes = 0;
      SMX.repair_calls = 0;
      SMX.pol_delta = 1e-3;
      for (int i = 0; i < 8; ++i) SMX.prof[i] = 0;
      for (int i = 0; i < MM; ++i) SMX.zero[i] = 0.0;
    }
    __syncthreads();
  }

  // ---- select_setup's evaluate (setup_search.cpp:187-211) -> one record ---------------
  __device__ void evaluate_setup(long long inst, rw_setup_record* rec) {
    const long long k = inst % jb.n_setups;
    rw_opt_context opt = jb.opt;
    if (jb.taus) opt.tau_ms = jb.taus[inst / jb.n_setups];
    const rw_beta_params bp = jb.bps ? jb.bps[inst / jb.n_setups] : jb.bp;
    pidx = jb.prof_idx + (size_t)k * m;
    reset_counters();
    optimize_beta(opt, bp, nullptr, 0);
    int bisect = SMX.n_trace;
    double e_score = 0.0, e_lat = 0.0;
    if (!SMX.status && !SMX.b_feasible) {
      if (SMX.n_trace > 0) {
        e_score = SMX.tr_best_score;
        e_lat = SMX.tr_best_lat;
      } else {  // degenerate bracket: evaluate the top penalty once
        double beta_hi = bp.beta_max;
        if (beta_hi < 0.0) beta_hi = __ddiv_rn(10.0, opt.tau_ms);
        optimize_fractions(beta_hi, opt, bp.pga);
        e_score = SMX.fr_score;
        e_lat = SMX.fr_lat;
      }
    }
    __syncthreads();
    if (tid == 0) {
      rec->setup_id = jb.setup_ids ? jb.setup_ids[k] : k;
      rec->status = SMX.status;
      rec->feasible = (!SMX.status && SMX.b_feasible) ? 1 : 0;
      rec->score = SMX.b_feasible ? SMX.bst_score : e_score;
      rec->latency_ms = SMX.b_feasible ? SMX.bst_lat : e_lat;
      rec->beta = SMX.b_feasible ? SMX.beta_star : 0.0;
      rec->tau_ms = opt.tau_ms;
      for (int i = 0; i < RW_MAX_MODELS; ++i)
        rec->w[i] = (SMX.b_feasible && i < m) ? SMX.bst_w[i] : 0.0;
      rec->out_of_range = SMX.b_feasible ? SMX.bst_oor : 0u;
      rec->bisect_steps = bisect;
      rec->eval_passes = SMX.eval_passes;
      rec->polish_passes = SMX.polish_passes;
      rec->repair_calls = SMX.repair_calls;
    }
    __syncthreads();
  }
};

#undef SMX

// ---------------------------------------------------------------------------------------
template <int MM, int L, int T>
__global__ void __launch_bounds__(T, (MM <= 16 && T <= 256) ? 2 : 1) solver_kernel(const Job jb) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  using SM = Smem<MM, L, T>;
  SM& sm = *reinterpret_cast<SM*>(smem_raw);
  const int slot = blockIdx.x;
  uint8_t* mo = jb.ws_model_of + (size_t)slot * jb.n;
  unsigned long long* keys = reinterpret_cast<unsigned long long*>(jb.ws_keys) + (size_t)slot * jb.n;
  Solver<MM, L, T> s(jb, mo, keys);
  const int tid = threadIdx.x;
  const int m = jb.m, n = jb.n;

  if (jb.kind == JOB_SWEEP) {
    for (;;) {
      if (tid == 0) sm.cur_item = (long long)atomicAdd(jb.queue, 1ull);
      __syncthreads();
      const long long item = sm.cur_item;
      __syncthreads();
      const long long k = (long long)jb.shard_rank + item * jb.shard_count;
      if (k >= jb.n_items) break;
      s.evaluate_setup(k, jb.records + item);
      if (tid == 0 && jb.prof_out)
        for (int i = 0; i < 8; ++i)
          atomicAdd((unsigned long long*)jb.prof_out + i, (unsigned long long)sm.prof[i]);
      if (tid == 0 && sm.status && jb.status_out) atomicCAS(jb.status_out, 0, sm.status);
    }
    return;
  }
  if (blockIdx.x != 0) return;
  s.reset_counters();
  if (jb.kind == JOB_EVAL) {
    if (tid == 0)
      for (int i = 0; i < m; ++i) {
        sm.c[i] = jb.c[i];
        sm.alpha[i] = jb.vec[i];
      }
    __syncthreads();
    double g = s.eval_dual(sm.alpha, true, mo);
    for (int j = tid; j < n; j += T) jb.assign_out[j] = mo[j];
    if (tid == 0) {
      jb.dvec_out[0] = g;
      for (int i = 0; i < m; ++i) jb.ivec_out[i] = sm.counts[i];
    }
  } else if (jb.kind == JOB_SOLVE) {
    if (tid == 0)
      for (int i = 0; i < m; ++i) {
        sm.c[i] = jb.c[i];
        sm.init[i] = jb.vec[i];
      }
    __syncthreads();
    s.solve_dual(jb.bp.pga.dual, jb.has_vec != 0);
    if (!sm.status && jb.assign_out)
      for (int j = tid; j < n; j += T) jb.assign_out[j] = mo[j];
    if (tid == 0) {
      rw_dual_solution* o = jb.dual_out;
      for (int i = 0; i < RW_MAX_MODELS; ++i) {
        o->alpha_star[i] = i < m ? sm.alpha_star[i] : 0.0;
        o->count_residual[i] = i < m ? sm.resid[i] : 0.0;
        o->counts[i] = i < m ? sm.counts[i] : 0;
      }
      o->score = sm.score;
      o->dual_bound = sm.dual_bound;
      o->duality_gap = sm.gap;
      o->iterations = sm.iterations;
      o->converged = sm.converged;
      o->eval_passes = sm.eval_passes;
    }
  } else if (jb.kind == JOB_OPTFRAC) {
    s.pidx = jb.prof_idx;
    s.optimize_fractions(jb.beta, jb.opt, jb.bp.pga);
    if (tid == 0 && !sm.status) {
      rw_relaxed_result* o = jb.relaxed_out;
      for (int i = 0; i < RW_MAX_MODELS; ++i) o->w[i] = i < m ? sm.fr_w[i] : 0.0;
      o->objective = sm.fr_obj;
      o->score = sm.fr_score;
      o->latency_ms = sm.fr_lat;
      o->iterations = sm.fr_iters;
      o->converged = sm.fr_conv;
      o->out_of_range = sm.fr_oor;
      o->pad_ = 0;
      o->eval_passes = sm.eval_passes;
    }
  } else if (jb.kind == JOB_OPTBETA) {
    s.pidx = jb.prof_idx;
    s.optimize_beta(jb.opt, jb.bp, jb.trace_out, jb.trace_cap);
    if (tid == 0 && !sm.status) {
      rw_beta_result* o = jb.beta_out;
      o->feasible = sm.b_feasible;
      o->has_beta_star = sm.b_has;
      o->beta_star = sm.beta_star;
      for (int i = 0; i < RW_MAX_MODELS; ++i) {
        o->w_star[i] = i < m ? sm.w_star[i] : 0.0;
        o->best.w[i] = i < m ? sm.bst_w[i] : 0.0;
      }
      o->best.objective = sm.bst_obj;
      o->best.score = sm.bst_score;
      o->best.latency_ms = sm.bst_lat;
      o->best.iterations = sm.bst_iters;
      o->best.converged = sm.bst_conv;
      o->best.out_of_range = sm.bst_oor;
      o->best.pad_ = 0;
      o->best.eval_passes = 0;
      o->n_trace = sm.n_trace;
      o->pad_ = 0;
      o->eval_passes = sm.eval_passes;
    }
  } else if (jb.kind == JOB_BENCH_PASS) {
    // diagnostics: trip_count eval passes at fixed prices (alpha, c from the job)
    if (tid == 0)
      for (int i = 0; i < m; ++i) {
        sm.c[i] = jb.c[i];
        sm.alpha[i] = jb.vec[i];
      }
    __syncthreads();
    double g = 0.0;
    for (int it = 0; it < jb.trace_cap; ++it) g = s.eval_dual(sm.alpha, true, nullptr);
    if (tid == 0) {
      jb.dvec_out[0] = g;
      for (int i = 0; i < m; ++i) jb.ivec_out[i] = sm.counts[i];
    }
  } else if (jb.kind == JOB_SIMPLEX) {
    if (tid == 0) {
      if (!project_simplex(m, jb.vec, jb.dvec_out, sm.tmp)) sm.status = RW_ERR_VALIDATION;
    }
  } else if (jb.kind == JOB_LATENCY) {
    if (tid == 0) {
      unsigned oor = 0;
      double* d = jb.dvec_out;
      d[0] = system_latency(jb, jb.prof_idx, m, jb.vec, jb.opt.lambda_rps, jb.opt.kappa, &oor,
                            d + 1, d + 1 + m);
      system_latency_grad(jb, jb.prof_idx, m, jb.vec, jb.opt.lambda_rps, d + 1 + 2 * m);
      for (int i = 0; i < m; ++i) jb.ivec_out[i] = (oor >> i) & 1u;
    }
  }
  __syncthreads();
  if (tid == 0 && sm.status && jb.status_out) atomicCAS(jb.status_out, 0, sm.status);
  if (tid == 0 && jb.prof_out)
    for (int i = 0; i < 8; ++i) atomicAdd((unsigned long long*)jb.prof_out + i, (unsigned long long)sm.prof[i]);
}

}  // namespace rw
