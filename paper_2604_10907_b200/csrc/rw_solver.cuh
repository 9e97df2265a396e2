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
  static constexpr int BPAD = R + R / 16;
  double b[BPAD];                       // tile's b_j (padded: 1 slot per 16 against conflicts)
  long long q0[T], q1[T];               // per-thread chunk quanta
  long long wq0[W], wq1[W];             // per-warp composed quanta
  double scan_x[W], scan_y[W];
  unsigned hist[256];
  unsigned char safe[T];
  unsigned char wuni[W];
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

template <int MM, int L, int T>
struct Solver {
  using SM = Smem<MM, L, T>;
  static constexpr int R = SM::R;
  static constexpr int W = SM::W;
  static constexpr int NPK = (MM + 3) / 4;  // packed 16-bit count words

  SM& sm;
  const Job& jb;
  const int n, m;
  const int tid, lane, wid;
  uint8_t* mo;               // this CTA's model_of workspace [n]
  unsigned long long* keys;  // this CTA's radix-select workspace [n]
  const int32_t* pidx;       // current setup's profile indices [m]

  __device__ Solver(SM& s, const Job& j, uint8_t* mo_, unsigned long long* keys_)
      : sm(s), jb(j), n(j.n), m(j.m), tid(threadIdx.x), lane(threadIdx.x & 31),
        wid(threadIdx.x >> 5), mo(mo_), keys(keys_), pidx(nullptr) {}

  __device__ __forceinline__ static int pad(int i) { return i + (i >> 4); }

  __device__ void fail(int code) {
    if (tid == 0 && sm.status == 0) sm.status = code;
  }

  // ---- one pass over the N x M matrix (score_dual.cpp:25-49) ------------------------
  // PASS_EVAL : b_j = max_i (s_ji - alpha_i), arg = first max; counts; optional model_of.
  // PASS_FIXED: b_j = s_j,mo[j] (mo == null -> column 0).
  // Result: sm.S = the reference's sequential FP64 sum of b_j, bit for bit.
  __device__ void pass(int mode, const double* alpha_s, bool want_counts, uint8_t* mo_out,
                       const uint8_t* mo_in) {
    __syncthreads();  // callers may still be reading the previous pass's sm.S / counts
    double a[MM];
#pragma unroll
    for (int i = 0; i < MM; ++i) a[i] = (i < m) ? alpha_s[i] : 0.0;
    if (tid == 0) {
      sm.S = 0.0;
      sm.P = 0.0;
      sm.A = 0.0;
      if (mode == PASS_EVAL) sm.eval_passes++;
    }
    if (tid < MM) sm.counts[tid] = 0;
    __syncthreads();
    const double* __restrict__ sc = jb.scores;
    const bool vec2 = ((m & 1) == 0);
    for (int base = 0; base < n; base += R) {
      const int len = min(R, n - base);
      // -- phase 1: coalesced rows -> b_j, argmax, packed counts -----------------------
      unsigned long long pk[NPK];
#pragma unroll
      for (int q = 0; q < NPK; ++q) pk[q] = 0ull;
#pragma unroll 2
      for (int r = 0; r < L; ++r) {
        const int k = r * T + tid;
        if (k < len) {
          const int j = base + k;
          const double* row = sc + (size_t)j * m;
          double bj;
          int arg;
          if (mode == PASS_EVAL) {
            double v[MM];
            if (vec2) {
              const double2* r2 = reinterpret_cast<const double2*>(row);
#pragma unroll
              for (int i = 0; i < MM / 2; ++i) {
                if (2 * i < m) {
                  double2 x = __ldg(r2 + i);
                  v[2 * i] = x.x;
                  v[2 * i + 1] = x.y;
                } else {
                  v[2 * i] = 0.0;
                  v[2 * i + 1] = 0.0;
                }
              }
            } else {
#pragma unroll
              for (int i = 0; i < MM; ++i) v[i] = (i < m) ? __ldg(row + i) : 0.0;
            }
            bj = __dsub_rn(v[0], a[0]);
            arg = 0;
#pragma unroll
            for (int i = 1; i < MM; ++i) {
              if (i < m) {
                double x = __dsub_rn(v[i], a[i]);
                if (x > bj) {
                  bj = x;
                  arg = i;
                }
              }
            }
          } else {
            arg = mo_in ? (int)mo_in[j] : 0;
            bj = __ldg(row + arg);
          }
          sm.b[pad(k)] = bj;
          if (want_counts) {
#pragma unroll
            for (int q = 0; q < NPK; ++q)
              pk[q] += ((arg >> 2) == q) ? (1ull << ((arg & 3) * 16)) : 0ull;
          }
          if (mo_out) mo_out[j] = (uint8_t)arg;
        }
      }
      if (want_counts) {
#pragma unroll
        for (int q = 0; q < NPK; ++q) {
          unsigned long long x = pk[q];
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) x += __shfl_down_sync(FULL, x, off);
          if (lane == 0) {
#pragma unroll
            for (int f = 0; f < 4; ++f) {
              int i = 4 * q + f;
              unsigned cnt = (unsigned)((x >> (16 * f)) & 0xffffull);
              if (i < m && cnt) atomicAdd(&sm.counts[i], (int)cnt);
            }
          }
        }
      }
      __syncthreads();
      // -- phase 2: chunk quanta --------------------------------------------------------
      const int c0 = tid * L;
      const int cnt = max(0, min(L, len - c0));
      double bl[L];
      double ps = 0.0, pa = 0.0;
#pragma unroll
      for (int r = 0; r < L; ++r) {
        bl[r] = (r < cnt) ? sm.b[pad(c0 + r)] : 0.0;
        ps += bl[r];
        pa += fabs(bl[r]);
      }
      // block exclusive scan of (ps, pa) (approximate: only used with an error margin)
      double ix = ps, iy = pa;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        double tx = __shfl_up_sync(FULL, ix, off), ty = __shfl_up_sync(FULL, iy, off);
        if (lane >= off) {
          ix += tx;
          iy += ty;
        }
      }
      if (lane == 31) {
        sm.scan_x[wid] = ix;
        sm.scan_y[wid] = iy;
      }
      double ex = __shfl_up_sync(FULL, ix, 1), ey = __shfl_up_sync(FULL, iy, 1);
      if (lane == 0) {
        ex = 0.0;
        ey = 0.0;
      }
      __syncthreads();
      double wx = 0.0, wy = 0.0, tx = 0.0, ty = 0.0;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        double sx = sm.scan_x[w], sy = sm.scan_y[w];
        if (w < wid) {
          wx += sx;
          wy += sy;
        }
        tx += sx;
        ty += sy;
      }
      double P = sm.P + (wx + ex);
      double A = sm.A + (wy + ey);
      const long long jg = (long long)base + c0;
      int safe = cnt > 0;
      int e_ref = 0, neg_ref = 0;
#pragma unroll
      for (int r = 0; r <= L; ++r) {
        if (r <= cnt && safe) {
          double Ab = A + ((r < cnt) ? fabs(bl[r]) : 0.0);
          double E = (double)(jg + r + 64) * 0x1p-51 * Ab;
          int e, ng;
          if (!in_binade(P, E, e, ng)) safe = 0;
          else if (r == 0) {
            e_ref = e;
            neg_ref = ng;
          } else if (e != e_ref || ng != neg_ref) safe = 0;
        }
        if (r < cnt) {
          P += bl[r];
          A += fabs(bl[r]);
        }
      }
      long long Q0 = 0, Q1 = 0;
      if (safe) {
        const double scale = __longlong_as_double((long long)(52 - e_ref + 1023) << 52);
#pragma unroll
        for (int r = 0; r < L; ++r) {
          if (r < cnt) {
            double y = bl[r] * scale;  // exact (power-of-two scaling)
            double fy = floor(y);
            double fr = y - fy;        // exact
            long long qf = (long long)fy;
            if (fr == 0.5) {  // half-ulp tie: RNE to the even result
              Q0 += ((Q0 + qf) & 1) ? qf + 1 : qf;
              Q1 += ((1 + Q1 + qf) & 1) ? qf + 1 : qf;
            } else {
              long long q = (fr > 0.5) ? qf + 1 : qf;
              Q0 += q;
              Q1 += q;
            }
          }
        }
      }
      sm.q0[tid] = Q0;
      sm.q1[tid] = Q1;
      sm.safe[tid] = (unsigned char)safe;
      const int key = safe ? (e_ref * 2 + neg_ref) : (100000 + lane);
      const bool uni = __all_sync(FULL, key == __shfl_sync(FULL, key, 0));
      if (uni) {  // ordered tree composition of the 32 chunk maps
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          long long o0 = __shfl_down_sync(FULL, Q0, d), o1 = __shfl_down_sync(FULL, Q1, d);
          if ((lane & (2 * d - 1)) == 0) {
            long long n0 = Q0 + ((Q0 & 1) ? o1 : o0);
            long long n1 = Q1 + (((1 + Q1) & 1) ? o1 : o0);
            Q0 = n0;
            Q1 = n1;
          }
        }
      }
      if (lane == 0) {
        sm.wuni[wid] = uni ? 1 : 0;
        sm.wq0[wid] = Q0;
        sm.wq1[wid] = Q1;
        if (wid == 0) {
          sm.tileP = tx;
          sm.tileA = ty;
        }
      }
      __syncthreads();
      // -- phase 3: ordered walk (one thread) -------------------------------------------
      if (tid == 0) {
        double S = sm.S;
        const int nw = min(W, (len + 32 * L - 1) / (32 * L));
        for (int w = 0; w < nw; ++w) {
          if (sm.wuni[w]) {
            S = apply_quanta(S, sm.wq0[w], sm.wq1[w]);
            continue;
          }
          for (int l = 0; l < 32; ++l) {
            const int t = w * 32 + l;
            const int tc0 = t * L;
            const int tcnt = min(L, len - tc0);
            if (tcnt <= 0) break;
            if (sm.safe[t]) {
              S = apply_quanta(S, sm.q0[t], sm.q1[t]);
            } else {
              for (int r = 0; r < tcnt; ++r) S = __dadd_rn(S, sm.b[pad(tc0 + r)]);
            }
          }
        }
        sm.S = S;
        sm.P += sm.tileP;
        sm.A += sm.tileA;
      }
      __syncthreads();
    }
  }

  // g(alpha) = (sum_j best_j + sum_i alpha_i c_i) / N   (score_dual.cpp:47-48)
  __device__ double eval_dual(const double* alpha_s, bool want_counts, uint8_t* mo_out) {
    pass(PASS_EVAL, alpha_s, want_counts, mo_out, nullptr);
    double g = sm.S;
    for (int i = 0; i < m; ++i) g = __dadd_rn(g, __dmul_rn(alpha_s[i], sm.c[i]));
    return __ddiv_rn(g, (double)n);  // every thread computes the same value
  }

  // ---- radix select: k-th largest key among keys[0..n) (nth_element, :71-72) ----------
  __device__ __forceinline__ void hist_add(bool ok, unsigned d) {
    unsigned act = __activemask();
    unsigned key = ok ? d : 0xffffffffu;
    unsigned peers = __match_any_sync(act, key);
    if (ok && lane == __ffs(peers) - 1) atomicAdd(&sm.hist[d], __popc(peers));
  }
  // Picks the digit holding the sel_k-th largest among counted candidates (warp 0).
  __device__ void select_digit(int shift) {
    if (wid == 0) {
      // lane l covers bins [248 - 8l, 255 - 8l], top bins first
      const int top = 255 - 8 * lane;
      int local = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) local += (int)sm.hist[top - q];
      int incl = local;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        int t = __shfl_up_sync(FULL, incl, off);
        if (lane >= off) incl += t;
      }
      const int excl = incl - local;
      const int k = sm.sel_k;
      if (excl < k && k <= incl) {
        int above = excl;
        for (int q = 0; q < 8; ++q) {
          int h = (int)sm.hist[top - q];
          if (above + h >= k) {
            sm.sel_prefix |= (unsigned long long)(top - q) << shift;
            sm.sel_k = k - above;
            break;
          }
          above += h;
        }
      }
    }
  }

  // ---- polish_pass (score_dual.cpp:54-76) on sm.polished --------------------------------
  __device__ void polish_pass() {
    if (tid == 0) {
      sm.max_delta = 0.0;
      sm.polish_passes++;
    }
    for (int i = 0; i < m; ++i) {
      __syncthreads();
      double a[MM];
#pragma unroll
      for (int q = 0; q < MM; ++q) a[q] = (q < m) ? sm.polished[q] : 0.0;
      const double ci = sm.c[i];
      int k = ci > 1e-12 ? (int)ceil(__dsub_rn(ci, 1e-9)) : 1;
      k = max(1, min(k, n));
      if (tid < 256) sm.hist[tid] = 0u;
      if (tid == 0) {
        sm.sel_prefix = 0ull;
        sm.sel_k = k;
      }
      __syncthreads();
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
        unsigned long long key = dkey(__dsub_rn(vi, rest));
        keys[j] = key;
        hist_add(true, (unsigned)(key >> 56));
      }
      __syncthreads();
      select_digit(56);
      for (int shift = 48; shift >= 0; shift -= 8) {
        __syncthreads();
        if (tid < 256) sm.hist[tid] = 0u;
        __syncthreads();
        const unsigned long long hi = sm.sel_prefix >> (shift + 8);
        for (int j = tid; j < n; j += T) {
          unsigned long long key = keys[j];
          hist_add((key >> (shift + 8)) == hi, (unsigned)((key >> shift) & 0xffull));
        }
        __syncthreads();
        select_digit(shift);
      }
      __syncthreads();
      if (tid == 0) {
        double next = dkey_inv(sm.sel_prefix);
        sm.max_delta = smax(sm.max_delta, fabs(__dsub_rn(next, sm.polished[i])));
        sm.polished[i] = next;
      }
    }
    __syncthreads();
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
      sm.red_d[wid] = val;
      sm.red_j[wid] = j;
      sm.red_v[wid] = v;
    }
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < W; ++w) {
        double ov = sm.red_d[w];
        int oj = sm.red_j[w];
        if (oj >= 0 && (sm.red_j[0] < 0 || ov < sm.red_d[0] ||
                        (ov == sm.red_d[0] && oj < sm.red_j[0]))) {
          sm.red_d[0] = ov;
          sm.red_j[0] = oj;
          sm.red_v[0] = sm.red_v[w];
        }
      }
    }
    __syncthreads();
    val = sm.red_d[0];
    j = sm.red_j[0];
    v = sm.red_v[0];
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
      sm.red_d[wid] = val;
      sm.red_j[wid] = j;
    }
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < W; ++w) {
        double ov = sm.red_d[w];
        int oj = sm.red_j[w];
        if (oj >= 0 && (sm.red_j[0] < 0 || ov > sm.red_d[0] ||
                        (ov == sm.red_d[0] && oj < sm.red_j[0]))) {
          sm.red_d[0] = ov;
          sm.red_j[0] = oj;
        }
      }
    }
    __syncthreads();
    val = sm.red_d[0];
    j = sm.red_j[0];
    __syncthreads();
  }

  // ---- repair_counts (score_dual.cpp:81-185); counts in sm.counts, targets in sm.target
  __device__ double repair() {
    if (tid == 0) {
      sm.repair_calls++;
      for (int i = 0; i < m; ++i) sm.delta[i] = sm.counts[i] - sm.target[i];
    }
    __syncthreads();
    // Phase 1: min-loss single moves while any surplus remains (:96-118)
    for (;;) {
      bool over = false;
      for (int i = 0; i < m; ++i) over = over || sm.delta[i] > 0;
      if (!over) break;
      double bl = CUDART_INF;
      int bj = -1, bv = -1;
      for (int j = tid; j < n; j += T) {
        int u = mo[j];
        if (sm.delta[u] <= 0) continue;
        const double* row = jb.scores + (size_t)j * m;
        double su = __ldg(row + u);
        for (int v = 0; v < m; ++v) {
          if (sm.delta[v] >= 0) continue;
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
        sm.counts[u]--;
        sm.counts[bv]++;
        sm.delta[u]--;
        sm.delta[bv]++;
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
              sm.gain[u * m + v] = (j >= 0) ? g : -CUDART_INF;
              sm.witness[u * m + v] = j;
            }
          }
        }
        __syncthreads();
        if (tid == 0) {
          double best = 1e-15;
          int cu = -1, cv = -1, cw = -1;
          for (int u = 0; u < m; ++u)
            for (int v = u + 1; v < m; ++v) {
              double g = __dadd_rn(sm.gain[u * m + v], sm.gain[v * m + u]);
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
                double g = __dadd_rn(__dadd_rn(sm.gain[u * m + v], sm.gain[v * m + w]),
                                     sm.gain[w * m + u]);
                if (g > best) {
                  best = g;
                  cu = u;
                  cv = v;
                  cw = w;
                }
              }
            }
          sm.flag = (cu < 0);
          if (cu >= 0) {
            auto move = [&](int j, int v) {
              int uu = mo[j];
              mo[j] = (uint8_t)v;
              sm.counts[uu]--;
              sm.counts[v]++;
              sm.delta[uu]--;
              sm.delta[v]++;
            };
            if (cw < 0) {
              int j1 = sm.witness[cu * m + cv], j2 = sm.witness[cv * m + cu];
              move(j1, cv);
              move(j2, cu);
            } else {
              int j1 = sm.witness[cu * m + cv], j2 = sm.witness[cv * m + cw],
                  j3 = sm.witness[cw * m + cu];
              move(j1, cv);
              move(j2, cw);
              move(j3, cu);
            }
          }
        }
        __syncthreads();
        if (sm.flag) break;
        __syncthreads();
      }
    }
    __syncthreads();
    // exact sequential mean of the repaired assignment (:182-184)
    pass(PASS_FIXED, sm.zero, false, nullptr, mo);
    return __ddiv_rn(sm.S, (double)n);
  }

  // ---- solve_dual (score_dual.cpp:232-327) ---------------------------------------------
  // in: sm.c (targets), sm.init (when has_init); out: sm.alpha_star, score, dual_bound, gap,
  // resid, iterations, converged, sm.counts (realised), mo (assignment)
  __device__ void solve_dual(const rw_subgradient_params& p, bool has_init) {
    if (tid == 0) {  // TargetCounts::validate (:195-205)
      double t = 0.0;
      bool ok = true;
      for (int i = 0; i < m; ++i) {
        if (!isfinite(sm.c[i]) || sm.c[i] < -1e-9) ok = false;
        t = __dadd_rn(t, sm.c[i]);
      }
      double scale = (double)n > 1.0 ? (double)n : 1.0;
      if (!(fabs(__dsub_rn(t, (double)n)) <= __dmul_rn(1e-6, scale))) ok = false;
      if (!ok && sm.status == 0) sm.status = RW_ERR_VALIDATION;
    }
    __syncthreads();
    if (sm.status) return;
    if (m == 1) {  // :239-249
      pass(PASS_FIXED, sm.zero, false, nullptr, nullptr);
      for (int j = tid; j < n; j += T) mo[j] = 0;
      if (tid == 0) {
        sm.alpha_star[0] = 0.0;
        sm.score = sm.dual_bound = __ddiv_rn(sm.S, (double)n);
        sm.gap = 0.0;
        sm.resid[0] = __ddiv_rn(__dsub_rn((double)n, sm.c[0]), (double)n);
        sm.counts[0] = n;
        sm.iterations = 0;
        sm.converged = 1;
      }
      __syncthreads();
      return;
    }
    if (tid == 0) {
      for (int i = 0; i < m; ++i) {
        sm.alpha[i] = has_init ? sm.init[i] : 0.0;
        sm.best_alpha[i] = sm.alpha[i];
        sm.zero[i] = 0.0;
      }
      sm.best_g = CUDART_INF;
      sm.converged = 0;
      sm.iterations = 0;
    }
    __syncthreads();
    {  // consider(0, g(0))  (:271-274)
      double g = eval_dual(sm.zero, false, nullptr);
      if (tid == 0 && g < sm.best_g) {
        sm.best_g = g;
        for (int i = 0; i < m; ++i) sm.best_alpha[i] = 0.0;
      }
    }
    for (int t = 0; t < p.max_iters; ++t) {  // :279-292
      double g = eval_dual(sm.alpha, true, nullptr);
      if (tid == 0) {
        if (g < sm.best_g) {
          sm.best_g = g;
          for (int i = 0; i < m; ++i) sm.best_alpha[i] = sm.alpha[i];
        }
        sm.iterations = t + 1;
        double resid = 0.0;
        for (int i = 0; i < m; ++i)
          resid = smax(resid, fabs(__dsub_rn((double)sm.counts[i], sm.c[i])));
        resid = __ddiv_rn(resid, (double)n);
        if (resid <= p.residual_tol) {
          sm.converged = 1;
          sm.flag = 1;
        } else {
          sm.flag = 0;
          double eta = __ddiv_rn(p.eta0, sqrt(__dadd_rn((double)t, 1.0)));
          for (int i = 0; i < m; ++i)
            sm.alpha[i] = __dadd_rn(
                sm.alpha[i],
                __ddiv_rn(__dmul_rn(eta, __dsub_rn((double)sm.counts[i], sm.c[i])), (double)n));
        }
      }
      __syncthreads();
      if (sm.flag) break;
    }
    if (tid == 0)
      for (int i = 0; i < m; ++i) sm.polished[i] = sm.best_alpha[i];
    for (int ps = 0; ps < p.polish_passes; ++ps) {  // :297-306
      polish_pass();
      double g = eval_dual(sm.polished, false, nullptr);
      if (tid == 0) {
        if (g < sm.best_g) {
          sm.best_g = g;
          for (int i = 0; i < m; ++i) sm.best_alpha[i] = sm.polished[i];
        }
        sm.flag = (sm.max_delta <= 1e-15);
        if (sm.flag) sm.converged = 1;
      }
      __syncthreads();
      if (sm.flag) break;
    }
    if (tid == 0) {  // gauge (:309-310)
      double lo = sm.best_alpha[0];
      for (int i = 1; i < m; ++i)
        if (sm.best_alpha[i] < lo) lo = sm.best_alpha[i];
      for (int i = 0; i < m; ++i) {
        sm.best_alpha[i] = __dsub_rn(sm.best_alpha[i], lo);
        sm.alpha_star[i] = sm.best_alpha[i];
      }
    }
    __syncthreads();
    double db = eval_dual(sm.best_alpha, true, mo);  // :313
    bool integral = true;
    for (int i = 0; i < m; ++i)
      if (fabs(__dsub_rn(sm.c[i], round(sm.c[i]))) > 1e-9) integral = false;
    if (tid == 0) {
      sm.dual_bound = db;
      for (int i = 0; i < m; ++i)
        sm.resid[i] = __ddiv_rn(__dsub_rn((double)sm.counts[i], sm.c[i]), (double)n);
      if (integral)
        for (int i = 0; i < m; ++i) sm.target[i] = (int)llround(sm.c[i]);
    }
    __syncthreads();
    if (integral) {  // :317-321
      double sc = repair();
      if (tid == 0) {
        sm.score = sc;
        sm.gap = __dsub_rn(sm.dual_bound, sc);
      }
    } else if (tid == 0) {
      sm.score = sm.dual_bound;
      sm.gap = 0.0;
    }
    __syncthreads();
  }

  // ---- optimize_fractions (routing_opt.cpp:70-136) -------------------------------------
  // out: sm.fr_w, fr_score, fr_lat, fr_obj, fr_iters, fr_conv, fr_oor
  __device__ void optimize_fractions(double beta, const rw_opt_context& opt,
                                     const rw_pga_params& p) {
    if (tid == 0) {
      for (int i = 0; i < m; ++i) {
        sm.w[i] = __ddiv_rn(1.0, (double)m);
        sm.best_w[i] = sm.w[i];
      }
      sm.best_obj = -CUDART_INF;
      sm.have_warm = 0;
      sm.fr_iters = 0;
      sm.fr_conv = 0;
    }
    __syncthreads();
    for (int t = 0; t < p.max_iters; ++t) {
      if (tid == 0)
        for (int i = 0; i < m; ++i) {
          sm.c[i] = __dmul_rn((double)n, sm.w[i]);
          sm.init[i] = sm.warm[i];
        }
      __syncthreads();
      solve_dual(p.dual, sm.have_warm != 0);
      if (sm.status) return;
      if (tid == 0) {
        for (int i = 0; i < m; ++i) sm.warm[i] = sm.alpha_star[i];
        sm.have_warm = 1;
        double lat = system_latency(jb, pidx, m, sm.w, opt.lambda_rps, opt.kappa, nullptr,
                                    nullptr, nullptr);
        double obj = __dsub_rn(sm.dual_bound, __dmul_rn(beta, __dsub_rn(lat, opt.tau_ms)));
        if (obj > sm.best_obj) {
          sm.best_obj = obj;
          for (int i = 0; i < m; ++i) sm.best_w[i] = sm.w[i];
        }
        sm.fr_iters = t + 1;
        system_latency_grad(jb, pidx, m, sm.w, opt.lambda_rps, sm.grad);
        for (int i = 0; i < m; ++i)
          sm.step[i] = __dadd_rn(
              sm.w[i], __dmul_rn(p.eta, __dsub_rn(sm.alpha_star[i], __dmul_rn(beta, sm.grad[i]))));
        if (!project_simplex(m, sm.step, sm.nextw, sm.tmp)) {
          if (sm.status == 0) sm.status = RW_ERR_VALIDATION;
          sm.flag = 1;
        } else {
          double moved = 0.0;
          for (int i = 0; i < m; ++i) moved = smax(moved, fabs(__dsub_rn(sm.nextw[i], sm.w[i])));
          for (int i = 0; i < m; ++i) sm.w[i] = sm.nextw[i];
          sm.flag = (moved <= p.w_tol);
          if (sm.flag) sm.fr_conv = 1;
        }
      }
      __syncthreads();
      if (sm.status) return;
      if (sm.flag) break;
    }
    if (tid == 0)
      for (int i = 0; i < m; ++i) sm.c[i] = __dmul_rn((double)n, sm.best_w[i]);
    __syncthreads();
    solve_dual(p.dual, false);  // canonical cold re-solve (:121-123)
    if (sm.status) return;
    if (tid == 0) {
      unsigned oor = 0;
      double lat = system_latency(jb, pidx, m, sm.best_w, opt.lambda_rps, opt.kappa, &oor,
                                  nullptr, nullptr);
      for (int i = 0; i < m; ++i) sm.fr_w[i] = sm.best_w[i];
      sm.fr_score = sm.score;
      sm.fr_lat = lat;
      sm.fr_obj = __dsub_rn(sm.score, __dmul_rn(beta, __dsub_rn(lat, opt.tau_ms)));
      sm.fr_oor = oor;
    }
    __syncthreads();
  }

  // ---- optimize_beta (routing_opt.cpp:138-173) ------------------------------------------
  __device__ void optimize_beta(const rw_opt_context& opt, const rw_beta_params& bp,
                                rw_beta_step* trace, int trace_cap) {
    if (tid == 0) {
      double lo = bp.beta_min, hi = bp.beta_max;
      if (hi < 0.0) {
        if (!(opt.tau_ms > 0.0)) sm.status = RW_ERR_VALIDATION;
        hi = __ddiv_rn(10.0, opt.tau_ms);
      }
      double eps = bp.epsilon;
      if (eps < 0.0) eps = __ddiv_rn(__dsub_rn(hi, lo), 1024.0);
      if (!(lo >= 0.0) || !(lo < hi)) sm.status = RW_ERR_VALIDATION;
      if (!(eps > 0.0)) sm.status = RW_ERR_VALIDATION;
      sm.lo = lo;
      sm.hi = hi;
      sm.eps = eps;
      sm.b_feasible = 0;
      sm.b_has = 0;
      sm.n_trace = 0;
      sm.beta_star = 0.0;
      sm.bst_score = sm.bst_lat = sm.bst_obj = 0.0;
      sm.bst_iters = sm.bst_conv = 0;
      sm.bst_oor = 0;
      for (int i = 0; i < m; ++i) {
        sm.w_star[i] = 0.0;
        sm.bst_w[i] = 0.0;
      }
      sm.tr_best_lat = 0.0;
      sm.tr_best_score = 0.0;
    }
    __syncthreads();
    if (sm.status) return;
    while (__dsub_rn(sm.hi, sm.lo) > sm.eps) {
      const double mid = __dmul_rn(0.5, __dadd_rn(sm.lo, sm.hi));
      optimize_fractions(mid, opt, bp.pga);
      if (sm.status) return;
      if (tid == 0) {
        bool ok = sm.fr_lat <= opt.tau_ms && sm.fr_oor == 0u;
        if (trace && sm.n_trace < trace_cap) {
          trace[sm.n_trace].beta = mid;
          trace[sm.n_trace].score = sm.fr_score;
          trace[sm.n_trace].latency_ms = sm.fr_lat;
          trace[sm.n_trace].feasible = ok ? 1 : 0;
          trace[sm.n_trace].pad_ = 0;
        }
        if (sm.n_trace == 0 || sm.fr_lat < sm.tr_best_lat) {  // setup_search.cpp:200-202
          sm.tr_best_lat = sm.fr_lat;
          sm.tr_best_score = sm.fr_score;
        }
        sm.n_trace++;
        if (ok) {
          sm.b_feasible = 1;
          sm.b_has = 1;
          sm.beta_star = mid;
          for (int i = 0; i < m; ++i) {
            sm.w_star[i] = sm.fr_w[i];
            sm.bst_w[i] = sm.fr_w[i];
          }
          sm.bst_score = sm.fr_score;
          sm.bst_lat = sm.fr_lat;
          sm.bst_obj = sm.fr_obj;
          sm.bst_iters = sm.fr_iters;
          sm.bst_conv = sm.fr_conv;
          sm.bst_oor = sm.fr_oor;
          sm.hi = mid;
        } else {
          sm.lo = mid;
        }
      }
      __syncthreads();
    }
  }

  __device__ void reset_counters() {
    if (tid == 0) {
      sm.status = 0;
      sm.eval_passes = 0;
      sm.polish_passes = 0;
      sm.repair_calls = 0;
      for (int i = 0; i < MM; ++i) sm.zero[i] = 0.0;
    }
    __syncthreads();
  }

  // ---- select_setup's evaluate (setup_search.cpp:187-211) -> one record ---------------
  __device__ void evaluate_setup(long long k, rw_setup_record* rec) {
    pidx = jb.prof_idx + (size_t)k * m;
    reset_counters();
    optimize_beta(jb.opt, jb.bp, nullptr, 0);
    int bisect = sm.n_trace;
    double e_score = 0.0, e_lat = 0.0;
    if (!sm.status && !sm.b_feasible) {
      if (sm.n_trace > 0) {
        e_score = sm.tr_best_score;
        e_lat = sm.tr_best_lat;
      } else {  // degenerate bracket: evaluate the top penalty once
        double beta_hi = jb.bp.beta_max;
        if (beta_hi < 0.0) beta_hi = __ddiv_rn(10.0, jb.opt.tau_ms);
        optimize_fractions(beta_hi, jb.opt, jb.bp.pga);
        e_score = sm.fr_score;
        e_lat = sm.fr_lat;
      }
    }
    __syncthreads();
    if (tid == 0) {
      rec->setup_id = jb.setup_ids ? jb.setup_ids[k] : k;
      rec->status = sm.status;
      rec->feasible = (!sm.status && sm.b_feasible) ? 1 : 0;
      rec->score = sm.b_feasible ? sm.bst_score : e_score;
      rec->latency_ms = sm.b_feasible ? sm.bst_lat : e_lat;
      rec->beta = sm.b_feasible ? sm.beta_star : 0.0;
      for (int i = 0; i < RW_MAX_MODELS; ++i)
        rec->w[i] = (sm.b_feasible && i < m) ? sm.bst_w[i] : 0.0;
      rec->out_of_range = sm.b_feasible ? sm.bst_oor : 0u;
      rec->bisect_steps = bisect;
      rec->eval_passes = sm.eval_passes;
      rec->polish_passes = sm.polish_passes;
      rec->repair_calls = sm.repair_calls;
    }
    __syncthreads();
  }
};

// ---------------------------------------------------------------------------------------
template <int MM, int L, int T>
__global__ void __launch_bounds__(T) solver_kernel(const Job jb) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  using SM = Smem<MM, L, T>;
  SM& sm = *reinterpret_cast<SM*>(smem_raw);
  const int slot = blockIdx.x;
  uint8_t* mo = jb.ws_model_of + (size_t)slot * jb.n;
  unsigned long long* keys = reinterpret_cast<unsigned long long*>(jb.ws_keys) + (size_t)slot * jb.n;
  Solver<MM, L, T> s(sm, jb, mo, keys);
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
}

}  // namespace rw
