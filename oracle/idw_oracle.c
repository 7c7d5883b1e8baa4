/*
 * idw_oracle.c -- CPU restatement of the reference's IDW loops.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path links or calls this
 * file: it is the parity checker used by tests/, __graft_entry__.smoke() and
 * the cpu_baseline / --impl reference legs of bench.py.
 *
 * The reference (idwlayout 0.1.0) is Python whose loops numba compiles to
 * scalar IEEE x86 (vdivss/vdivsd, vmuls*, vadds*; no FMA contraction, no SIMD
 * -- SURVEY.md section 0).  Compiled with -ffp-contract=off and no fast-math,
 * these C loops perform the same IEEE operations in the same order, so p = 2
 * results are bit-identical; general p goes through libm pow/powf exactly as
 * numba's llvm.pow lowering does.  The restatement is pinned against outputs
 * of the reference itself (tests/golden/, made by tests/golden/make_golden.py).
 *
 * Each function cites the reference loop it restates (paths relative to
 * /root/reference/pkg/src/idwlayout).  Component pointers are strided views:
 * element i of x lives at xs[i * sx] (layouts.py:161-170 _make_views).
 */
#define _GNU_SOURCE
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <stdatomic.h>
#include <unistd.h>

#define NO_HIT ((int64_t)1 << 62) /* kernels.py:17 */

static int64_t next_pow2(int64_t n) { /* kernels.py:27-31 */
  int64_t p = 1;
  while (p < n) p *= 2;
  return p;
}

static inline float pw_f32(float d2, float wexp) { return powf(d2, wexp); }
static inline double pw_f64(double d2, double wexp) { return pow(d2, wexp); }

/* ---- kernels.predict_block (kernels.py:34-67) ------------------------- */
#define DEF_PREDICT(T, SFX)                                                                          \
  void oracle_predict_##SFX(const T *qx, const T *qy, int64_t q0, int64_t q1, const T *xs, int64_t sx, \
                            const T *ys, int64_t sy, const T *zs, int64_t sz, int64_t n, int fast,     \
                            T wexp, T eps, T *out) {                                                   \
    const T zero = (T)0, one = (T)1;                                                                   \
    for (int64_t q = q0; q < q1; ++q) {                                                                \
      const T px = qx[q], py = qy[q];                                                                  \
      T sw = zero, swz = zero, hz = zero;                                                              \
      int64_t hit = NO_HIT;                                                                            \
      for (int64_t i = 0; i < n; ++i) {                                                                \
        const T dx = px - xs[i * sx];                                                                  \
        const T dy = py - ys[i * sy];                                                                  \
        const T d2 = dx * dx + dy * dy;                                                                \
        if (d2 <= eps) {                                                                               \
          if (hit == NO_HIT) {                                                                         \
            hit = i;                                                                                   \
            hz = zs[i * sz];                                                                           \
          }                                                                                            \
        } else {                                                                                       \
          const T w = fast ? one / d2 : pw_##SFX(d2, wexp);                                            \
          sw = sw + w;                                                                                 \
          swz = swz + w * zs[i * sz];                                                                  \
        }                                                                                              \
      }                                                                                                \
      out[q] = hit != NO_HIT ? hz : swz / sw;                                                          \
    }                                                                                                  \
  }
DEF_PREDICT(float, f32)
DEF_PREDICT(double, f64)

/* ---- run_tiled: load_tile + tile_accumulate + finalize_block
 *      (strategies.py:188-196, layouts.py:215-229, kernels.py:70-108) ------ */
#define DEF_TILED(T, SFX)                                                                              \
  void oracle_tiled_##SFX(const T *qx, const T *qy, int64_t q0, int64_t q1, const T *xs, int64_t sx,     \
                          const T *ys, int64_t sy, const T *zs, int64_t sz, int64_t n, int64_t tile,     \
                          int fast, T wexp, T eps, T *out) {                                             \
    const T zero = (T)0, one = (T)1;                                                                     \
    T *tx = (T *)malloc(sizeof(T) * 3 * (size_t)tile), *ty = tx + tile, *tz = ty + tile;                 \
    int64_t m = q1 - q0;                                                                                 \
    T *sw = (T *)calloc((size_t)(m ? m : 1), sizeof(T)), *swz = (T *)calloc((size_t)(m ? m : 1), sizeof(T)); \
    T *hz = (T *)calloc((size_t)(m ? m : 1), sizeof(T));                                                 \
    int64_t *hit = (int64_t *)malloc(sizeof(int64_t) * (size_t)(m ? m : 1));                            \
    for (int64_t k = 0; k < m; ++k) hit[k] = NO_HIT;                                                     \
    for (int64_t lo = 0; lo < n; lo += tile) {                                                           \
      const int64_t hi = lo + tile < n ? lo + tile : n, cnt = hi - lo;                                   \
      for (int64_t i = 0; i < cnt; ++i) {                                                                \
        tx[i] = xs[(lo + i) * sx];                                                                       \
        ty[i] = ys[(lo + i) * sy];                                                                       \
        tz[i] = zs[(lo + i) * sz];                                                                       \
      }                                                                                                  \
      for (int64_t k = 0; k < m; ++k) {                                                                  \
        const T px = qx[q0 + k], py = qy[q0 + k];                                                        \
        T s = sw[k], sz2 = swz[k];                                                                       \
        for (int64_t i = 0; i < cnt; ++i) {                                                              \
          const T dx = px - tx[i], dy = py - ty[i];                                                      \
          const T d2 = dx * dx + dy * dy;                                                                \
          if (d2 <= eps) {                                                                               \
            if (hit[k] == NO_HIT) {                                                                      \
              hit[k] = lo + i;                                                                           \
              hz[k] = tz[i];                                                                             \
            }                                                                                            \
          } else {                                                                                       \
            const T w = fast ? one / d2 : pw_##SFX(d2, wexp);                                            \
            s = s + w;                                                                                   \
            sz2 = sz2 + w * tz[i];                                                                       \
          }                                                                                              \
        }                                                                                                \
        sw[k] = s;                                                                                       \
        swz[k] = sz2;                                                                                    \
      }                                                                                                  \
    }                                                                                                    \
    for (int64_t k = 0; k < m; ++k) out[q0 + k] = hit[k] != NO_HIT ? hz[k] : swz[k] / sw[k];             \
    (void)zero;                                                                                          \
    free(tx); free(sw); free(swz); free(hz); free(hit);                                                  \
  }
DEF_TILED(float, f32)
DEF_TILED(double, f64)

/* ---- kernels._tree_combine (kernels.py:111-133) ----------------------- */
#define DEF_TREE(T, SFX)                                                                             \
  void oracle_tree_##SFX(T *wp, T *wzp, int64_t *hitp, T *hzp, int64_t width) {                       \
    for (int64_t mm = width; mm > 1; mm /= 2) {                                                        \
      const int64_t half = mm / 2;                                                                     \
      for (int64_t j = 0; j < half; ++j) {                                                             \
        const int64_t a = 2 * j, b = a + 1;                                                            \
        wp[j] = wp[a] + wp[b];                                                                         \
        wzp[j] = wzp[a] + wzp[b];                                                                      \
        if (hitp[b] < hitp[a]) {                                                                       \
          hitp[j] = hitp[b];                                                                           \
          hzp[j] = hzp[b];                                                                             \
        } else {                                                                                       \
          hitp[j] = hitp[a];                                                                           \
          hzp[j] = hzp[a];                                                                             \
        }                                                                                              \
      }                                                                                                \
    }                                                                                                  \
  }
DEF_TREE(float, f32)
DEF_TREE(double, f64)

/* ---- kernels.nested_improved_block (kernels.py:136-185) ---------------- */
#define DEF_NEST_IMP(T, SFX)                                                                           \
  void oracle_nested_improved_##SFX(const T *qx, const T *qy, int64_t q0, int64_t q1, const T *xs,       \
                                    int64_t sx, const T *ys, int64_t sy, const T *zs, int64_t sz,        \
                                    int64_t n, int64_t group, int fast, T wexp, T eps, T *out) {         \
    const T zero = (T)0, one = (T)1;                                                                     \
    const int64_t p2 = next_pow2(group < 1 ? 1 : group);                                                 \
    T *wp = (T *)malloc(sizeof(T) * (size_t)p2), *wzp = (T *)malloc(sizeof(T) * (size_t)p2);             \
    T *hzp = (T *)malloc(sizeof(T) * (size_t)p2);                                                        \
    int64_t *hitp = (int64_t *)malloc(sizeof(int64_t) * (size_t)p2);                                     \
    const int64_t chunks = (n + group - 1) / group;                                                      \
    for (int64_t q = q0; q < q1; ++q) {                                                                  \
      for (int64_t t = 0; t < p2; ++t) {                                                                 \
        wp[t] = zero; wzp[t] = zero; hitp[t] = NO_HIT; hzp[t] = zero;                                    \
      }                                                                                                  \
      const T px = qx[q], py = qy[q];                                                                    \
      for (int64_t t = 0; t < group; ++t) {                                                              \
        T sw = zero, swz = zero, hz = zero;                                                              \
        int64_t hit = NO_HIT, k = t;                                                                     \
        for (int64_t c = 0; c < chunks; ++c, k += group) {                                               \
          if (k < n) {                                                                                   \
            const T dx = px - xs[k * sx], dy = py - ys[k * sy];                                          \
            const T d2 = dx * dx + dy * dy;                                                              \
            if (d2 <= eps) {                                                                             \
              if (hit == NO_HIT) {                                                                       \
                hit = k;                                                                                 \
                hz = zs[k * sz];                                                                         \
              }                                                                                          \
            } else {                                                                                     \
              const T w = fast ? one / d2 : pw_##SFX(d2, wexp);                                          \
              sw = sw + w;                                                                               \
              swz = swz + w * zs[k * sz];                                                                \
            }                                                                                            \
          }                                                                                              \
        }                                                                                                \
        wp[t] = sw; wzp[t] = swz; hitp[t] = hit; hzp[t] = hz;                                            \
      }                                                                                                  \
      oracle_tree_##SFX(wp, wzp, hitp, hzp, p2);                                                         \
      out[q] = hitp[0] != NO_HIT ? hzp[0] : wzp[0] / wp[0];                                              \
    }                                                                                                    \
    free(wp); free(wzp); free(hzp); free(hitp);                                                          \
  }
DEF_NEST_IMP(float, f32)
DEF_NEST_IMP(double, f64)

/* ---- kernels.nested_original_block (kernels.py:188-248) ---------------- */
#define DEF_NEST_ORIG(T, SFX)                                                                          \
  int64_t oracle_nested_original_##SFX(const T *qx, const T *qy, int64_t q0, int64_t q1, const T *xs,    \
                                       int64_t sx, const T *ys, int64_t sy, const T *zs, int64_t sz,     \
                                       int64_t n, int64_t group, int fast, T wexp, T eps, T *out) {      \
    const T zero = (T)0, one = (T)1;                                                                     \
    const int64_t p2 = next_pow2(group < 1 ? 1 : group), ngroups = (n + group - 1) / group;              \
    T *wp = (T *)malloc(sizeof(T) * (size_t)p2), *wzp = (T *)malloc(sizeof(T) * (size_t)p2);             \
    T *hzp = (T *)malloc(sizeof(T) * (size_t)p2);                                                        \
    int64_t *hitp = (int64_t *)malloc(sizeof(int64_t) * (size_t)p2), merges = 0;                         \
    for (int64_t q = q0; q < q1; ++q) {                                                                  \
      const T px = qx[q], py = qy[q];                                                                    \
      T ssw = zero, sswz = zero, shz = zero;                                                             \
      int64_t shit = NO_HIT;                                                                             \
      for (int64_t g = 0; g < ngroups; ++g) {                                                            \
        const int64_t base = g * group;                                                                  \
        const int64_t cnt = n - base > group ? group : n - base;                                         \
        for (int64_t t = 0; t < p2; ++t) {                                                               \
          wp[t] = zero; wzp[t] = zero; hitp[t] = NO_HIT; hzp[t] = zero;                                  \
          if (t < cnt) {                                                                                 \
            const int64_t i = base + t;                                                                  \
            const T dx = px - xs[i * sx], dy = py - ys[i * sy];                                          \
            const T d2 = dx * dx + dy * dy;                                                              \
            if (d2 <= eps) {                                                                             \
              hitp[t] = i;                                                                               \
              hzp[t] = zs[i * sz];                                                                       \
            } else {                                                                                     \
              const T w = fast ? one / d2 : pw_##SFX(d2, wexp);                                          \
              wp[t] = w;                                                                                 \
              wzp[t] = w * zs[i * sz];                                                                   \
            }                                                                                            \
          }                                                                                              \
        }                                                                                                \
        oracle_tree_##SFX(wp, wzp, hitp, hzp, p2);                                                       \
        ssw = ssw + wp[0];                                                                               \
        sswz = sswz + wzp[0];                                                                            \
        if (hitp[0] < shit) {                                                                            \
          shit = hitp[0];                                                                                \
          shz = hzp[0];                                                                                  \
        }                                                                                                \
        ++merges;                                                                                        \
      }                                                                                                  \
      out[q] = shit != NO_HIT ? shz : sswz / ssw;                                                        \
    }                                                                                                    \
    free(wp); free(wzp); free(hzp); free(hitp);                                                          \
    return merges;                                                                                       \
  }
DEF_NEST_ORIG(float, f32)
DEF_NEST_ORIG(double, f64)

/* ---- fp64 "fsum" truth (tests/oracle_idw.py:11-38 brute_idw) -----------
 * The run-precision inputs are widened to double; d2 and w = d2**(-p/2)
 * (1/d2 for p = 2) are evaluated in double; both sums are carried in
 * double-double (TwoSum), i.e. exact to ~2^-100 relative, which is what
 * math.fsum's exactly rounded sum buys the reference's own oracle.  Inputs
 * are passed as double arrays (already rounded to the run precision). */
static inline void dd_add(double *hi, double *lo, double b) {
  const double s = *hi + b, bb = s - *hi;
  const double e = (*hi - (s - bb)) + (b - bb);
  *hi = s;
  *lo += e;
}
void oracle_truth_f64(const double *qx, const double *qy, int64_t q0, int64_t q1, const double *xs,
                      const double *ys, const double *zs, int64_t n, double p, double eps, double *out) {
  for (int64_t q = q0; q < q1; ++q) {
    double swh = 0, swl = 0, szh = 0, szl = 0;
    int64_t hit = NO_HIT;
    for (int64_t i = 0; i < n; ++i) {
      const double dx = qx[q] - xs[i], dy = qy[q] - ys[i];
      const double d2 = dx * dx + dy * dy;
      if (d2 <= eps) {
        if (hit == NO_HIT) hit = i;
        continue;
      }
      const double w = p == 2.0 ? 1.0 / d2 : pow(d2, -p / 2.0);
      dd_add(&swh, &swl, w);
      dd_add(&szh, &szl, w * zs[i]);
    }
    out[q] = hit != NO_HIT ? zs[hit] : (szh + szl) / (swh + swl);
  }
}

/* ---- multi-threaded drivers (the CPU baseline legs of bench.py) ------
 * Dynamic 256-query blocks (64 for the nested variant, like _NESTED_BLOCK)
 * pulled by `threads` pthreads from an atomic counter, the analogue of
 * run_naive's ThreadPoolExecutor over _NAIVE_BLOCK blocks
 * (strategies.py:37-38,141-145,160-165).  Per-query results do not depend
 * on the thread count. */
typedef struct {
  int variant; /* 0 predict, 1 nested_improved, 2 truth */
  int dbl;
  const void *qx, *qy, *xs, *ys, *zs;
  int64_t m, sx, sy, sz, n, group, block;
  int fast;
  double wexp, eps, p;
  void *out;
  atomic_llong next;
} mt_job;

static void *mt_worker(void *arg) {
  mt_job *j = (mt_job *)arg;
  for (;;) {
    const int64_t b = atomic_fetch_add(&j->next, 1);
    const int64_t lo = b * j->block;
    if (lo >= j->m) break;
    const int64_t hi = lo + j->block < j->m ? lo + j->block : j->m;
    if (j->variant == 2) {
      oracle_truth_f64((const double *)j->qx, (const double *)j->qy, lo, hi, (const double *)j->xs,
                       (const double *)j->ys, (const double *)j->zs, j->n, j->p, j->eps, (double *)j->out);
    } else if (j->dbl) {
      if (j->variant == 0)
        oracle_predict_f64(j->qx, j->qy, lo, hi, j->xs, j->sx, j->ys, j->sy, j->zs, j->sz, j->n, j->fast,
                           j->wexp, j->eps, j->out);
      else
        oracle_nested_improved_f64(j->qx, j->qy, lo, hi, j->xs, j->sx, j->ys, j->sy, j->zs, j->sz, j->n,
                                   j->group, j->fast, j->wexp, j->eps, j->out);
    } else {
      if (j->variant == 0)
        oracle_predict_f32(j->qx, j->qy, lo, hi, j->xs, j->sx, j->ys, j->sy, j->zs, j->sz, j->n, j->fast,
                           (float)j->wexp, (float)j->eps, j->out);
      else
        oracle_nested_improved_f32(j->qx, j->qy, lo, hi, j->xs, j->sx, j->ys, j->sy, j->zs, j->sz, j->n,
                                   j->group, j->fast, (float)j->wexp, (float)j->eps, j->out);
    }
  }
  return NULL;
}

static void mt_run(mt_job *j, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 1024) threads = 1024;
  /* shrink blocks when m is small so every thread gets work (results do not
   * depend on the block size: each query is computed independently) */
  const int64_t fair = j->m / ((int64_t)threads * 8);
  if (fair < j->block) j->block = fair > 1 ? fair : 1;
  atomic_init(&j->next, 0);
  pthread_t tid[1024];
  int started = 0;
  for (int t = 1; t < threads; ++t)
    if (pthread_create(&tid[started], NULL, mt_worker, j) == 0) ++started;
  mt_worker(j);
  for (int t = 0; t < started; ++t) pthread_join(tid[t], NULL);
}

int oracle_max_threads(void) {
  long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n > 0 ? (int)n : 1;
}

/* run_naive over all m queries; wexp/eps are given in double and cast to the
 * run dtype exactly like kernels.scalar_args (kernels.py:20-24). */
void oracle_predict_mt(int dbl, const void *qx, const void *qy, int64_t m, const void *xs, int64_t sx,
                       const void *ys, int64_t sy, const void *zs, int64_t sz, int64_t n, int fast, double wexp,
                       double eps, void *out, int threads) {
  mt_job j = {0, dbl, qx, qy, xs, ys, zs, m, sx, sy, sz, n, 1, 256, fast, wexp, eps, 0.0, out, 0};
  mt_run(&j, threads);
}
void oracle_nested_improved_mt(int dbl, const void *qx, const void *qy, int64_t m, const void *xs, int64_t sx,
                               const void *ys, int64_t sy, const void *zs, int64_t sz, int64_t n, int64_t group,
                               int fast, double wexp, double eps, void *out, int threads) {
  mt_job j = {1, dbl, qx, qy, xs, ys, zs, m, sx, sy, sz, n, group, 64, fast, wexp, eps, 0.0, out, 0};
  mt_run(&j, threads);
}
void oracle_truth_mt_f64(const double *qx, const double *qy, int64_t m, const double *xs, const double *ys,
                         const double *zs, int64_t n, double p, double eps, double *out, int threads) {
  mt_job j = {2, 1, qx, qy, xs, ys, zs, m, 1, 1, 1, n, 1, 16, 0, 0.0, eps, p, out, 0};
  mt_run(&j, threads);
}
