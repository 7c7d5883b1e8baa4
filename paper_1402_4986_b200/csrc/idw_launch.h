// idw_launch.h -- host-side launch plumbing shared by the per-variant
// translation units (compiled in parallel) and the C-ABI shim.
#pragma once
#include <cuda_runtime.h>

#include <string>
#include <type_traits>

#include "../../include/idw_b200.h"
#include "idw_common.cuh"

namespace idw {

// Everything a variant launcher needs; all pointers are device pointers.
struct Launch {
  int kind = 0, prec = 0, mode = 0, variant = 0;
  bool p2 = true, epsp = false;
  Bufs g{};
  long long n = 0;
  const void *qx = nullptr, *qy = nullptr;
  long long m = 0;
  double eps = 0.0, wexp = -1.0, eps_flag = 0.0;
  long long G = 1024, T = 1024;
  int splits = 0;
  void *out = nullptr;
  unsigned char *flags = nullptr;  // FAST: m bytes of screen flags
  unsigned long long *nfixed = nullptr;
  cudaStream_t st = nullptr;
  int dev = 0, sms = 148;
  int launches = 0;
};

void set_error(const std::string &msg);

#define IDW_CK(call)                                                                    \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess) {                                                            \
      ::idw::set_error(std::string(#call) + ": " + cudaGetErrorString(e_));             \
      return (int)IDW_E_CUDA;                                                           \
    }                                                                                   \
  } while (0)

#define IDW_CK_LAUNCH()                                                                 \
  do {                                                                                  \
    cudaError_t e_ = cudaGetLastError();                                                \
    if (e_ != cudaSuccess) {                                                            \
      ::idw::set_error(std::string("kernel launch: ") + cudaGetErrorString(e_));        \
      return (int)IDW_E_CUDA;                                                           \
    }                                                                                   \
  } while (0)

// Stream-ordered scratch released on scope exit (early error returns included).
struct StreamFree {
  void *p = nullptr;
  cudaStream_t st = nullptr;
  StreamFree() = default;
  StreamFree(const StreamFree &) = delete;
  StreamFree &operator=(const StreamFree &) = delete;
  ~StreamFree() {
    if (p) cudaFreeAsync(p, st);
  }
};

template <int V>
using IC = std::integral_constant<int, V>;
template <bool V>
using BC = std::integral_constant<bool, V>;

// Visit the legal (layout, dtype) pair of a launch (layouts.legal_pairs,
// layouts.py:317-319): SoAoS and Hybrid exist only in double precision.
template <class F>
int with_layout(const Launch &L, F &&f) {
  if (L.prec == IDW_SINGLE) {
    switch (L.kind) {
      case SOA: return f(IC<SOA>{}, float{});
      case AOS: return f(IC<AOS>{}, float{});
      case AOAS: return f(IC<AOAS>{}, float{});
      default: set_error("layout requires double precision"); return IDW_E_UNSUPPORTED;
    }
  }
  switch (L.kind) {
    case SOA: return f(IC<SOA>{}, double{});
    case AOS: return f(IC<AOS>{}, double{});
    case AOAS: return f(IC<AOAS>{}, double{});
    case SOAOS: return f(IC<SOAOS>{}, double{});
    case HYBRID: return f(IC<HYBRID>{}, double{});
    default: set_error("unknown layout kind"); return IDW_E_ARG;
  }
}

// Visit (mode, p == 2, zero_eps > 0).  EXACT with zero_eps > 0 keeps the
// per-pair coincidence bookkeeping; with zero_eps == 0 naive/tiled screen.
template <class F>
int with_arith(const Launch &L, F &&f) {
  if (L.mode == EXACT) {
    if (L.p2) return L.epsp ? f(IC<EXACT>{}, BC<true>{}, BC<true>{}) : f(IC<EXACT>{}, BC<true>{}, BC<false>{});
    return L.epsp ? f(IC<EXACT>{}, BC<false>{}, BC<true>{}) : f(IC<EXACT>{}, BC<false>{}, BC<false>{});
  }
  if (L.p2) return L.epsp ? f(IC<FAST>{}, BC<true>{}, BC<true>{}) : f(IC<FAST>{}, BC<true>{}, BC<false>{});
  return L.epsp ? f(IC<FAST>{}, BC<false>{}, BC<true>{}) : f(IC<FAST>{}, BC<false>{}, BC<false>{});
}

template <typename T>
inline Scal<T> make_scal(const Launch &L) {
  Scal<T> s;
  s.eps = (T)L.eps;
  s.wexp = (T)L.wexp;
  s.eps_flag = (T)L.eps_flag;
  const double twop = -4.0 * L.wexp;  // 2p (wexp = -p/2)
  s.jq = (!L.p2 && twop == (double)(long long)twop && twop >= 1.0 && twop <= 64.0) ? (int)twop : 0;
  return s;
}

// cudaFuncSetAttribute(max dynamic smem) + resident CTAs per SM for `kern`
// at (threads, smem), done once per (kernel, device) and cached: both calls
// cost host microseconds that small launches cannot hide.
int kernel_occupancy(const void *kern, int dev, int threads, int smem, int *occ);

// Per-variant launchers (one translation unit each).
int launch_naive(Launch &L);
int launch_tiled(Launch &L);
int launch_nested(Launch &L);
int launch_nested_orig(Launch &L);
int launch_fixup(Launch &L);

// Device-side layout packers/converters (idw_layout_dev.cu).
int pack_device(const double *x, const double *y, const double *z, long long n, int kind, int prec,
                unsigned char *const *dst, cudaStream_t st, int sms);
int convert_device(const unsigned char *const *src, int kin, unsigned char *const *dst, int kout, int prec,
                   long long n, cudaStream_t st, int sms);

// (m, 2) float64 query pairs -> qx, qy in the run dtype + non-finite flag.
int split_queries(const double *xy, long long m, int prec, void *qx, void *qy, unsigned int *bad, cudaStream_t st,
                  int sms);

// Does this launch write screen flags and need the fix-up pass?
inline bool needs_fixup(const Launch &L) {
  if (L.variant == IDW_NESTED_ORIGINAL) return false;
  if (L.mode == FAST) return true;
  return !L.epsp && L.variant != IDW_NESTED_ORIGINAL;  // screened EXACT
}

}  // namespace idw
