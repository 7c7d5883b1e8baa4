// Device-side layout packers and converters (the "layout packers/converters"
// subsystem of the north star), byte-identical to the reference's host code:
//   k_pack     <- LayoutStore.from_arrays  (layouts.py:172-186): fp64 x, y, z
//                 cast round-to-nearest to the run dtype (numpy astype) and
//                 written in the shape table's strides; pads written as zero
//   k_convert  <- LayoutStore.convert      (layouts.py:251-255): value copy
//                 between two layouts of the same precision
// One thread per point (grid-stride); each kernel is a single HBM pass.
#include <algorithm>

#include "idw_kernels.cuh"
#include "idw_launch.h"

namespace idw {

struct WBufs {
  unsigned char *b[3];
};

template <int K, typename T>
struct GStore;
template <typename T>
struct GStore<SOA, T> {
  static __device__ __forceinline__ void put(const WBufs &w, long long i, T x, T y, T z) {
    reinterpret_cast<T *>(w.b[0])[i] = x;
    reinterpret_cast<T *>(w.b[1])[i] = y;
    reinterpret_cast<T *>(w.b[2])[i] = z;
  }
};
template <typename T>
struct GStore<AOS, T> {
  static __device__ __forceinline__ void put(const WBufs &w, long long i, T x, T y, T z) {
    T *r = reinterpret_cast<T *>(w.b[0]) + 3 * i;
    r[0] = x;
    r[1] = y;
    r[2] = z;
  }
};
template <>
struct GStore<AOAS, float> {
  static __device__ __forceinline__ void put(const WBufs &w, long long i, float x, float y, float z) {
    reinterpret_cast<float4 *>(w.b[0])[i] = make_float4(x, y, z, 0.f);
  }
};
template <>
struct GStore<AOAS, double> {
  static __device__ __forceinline__ void put(const WBufs &w, long long i, double x, double y, double z) {
    double2 *r = reinterpret_cast<double2 *>(w.b[0]) + 2 * i;
    r[0] = make_double2(x, y);
    r[1] = make_double2(z, 0.0);
  }
};
template <>
struct GStore<SOAOS, double> {
  static __device__ __forceinline__ void put(const WBufs &w, long long i, double x, double y, double z) {
    reinterpret_cast<double2 *>(w.b[0])[i] = make_double2(x, y);
    reinterpret_cast<double2 *>(w.b[1])[i] = make_double2(z, 0.0);
  }
};
template <>
struct GStore<HYBRID, double> {
  static __device__ __forceinline__ void put(const WBufs &w, long long i, double x, double y, double z) {
    reinterpret_cast<double2 *>(w.b[0])[i] = make_double2(x, y);
    reinterpret_cast<double *>(w.b[1])[i] = z;
  }
};

template <int K, typename T>
__global__ void __launch_bounds__(256) k_pack(const double *__restrict__ x, const double *__restrict__ y,
                                              const double *__restrict__ z, long long n, WBufs w) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    GStore<K, T>::put(w, i, (T)x[i], (T)y[i], (T)z[i]);  // (float)double is RN == numpy astype
}

template <int KI, int KO, typename T>
__global__ void __launch_bounds__(256) k_convert(Bufs in, long long n, WBufs w) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    T x, y, z;
    GFetch<KI, T>::get(in, i, x, y, z);
    GStore<KO, T>::put(w, i, x, y, z);
  }
}

// Record layouts whose per-thread stores are not one aligned vector per point
// (AoS: 12/24-byte records written as 3 scalars; fp64 AoaS: two double2 at a
// 32-byte stride) are written through shared memory: each thread builds its
// record in a tile image, then the block streams the image out with 16-byte
// stores, contiguous across the warp.  Byte-identical output (the image holds
// the same bytes, pads included); measured 0.75-0.82 -> see tools/layout_bench.py.
constexpr int STAGE_PTS = 256;
template <int KO, typename T>
constexpr bool staged_out() {
  return KO == AOS || (KO == AOAS && sizeof(T) == 8);
}
template <int KO, typename T>
__device__ __forceinline__ void flush_tile(const WBufs &w, long long base, int cnt, unsigned char *img) {
  using LT = LayoutTraits<KO, T>;
  static_assert(LT::nbuf == 1, "staged layouts have one buffer");
  constexpr int bpp = LT::bpp(0);
  const int bytes = cnt * bpp;
  unsigned char *dst = w.b[0] + base * bpp;  // base * bpp is 16-B aligned (STAGE_PTS * bpp is)
  const int v16 = bytes >> 4;
  for (int k = threadIdx.x; k < v16; k += blockDim.x)
    reinterpret_cast<uint4 *>(dst)[k] = reinterpret_cast<const uint4 *>(img)[k];
  for (int k = (v16 << 4) + threadIdx.x; k < bytes; k += blockDim.x) dst[k] = img[k];
}

template <int K, typename T>
__global__ void __launch_bounds__(STAGE_PTS) k_pack_staged(const double *__restrict__ x, const double *__restrict__ y,
                                                          const double *__restrict__ z, long long n, WBufs w) {
  __shared__ __align__(16) unsigned char img[STAGE_PTS * LayoutTraits<K, T>::bpp(0)];
  const WBufs sw{{img, nullptr, nullptr}};
  for (long long base = blockIdx.x * (long long)STAGE_PTS; base < n; base += (long long)gridDim.x * STAGE_PTS) {
    const int cnt = (int)(n - base < STAGE_PTS ? n - base : STAGE_PTS);
    const long long i = base + threadIdx.x;
    if ((int)threadIdx.x < cnt) GStore<K, T>::put(sw, threadIdx.x, (T)x[i], (T)y[i], (T)z[i]);
    __syncthreads();
    flush_tile<K, T>(w, base, cnt, img);
    __syncthreads();
  }
}

template <int KI, int KO, typename T>
__global__ void __launch_bounds__(STAGE_PTS) k_convert_staged(Bufs in, long long n, WBufs w) {
  __shared__ __align__(16) unsigned char img[STAGE_PTS * LayoutTraits<KO, T>::bpp(0)];
  const WBufs sw{{img, nullptr, nullptr}};
  for (long long base = blockIdx.x * (long long)STAGE_PTS; base < n; base += (long long)gridDim.x * STAGE_PTS) {
    const int cnt = (int)(n - base < STAGE_PTS ? n - base : STAGE_PTS);
    if ((int)threadIdx.x < cnt) {
      T x, y, z;
      GFetch<KI, T>::get(in, base + threadIdx.x, x, y, z);
      GStore<KO, T>::put(sw, threadIdx.x, x, y, z);
    }
    __syncthreads();
    flush_tile<KO, T>(w, base, cnt, img);
    __syncthreads();
  }
}

static int grid_for(long long n, int sms) {
  return (int)std::max<long long>(1, std::min<long long>((n + 255) / 256, (long long)sms * 16));
}

// Visit the legal (layout, dtype) of a (kind, prec) pair.
template <class F>
static int visit_kind(int kind, int prec, F &&f) {
  Launch L;
  L.kind = kind;
  L.prec = prec;
  return with_layout(L, std::forward<F>(f));
}

int pack_device(const double *x, const double *y, const double *z, long long n, int kind, int prec,
                unsigned char *const *dst, cudaStream_t st, int sms) {
  WBufs w{{dst[0], dst[1], dst[2]}};
  return visit_kind(kind, prec, [&](auto KC, auto tv) -> int {
    using T = decltype(tv);
    constexpr int K = decltype(KC)::value;
    bool done = false;
    if constexpr (staged_out<K, T>()) {
      if (((uintptr_t)w.b[0] & 15) == 0) {  // 16-byte stores need an aligned buffer
        k_pack_staged<K, T><<<grid_for(n, sms), STAGE_PTS, 0, st>>>(x, y, z, n, w);
        done = true;
      }
    }
    if (!done) k_pack<K, T><<<grid_for(n, sms), 256, 0, st>>>(x, y, z, n, w);
    IDW_CK_LAUNCH();
    return 0;
  });
}

int convert_device(const unsigned char *const *src, int kin, unsigned char *const *dst, int kout, int prec,
                   long long n, cudaStream_t st, int sms) {
  Bufs in{{src[0], src[1], src[2]}};
  WBufs w{{dst[0], dst[1], dst[2]}};
  return visit_kind(kin, prec, [&](auto KIC, auto tv) -> int {
    using T = decltype(tv);
    constexpr int KI = decltype(KIC)::value;
    return visit_kind(kout, prec, [&](auto KOC, auto tv2) -> int {
      constexpr int KO = decltype(KOC)::value;
      if constexpr (std::is_same<T, decltype(tv2)>::value) {
        bool done = false;
        if constexpr (staged_out<KO, T>()) {
          if (((uintptr_t)w.b[0] & 15) == 0) {
            k_convert_staged<KI, KO, T><<<grid_for(n, sms), STAGE_PTS, 0, st>>>(in, n, w);
            done = true;
          }
        }
        if (!done) k_convert<KI, KO, T><<<grid_for(n, sms), 256, 0, st>>>(in, n, w);
        IDW_CK_LAUNCH();
        return 0;
      } else {
        return (int)IDW_E_UNSUPPORTED;
      }
    });
  });
}

// strategies._prepare on the device (strategies.py:125-134): the reference's
// (m, 2) float64 query array -> contiguous qx, qy in the run dtype (cast
// round-to-nearest, like numpy astype), with core.ensure_finite's test
// (core.py:113-116) folded into one flag word.
template <typename T>
__global__ void __launch_bounds__(256) k_split_queries(const double2 *__restrict__ xy, long long m,
                                                      T *__restrict__ qx, T *__restrict__ qy,
                                                      unsigned int *__restrict__ bad) {
  bool nf = false;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x) {
    const double2 v = xy[i];
    nf |= !isfinite(v.x) || !isfinite(v.y);
    qx[i] = (T)v.x;
    qy[i] = (T)v.y;
  }
  if (__any_sync(0xffffffffu, nf) && (threadIdx.x & 31) == 0) atomicOr(bad, 1u);
}

int split_queries(const double *xy, long long m, int prec, void *qx, void *qy, unsigned int *bad, cudaStream_t st,
                  int sms) {
  const double2 *src = reinterpret_cast<const double2 *>(xy);
  if (prec == IDW_SINGLE)
    k_split_queries<float><<<grid_for(m, sms), 256, 0, st>>>(src, m, (float *)qx, (float *)qy, bad);
  else
    k_split_queries<double><<<grid_for(m, sms), 256, 0, st>>>(src, m, (double *)qx, (double *)qy, bad);
  IDW_CK_LAUNCH();
  return 0;
}

}  // namespace idw
