// K2 launcher: shared-memory tiled kernel (reference tile_accumulate +
// finalize_block over LayoutStore.load_tile, kernels.py:70-108,
// layouts.py:215-229, strategies.py:169-199).
//
// Grid shaping.  Every query costs the same n pairs, so the kernel is balanced
// statically: the query range is cut into grid_x = waves * slots blocks
// (slots = SMs x resident CTAs per SM) and each block gets only as many
// consumer warps as its share needs, so the last wave is not a partial one.
// FAST runs with too few queries to fill the slots also split the data range
// (blockIdx.y) and fold the per-split partials in split order (k_combine).
#include <algorithm>

#include "idw_kernels.cuh"
#include "idw_launch.h"

namespace idw {

template <typename T, int MODE>
struct TiledCfg;
// fp32: 1024-point tiles; FAST packs 8 queries (4 pairs) per thread.
template <>
struct TiledCfg<float, FAST> {
  static constexpr int Q = 8, TILE = 1024, NC_MAX = 256;
};
template <>
struct TiledCfg<float, EXACT> {
  static constexpr int Q = 4, TILE = 1024, NC_MAX = 256;
};
template <>
struct TiledCfg<double, FAST> {
  static constexpr int Q = 4, TILE = 512, NC_MAX = 256;
};
template <>
struct TiledCfg<double, EXACT> {
  static constexpr int Q = 2, TILE = 512, NC_MAX = 256;
};

static inline long long cdiv(long long a, long long b) { return (a + b - 1) / b; }

int launch_tiled(Launch &L) {
  return with_layout(L, [&](auto KC, auto tv) -> int {
    using T = decltype(tv);
    constexpr int K = decltype(KC)::value;
    return with_arith(L, [&](auto MC, auto PC, auto EC) -> int {
      constexpr int MODE = decltype(MC)::value;
      constexpr bool P2 = decltype(PC)::value, EPS = decltype(EC)::value;
      using C = TiledCfg<T, MODE>;
      constexpr int Q = C::Q, TILE = C::TILE;
      auto kern = k_tiled<K, T, MODE, P2, EPS, Q, TILE>;
      const int smem = tiled_smem_bytes<K, T, TILE>();
      IDW_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      int occ = 0;
      IDW_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, C::NC_MAX + 32, smem));
      if (occ < 1) occ = 1;
      const long long slots = (long long)L.sms * occ;
      const long long ntiles = cdiv(L.n, TILE);
      const long long cap = (long long)C::NC_MAX * Q;
      long long blocks = cdiv(L.m, cap);
      long long splits = 1;
      if (MODE == FAST) {
        if (L.splits > 0) {
          splits = L.splits;
        } else if (blocks < slots) {
          splits = std::max<long long>(1, slots / blocks);
        }
        splits = std::min(splits, ntiles);
      }
      long long qpc;
      if (blocks >= slots) {
        const long long waves = cdiv(blocks, slots);
        blocks = waves * slots;
        qpc = cdiv(L.m, blocks);
        qpc = cdiv(qpc, Q) * Q;
      } else {
        qpc = std::min<long long>(cap, cdiv(L.m, Q) * Q);
      }
      blocks = cdiv(L.m, qpc);
      int nc = (int)cdiv(cdiv(qpc, Q), 32) * 32;
      const long long tps = cdiv(ntiles, splits);
      splits = cdiv(ntiles, tps);

      SplitOut<T> so{nullptr, nullptr, nullptr, nullptr, nullptr};
      void *ws = nullptr;
      if (splits > 1) {
        const size_t per = (size_t)splits * (size_t)L.m;
        IDW_CK(cudaMallocAsync(&ws, per * (4 * sizeof(T) + 1), L.st));
        T *base = (T *)ws;
        so.shi = base;
        so.slo = base + per;
        so.zhi = base + 2 * per;
        so.zlo = base + 3 * per;
        so.flag = (unsigned char *)(base + 4 * per);
      }
      dim3 grid((unsigned)blocks, (unsigned)splits);
      kern<<<grid, nc + 32, smem, L.st>>>(L.g, L.n, (const T *)L.qx, (const T *)L.qy, L.m, qpc, tps,
                                          make_scal<T>(L), (T *)L.out, L.flags, so);
      IDW_CK_LAUNCH();
      ++L.launches;
      if (splits > 1) {
        if constexpr (MODE == FAST) {
          k_combine<T><<<(unsigned)cdiv(L.m, 256), 256, 0, L.st>>>(L.m, (int)splits, so, (T)L.eps_flag,
                                                                   (T *)L.out, L.flags);
          IDW_CK_LAUNCH();
          ++L.launches;
        }
        IDW_CK(cudaFreeAsync(ws, L.st));
      }
      return 0;
    });
  });
}

}  // namespace idw
