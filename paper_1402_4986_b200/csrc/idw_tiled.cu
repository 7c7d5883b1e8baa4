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
#include <cstdlib>

#include "idw_kernels.cuh"
#include "idw_launch.h"

namespace idw {

template <typename T, int MODE>
struct TiledCfg;
// fp32: 256-point warp tiles; FAST packs 8 queries (4 pairs) per thread.
template <>
struct TiledCfg<float, FAST> {
  static constexpr int Q = 8, TILE = 256, NC_MAX = 256;
};
template <>
struct TiledCfg<float, EXACT> {
  static constexpr int Q = 4, TILE = 256, NC_MAX = 256;
};
template <>
struct TiledCfg<double, FAST> {
  static constexpr int Q = 4, TILE = 128, NC_MAX = 256;
};
template <>
struct TiledCfg<double, EXACT> {
  static constexpr int Q = 2, TILE = 128, NC_MAX = 256;
};

static inline long long cdiv(long long a, long long b) { return (a + b - 1) / b; }

// Choose (query block size, data splits) so that blocks x splits fills the
// resident slots in whole waves: every CTA costs qpc x tiles_per_split pair
// units, and the search minimises waves x that cost (ties -> fewer splits).
// Query blocks keep >= 4 warps busy unless m itself is smaller.
struct Shape {
  long long qpc, blocks, splits, tps;
};
static Shape shape_grid(long long m, long long ntiles, long long slots, int Q, int nc_max, bool allow_split,
                        int forced_splits, long long sms) {
  const long long cap = (long long)nc_max * Q;
  (void)sms;  // full blocks on fewer SMs measured faster than thin blocks on all
              // SMs for EXACT (C2: 2120 vs 1978 GPairs/s)
  const long long min_q = std::min<long long>(cap / 2, cdiv(m, Q) * Q);
  Shape best{0, 0, 0, 0};
  double best_cost = 0;
  const long long smax = allow_split ? std::min<long long>(ntiles, 256) : 1;
  for (long long S = 1; S <= smax; ++S) {
    if (forced_splits > 0 && S != std::min<long long>(forced_splits, ntiles)) continue;
    const long long tps = cdiv(ntiles, S);
    const long long splits = cdiv(ntiles, tps);
    for (long long W = 1; W <= 64; ++W) {
      long long blocks = std::max<long long>(1, (W * slots) / splits);
      long long qpc = cdiv(cdiv(m, blocks), Q) * Q;
      if (qpc > cap) continue;  // too few blocks for this many waves
      if (qpc < min_q) break;   // more waves only shrink blocks further
      blocks = cdiv(m, qpc);
      const long long waves = cdiv(blocks * splits, slots);
      // a CTA runs whole warps: charge the query slots its warps hold
      const long long qslots = cdiv(qpc, (long long)Q * 32) * Q * 32;
      const double cost = (double)waves * (double)qslots * (double)tps;
      if (best.qpc == 0 || cost < best_cost * 0.999) {
        best = {qpc, blocks, splits, tps};
        best_cost = cost;
      }
      break;  // smallest feasible W for this S is the one to take
    }
  }
  if (best.qpc == 0) {  // fall back: full blocks, no split
    const long long qpc = std::min<long long>(cap, cdiv(m, Q) * Q);
    best = {qpc, cdiv(m, qpc), 1, ntiles};
  }
  return best;
}

int launch_tiled(Launch &L) {
  return with_layout(L, [&](auto KC, auto tv) -> int {
    using T = decltype(tv);
    constexpr int K = decltype(KC)::value;
    return with_arith(L, [&](auto MC, auto PC, auto EC) -> int {
      constexpr int MODE = decltype(MC)::value;
      constexpr bool P2 = decltype(PC)::value, EPS = decltype(EC)::value;
      using C = TiledCfg<T, MODE>;
      auto run_q = [&](auto QC) -> int {
      constexpr int Q = decltype(QC)::value, TILE = C::TILE;
      constexpr int RING = tiled_ring_bytes<K, T, TILE>();
      auto kern = k_tiled<K, T, MODE, P2, EPS, Q, TILE>;
      bool prod_used = false;
      if constexpr (std::is_same<T, float>::value && MODE == FAST && P2 && !EPS) {
        // One of the four packed query pairs per point shares a reciprocal
        // (measured on C3: 0 -> 4196, 1 -> 4546, 2 -> 4533 GPairs/s; the mix of
        // MUFU and FMA-pipe work is best balanced at 1).  IDW_PROD overrides.
        static const int prod = [] { const char *e = getenv("IDW_PROD"); return e ? atoi(e) : 1; }();
        if (prod == 1) kern = k_tiled<K, T, MODE, P2, EPS, Q, TILE, 1>;
        if (prod == 2) kern = k_tiled<K, T, MODE, P2, EPS, Q, TILE, 2>;
        prod_used = prod == 1 || prod == 2;
      }
      if constexpr (sizeof(T) == 8 && MODE == FAST && !P2) {
        // compile-time powers for the common half-integer p (p = 3: jq 6, p = 3.5: jq 7)
        const int jq = make_scal<T>(L).jq;
        if (jq == 7) kern = k_tiled<K, T, MODE, P2, EPS, Q, TILE, 0, 7>;
        if (jq == 6) kern = k_tiled<K, T, MODE, P2, EPS, Q, TILE, 0, 6>;
      }
      if constexpr (sizeof(T) == 4 && MODE == FAST && !P2 && Q % 2 == 0) {
        // integer p = 1, 3, 4: one MUFU per pair (rsqrt / rcp powers) instead of lg2 + ex2
        const int jq = make_scal<T>(L).jq;
        if (jq == 2) kern = k_tiled<K, T, MODE, P2, EPS, Q, TILE, 0, 2>;
        if (jq == 6) kern = k_tiled<K, T, MODE, P2, EPS, Q, TILE, 0, 6>;
        if (jq == 8) kern = k_tiled<K, T, MODE, P2, EPS, Q, TILE, 0, 8>;
      }
      const int smem_max = (C::NC_MAX / 32) * RING;
      int occ = 0;
      if (int rc = kernel_occupancy((const void *)kern, L.dev, C::NC_MAX, smem_max, &occ)) return rc;
      if (occ < 1) occ = 1;
      const long long slots = (long long)L.sms * occ;
      const long long ntiles = cdiv(L.n, TILE);
      const Shape sh = shape_grid(L.m, ntiles, slots, Q, C::NC_MAX, MODE == FAST, L.splits, L.sms);
      const int nc = (int)cdiv(cdiv(sh.qpc, Q), 32) * 32;
      const int smem = (nc / 32) * RING;

      SplitOut<T> so{nullptr, nullptr, nullptr, nullptr, nullptr};
      void *ws = nullptr;
      float4 *dbox = nullptr;
      StreamFree free_box, free_ws;  // scratch goes back to the pool on every exit
      using AccT = typename AccSelNT<T, MODE, P2, EPS, Q>::type;
      constexpr bool EXACT_FR = std::is_same<AccT, AccExactScr2<Q>>::value ||
                               std::is_same<AccT, AccExactScr<double, true, Q>>::value;
      if (prod_used || EXACT_FR) {  // data box for the fast-path guards
        if (int rc = launch_bbox<K, T>(L, &dbox)) return rc;
        free_box.p = dbox;
        free_box.st = L.st;
      }
      if (sh.splits > 1) {
        const size_t per = (size_t)sh.splits * (size_t)L.m;
        IDW_CK(cudaMallocAsync(&ws, per * (4 * sizeof(T) + 1), L.st));
        free_ws.p = ws;
        free_ws.st = L.st;
        T *base = (T *)ws;
        so.shi = base;
        so.slo = base + per;
        so.zhi = base + 2 * per;
        so.zlo = base + 3 * per;
        so.flag = (unsigned char *)(base + 4 * per);
      }
      dim3 grid((unsigned)sh.blocks, (unsigned)sh.splits);
      kern<<<grid, nc, smem, L.st>>>(L.g, L.n, (const T *)L.qx, (const T *)L.qy, L.m, sh.qpc, sh.tps,
                                     make_scal<T>(L), (T *)L.out, L.flags, so, dbox);
      IDW_CK_LAUNCH();
      ++L.launches;
      if (sh.splits > 1) {
        if constexpr (MODE == FAST) {
          k_combine<T><<<(unsigned)cdiv(L.m, 256), 256, 0, L.st>>>(L.m, (int)sh.splits, so, (T)L.eps_flag,
                                                                   (T *)L.out, L.flags);
          IDW_CK_LAUNCH();
          ++L.launches;
        }
      }
      return 0;
      };
      if constexpr (std::is_same<T, float>::value && MODE == EXACT && P2 && !EPS) {
        // EXACT keeps the strict data order, so it cannot split the data: when
        // Q = 4 blocks would not cover the SMs once, halve the queries per
        // thread so the same queries spread over all SMs (C2, 100K queries:
        // 100 CTAs on 148 SMs -> 296 CTAs).  Per-query arithmetic unchanged.
        // Measured at C2: SoA 2093 -> 2609, AoaS 2240 -> 2645 GPairs/s; AoS
        // 2211 -> 2023, so AoS keeps Q = 4.  IDW_EXACT_Q2=0 disables.
        static const int q2 = [] { const char *e = getenv("IDW_EXACT_Q2"); return e ? atoi(e) : 1; }();
        if (K != AOS && q2 && cdiv(L.m, (long long)C::Q * C::NC_MAX) < L.sms) return run_q(IC<2>{});
      }
      if constexpr (std::is_same<T, float>::value && MODE == FAST) {
        // Small jobs: Q = 4 doubles the threads of a query block -- more warps to
        // hide the ring fill and MUFU latency when each CTA sees only a few
        // tiles.  Measured (graph replays): 10K x 10K 1694 -> 1960, 100K x 10K
        // 3251 -> 3817, 100K x 100K even, 1M x 131K (an 8-GPU shard) 4729 ->
        // 4555 GPairs/s -- hence the ~4e9-pair cap.  IDW_FAST_Q4=0 disables.
        static const int q4 = [] { const char *e = getenv("IDW_FAST_Q4"); return e ? atoi(e) : 1; }();
        if (q4 && (double)L.n * (double)L.m <= 4e9 && cdiv(L.m, (long long)C::Q * C::NC_MAX) < L.sms)
          return run_q(IC<4>{});
      }
      return run_q(IC<C::Q>{});
    });
  });
}

}  // namespace idw
