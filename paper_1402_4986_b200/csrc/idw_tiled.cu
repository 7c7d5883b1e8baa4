// K2 launcher: shared-memory tiled kernel (reference tile_accumulate +
// finalize_block over LayoutStore.load_tile, kernels.py:70-108,
// layouts.py:215-229, strategies.py:169-199).
//
// EXACT (k_tiled): every query costs the same n pairs in the reference's strict
// order, so the kernel is balanced statically: the query range is cut into
// grid_x = waves * slots blocks (slots = SMs x resident CTAs per SM) and each
// block gets only as many consumer warps as its share needs.
//
// FAST (k_tiled_chunks): the data tiles are cut into chunks whose size is a
// function of n alone (chunk_shape), and a persistent grid of warps takes
// (query group, chunk) work items from one counter; see idw_kernels.cuh.
#include <algorithm>
#include <cstdlib>

#include "idw_kernels.cuh"
#include "idw_launch.h"

namespace idw {

template <typename T, int MODE>
struct TiledCfg;
// fp32: 256-point warp tiles; FAST packs 8 queries (4 pairs) per thread.
#ifndef IDW_FAST_Q
#define IDW_FAST_Q 8
#endif
#ifndef IDW_FAST_TILE
#define IDW_FAST_TILE 256
#endif
template <>
struct TiledCfg<float, FAST> {
  static constexpr int Q = IDW_FAST_Q, TILE = IDW_FAST_TILE, NC_MAX = 256;
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

// EXACT query blocks: the smallest number of waves whose blocks still hold
// >= half a full block (>= 4 warps) of queries, unless m is smaller.
struct Shape {
  long long qpc, blocks;
};
static Shape shape_grid(long long m, long long slots, int Q, int nc_max) {
  const long long cap = (long long)nc_max * Q;
  // (full blocks on fewer SMs measured faster than thin blocks on all SMs
  // for EXACT, C2: 2120 vs 1978 GPairs/s)
  const long long min_q = std::min<long long>(cap / 2, cdiv(m, Q) * Q);
  for (long long W = 1; W <= 64; ++W) {
    const long long qpc = cdiv(cdiv(m, W * slots), Q) * Q;
    if (qpc > cap) continue;  // too few blocks for this many waves
    if (qpc < min_q) break;
    return {qpc, cdiv(m, qpc)};
  }
  const long long qpc = std::min<long long>(cap, cdiv(m, Q) * Q);
  return {qpc, cdiv(m, qpc)};
}

// FAST summation chunks: tiles per chunk and chunk count from n alone, so a
// query's result is the same for every m, shard and device count.  About 128
// chunks (>= 1 and <= 128 tiles each, <= 2048 chunks): work items small enough
// for the dynamic schedule to end evenly, large enough that a chunk partial
// costs < 0.1 % of its pairs and that the partials of a band (below) stay
// few.  `forced` (ExecConfig.splits) overrides.
static void chunk_shape(long long ntiles, int forced, long long *S, long long *tpc) {
  long long t;
  if (forced > 0) {
    t = cdiv(ntiles, std::min<long long>(forced, ntiles));
  } else {
    t = std::min<long long>(128, std::max<long long>(1, ntiles / 128));
    t = std::max<long long>(t, cdiv(ntiles, 2048));
    // experiment knob (changes the summation order, hence the bits)
    static const long long env_tpc = [] { const char *e = getenv("IDW_TPC"); return e ? atoll(e) : 0ll; }();
    if (env_tpc > 0) t = std::min<long long>(env_tpc, ntiles);
  }
  *tpc = t;
  *S = cdiv(ntiles, t);
}

template <int K, typename T, bool P2, bool EPS, bool INLINE_BOX>
static int launch_tiled_fast_box(Launch &L) {
  using C = TiledCfg<T, FAST>;
  constexpr int Q = C::Q, TILE = C::TILE, QG = 32 * Q, NC = 256;
  constexpr int RING = tiled_ring_bytes<K, T, TILE>();
  auto kern = k_tiled_chunks<K, T, P2, EPS, Q, TILE>;
  bool prod_used = false;
  if constexpr (std::is_same<T, float>::value && P2 && !EPS) {
    // One of the four packed query pairs per point shares a reciprocal
    // (measured on C3: 0 -> 4196, 1 -> 4546, 2 -> 4533 GPairs/s; the mix of
    // MUFU and FMA-pipe work is best balanced at 1).  IDW_PROD overrides
    // (it changes which queries pair up, hence the bits).
    static const int prod = [] { const char *e = getenv("IDW_PROD"); return e ? atoi(e) : 1; }();
    if (prod == 1) kern = k_tiled_chunks<K, T, P2, EPS, Q, TILE, 1, 0, INLINE_BOX>;
    if (prod == 2) kern = k_tiled_chunks<K, T, P2, EPS, Q, TILE, 2, 0, INLINE_BOX>;
    prod_used = prod == 1 || prod == 2;
  }
  if constexpr (sizeof(T) == 8 && !P2) {
    // compile-time powers for the common half-integer p (p = 3: jq 6, p = 3.5: jq 7)
    const int jq = make_scal<T>(L).jq;
    if (jq == 7) kern = k_tiled_chunks<K, T, P2, EPS, Q, TILE, 0, 7>;
    if (jq == 6) kern = k_tiled_chunks<K, T, P2, EPS, Q, TILE, 0, 6>;
  }
  if constexpr (sizeof(T) == 4 && !P2) {
    // integer p = 1, 3, 4: one MUFU per pair (rsqrt / rcp powers) instead of lg2 + ex2
    const int jq = make_scal<T>(L).jq;
    if (jq == 2) kern = k_tiled_chunks<K, T, P2, EPS, Q, TILE, 0, 2>;
    if (jq == 6) kern = k_tiled_chunks<K, T, P2, EPS, Q, TILE, 0, 6>;
    if (jq == 8) kern = k_tiled_chunks<K, T, P2, EPS, Q, TILE, 0, 8>;
  }
  const int smem = (NC / 32) * RING;
  int occ = 0, occ_big = 0;
  constexpr int WMAX = CHUNK_THREADS_MAX / 32;  // warps of the largest small-job CTA
  if (int rc = kernel_occupancy((const void *)kern, L.dev, 32 * WMAX, WMAX * RING, &occ_big)) return rc;
  if (int rc = kernel_occupancy((const void *)kern, L.dev, NC, smem, &occ)) return rc;
  if (occ < 1) occ = 1;
  const long long ntiles = cdiv(L.n, TILE);
  long long S = 1, tpc = 1;
  chunk_shape(ntiles, L.splits, &S, &tpc);
  const long long groups = cdiv(L.m, QG);
  if (groups >= (1ll << 31) || ntiles >= (1ll << 31)) {
    set_error("too many points for one call");
    return IDW_E_ARG;
  }
  const long long items = groups * S;
  const long long slots = (long long)L.sms * occ;
  const long long warps = slots * (NC / 32);
  // Grid: a full persistent grid when the items outnumber its warps; otherwise
  // one CTA per SM with an equal share of warps (one item each), so no SM
  // holds two CTAs while another holds one (C1: 1600 items on 148 SMs).
  long long blocks = slots;
  int threads = NC, smem_l = smem;
  if (items < warps && occ_big >= 1) {
    const long long w = std::max<long long>(1, std::min<long long>(WMAX, cdiv(items, L.sms)));
    blocks = std::min<long long>(L.sms, cdiv(items, w));
    threads = (int)w * 32;
    smem_l = (int)w * RING;
  }
  // Item order: a store larger than a quarter of L2 is swept by bands of B
  // groups (chunk-major inside a band), so HBM streams it once per band
  // instead of once per ~warps/S groups (C5, 10M x 100K: 60.7 GB -> 0.6 GB
  // read per launch); B holds a band's chunk partials to 64 MB.  The order of
  // work items never changes the bits (each group folds its chunks in chunk
  // order).
  long long B = 1;
  if (S > 1 && (double)L.n * 4 * sizeof(T) > 32e6) {
    const long long per_group = S * 2 * QG * (long long)sizeof(T);
    B = std::max<long long>(1, std::min<long long>(groups, (64ll << 20) / per_group));
  }
  static const long long env_band = [] { const char *e = getenv("IDW_BAND"); return e ? atoll(e) : 0ll; }();
  if (env_band > 0) B = std::min<long long>(groups, env_band);
  // ring slots: two bands plus ~4x the groups a full grid has in flight, so a
  // slot's previous group is long folded when the slot comes round again
  // (R >= B is what progress needs: group g - R then lies in an earlier band,
  // whose items were all taken before any of g's)
  const long long R = S > 1 ? std::min<long long>(groups, 2 * B + 4 * cdiv(warps, S) + 4) : 0;

  // scratch: [next u64 | pad | done[R] | gen[R] | chunk boxes[S] | partials]
  const size_t ctl = ((size_t)(16 + 8 * R) + 255) / 256 * 256;
  const size_t boxb = prod_used && !INLINE_BOX ? ((size_t)S * sizeof(float4) + 255) / 256 * 256 : 0;
  const size_t part = (size_t)R * (size_t)S * 2 * QG * sizeof(T);
  unsigned char *ws = nullptr;
  StreamFree free_ws;  // scratch goes back to the pool on every exit
  IDW_CK(cudaMallocAsync((void **)&ws, ctl + boxb + part, L.st));
  free_ws.p = ws;
  free_ws.st = L.st;
  IDW_CK(cudaMemsetAsync(ws, 0, ctl, L.st));
  float4 *boxes = boxb ? (float4 *)(ws + ctl) : nullptr;
  if (boxes) {  // chunk data boxes for the shared-reciprocal guard
    k_chunk_boxes<K, T><<<(unsigned)cdiv(S * 32, 256), 256, 0, L.st>>>(L.g, L.n, tpc * TILE, (int)S, boxes);
    IDW_CK_LAUNCH();
    ++L.launches;
  }
  ChunkSched<T> cs;
  cs.next = (unsigned long long *)ws;
  cs.done = (unsigned int *)(ws + 16);
  cs.gen = cs.done + R;
  cs.boxes = boxes;
  cs.part = (T *)(ws + ctl + boxb);
  cs.groups = groups;
  cs.S = (int)S;
  cs.tpc = (int)tpc;
  cs.R = (int)R;
  cs.B = (int)B;
  kern<<<(unsigned)blocks, threads, smem_l, L.st>>>(L.g, L.n, (const T *)L.qx, (const T *)L.qy, L.m,
                                                    make_scal<T>(L), (T *)L.out, L.flags, cs);
  IDW_CK_LAUNCH();
  ++L.launches;
  return 0;
}

template <int K, typename T, bool P2, bool EPS>
static int launch_tiled_fast(Launch &L) {
  if constexpr (std::is_same<T, float>::value && P2 && !EPS) {
    // a job whose (group, chunk) items fit one round of a full grid: each
    // warp boxes its own chunk instead of waiting for a box pre-pass launch
    using C = TiledCfg<T, FAST>;
    long long S = 1, tpc = 1;
    chunk_shape(cdiv(L.n, C::TILE), L.splits, &S, &tpc);
    if (cdiv(L.m, 32 * C::Q) * S < (long long)L.sms * 16) return launch_tiled_fast_box<K, T, P2, EPS, true>(L);
  }
  return launch_tiled_fast_box<K, T, P2, EPS, false>(L);
}

template <int K, typename T, int MODE, bool P2, bool EPS, int Q>
static int launch_tiled_exact(Launch &L) {
  using C = TiledCfg<T, MODE>;
  constexpr int TILE = C::TILE;
  constexpr int RING = tiled_ring_bytes<K, T, TILE>();
  auto kern = k_tiled<K, T, MODE, P2, EPS, Q, TILE>;
  const int smem_max = (C::NC_MAX / 32) * RING;
  int occ = 0;
  if (int rc = kernel_occupancy((const void *)kern, L.dev, C::NC_MAX, smem_max, &occ)) return rc;
  if (occ < 1) occ = 1;
  const Shape sh = shape_grid(L.m, (long long)L.sms * occ, Q, C::NC_MAX);
  const int nc = (int)cdiv(cdiv(sh.qpc, Q), 32) * 32;
  const int smem = (nc / 32) * RING;
  float4 *dbox = nullptr;
  StreamFree free_box;
  using AccT = typename AccSelNT<T, MODE, P2, EPS, Q>::type;
  constexpr bool EXACT_FR = std::is_same<AccT, AccExactScr2<Q>>::value ||
                           std::is_same<AccT, AccExactScr<double, true, Q>>::value;
  if (EXACT_FR) {  // data box for the inline-reciprocal guard
    if (int rc = launch_bbox<K, T>(L, &dbox)) return rc;
    free_box.p = dbox;
    free_box.st = L.st;
  }
  kern<<<(unsigned)sh.blocks, nc, smem, L.st>>>(L.g, L.n, (const T *)L.qx, (const T *)L.qy, L.m, sh.qpc,
                                                make_scal<T>(L), (T *)L.out, L.flags, dbox);
  IDW_CK_LAUNCH();
  ++L.launches;
  return 0;
}

int launch_tiled(Launch &L) {
  return with_layout(L, [&](auto KC, auto tv) -> int {
    using T = decltype(tv);
    constexpr int K = decltype(KC)::value;
    return with_arith(L, [&](auto MC, auto PC, auto EC) -> int {
      constexpr int MODE = decltype(MC)::value;
      constexpr bool P2 = decltype(PC)::value, EPS = decltype(EC)::value;
      if constexpr (MODE == FAST) {
        return launch_tiled_fast<K, T, P2, EPS>(L);
      } else {
        using C = TiledCfg<T, MODE>;
        if constexpr (std::is_same<T, float>::value && P2 && !EPS) {
          // EXACT keeps the strict data order, so it cannot split the data: when
          // Q = 4 blocks would not cover the SMs once, halve the queries per
          // thread so the same queries spread over all SMs (C2, 100K queries:
          // 100 CTAs on 148 SMs -> 296 CTAs).  Per-query arithmetic unchanged.
          // Measured at C2: SoA 2093 -> 2609, AoaS 2240 -> 2645 GPairs/s; AoS
          // 2211 -> 2023, so AoS keeps Q = 4.  IDW_EXACT_Q2=0 disables.
          static const int q2 = [] { const char *e = getenv("IDW_EXACT_Q2"); return e ? atoi(e) : 1; }();
          if (K != AOS && q2 && cdiv(L.m, (long long)C::Q * C::NC_MAX) < L.sms)
            return launch_tiled_exact<K, T, MODE, P2, EPS, 2>(L);
        }
        return launch_tiled_exact<K, T, MODE, P2, EPS, C::Q>(L);
      }
    });
  });
}

}  // namespace idw

#ifdef IDW_TRACE
extern "C" int idw_trace_dump(unsigned long long *host) {
  return (int)cudaMemcpyFromSymbol(host, idw::g_idw_trace, sizeof(idw::g_idw_trace));
}
#endif
