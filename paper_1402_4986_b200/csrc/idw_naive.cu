// K1 launcher: one query per thread (reference kernels.predict_block,
// kernels.py:34-67, driven by strategies.run_naive, strategies.py:148-166).
#include "idw_kernels.cuh"
#include "idw_launch.h"

namespace idw {

int launch_naive(Launch &L) {
  return with_layout(L, [&](auto KC, auto tv) -> int {
    using T = decltype(tv);
    constexpr int K = decltype(KC)::value;
    return with_arith(L, [&](auto MC, auto PC, auto EC) -> int {
      constexpr int MODE = decltype(MC)::value;
      constexpr bool P2 = decltype(PC)::value, EPS = decltype(EC)::value;
      const int nt = 256;
      const long long grid = (L.m + nt - 1) / nt;
      float4 *dbox = nullptr;
      StreamFree free_box;
      if constexpr (MODE == EXACT && P2 && !EPS) {  // data box for the inline-reciprocal guard
        if (int rc = launch_bbox<K, T>(L, &dbox)) return rc;
        free_box.p = dbox;
        free_box.st = L.st;
      }
      k_naive<K, T, MODE, P2, EPS><<<(unsigned)grid, nt, 0, L.st>>>(
          L.g, L.n, (const T *)L.qx, (const T *)L.qy, L.m, make_scal<T>(L), (T *)L.out, L.flags, dbox);
      IDW_CK_LAUNCH();
      ++L.launches;
      return 0;
    });
  });
}

}  // namespace idw
