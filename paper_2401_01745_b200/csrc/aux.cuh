// aux.cuh — constants of the SYNTHETIC width stand-in EMRKC_MODEL_HH_AUX
// (include/emrkc.h): auxiliary variable a relaxes as
//   g_S,a = k_a ((s1_a V + s0_a) - z_a),
//   k_a = 0.002 (1 + a % 5), s1_a = 0.01 (a % 3), s0_a = 0.5 + 0.1 (a % 4),
// the same IEEE products / sums as the reference harness's HHAux
// (oracle/ref_driver.cpp) and the C oracle, folded at compile time.
#pragma once

#include "../../include/emrkc.h"

namespace emrkc_dev {

#define EMRKC_AUX_K(a) (0.002 * (double)(1 + (a) % 5))
#define EMRKC_AUX_S1(a) (0.01 * (double)((a) % 3))
#define EMRKC_AUX_S0(a) (0.5 + 0.1 * (double)((a) % 4))
#define EMRKC_AUX_ROW(M) \
  M(0), M(1), M(2), M(3), M(4), M(5), M(6), M(7), M(8), M(9), M(10), M(11), M(12), M(13), \
      M(14), M(15), M(16), M(17), M(18), M(19)

struct AuxConsts {
  double k[EMRKC_MAX_AUX], s1[EMRKC_MAX_AUX], s0[EMRKC_MAX_AUX];
};
static_assert(EMRKC_MAX_AUX == 20, "EMRKC_AUX_ROW lists EMRKC_MAX_AUX entries");
static __constant__ AuxConsts kAux = {{EMRKC_AUX_ROW(EMRKC_AUX_K)},
                                      {EMRKC_AUX_ROW(EMRKC_AUX_S1)},
                                      {EMRKC_AUX_ROW(EMRKC_AUX_S0)}};

// f_S aux row in the reference's operation order (no FMA): bit-identical.
__device__ __forceinline__ double aux_rate_ref(int a, double V, double z) {
  return __dmul_rn(kAux.k[a], __dsub_rn(__dadd_rn(__dmul_rn(kAux.s1[a], V), kAux.s0[a]), z));
}
// The same rate in FMA form (fast kernels; rounding-level differences).
__device__ __forceinline__ double aux_rate_fast(int a, double V, double z) {
  return kAux.k[a] * (fma(kAux.s1[a], V, kAux.s0[a]) - z);
}

}  // namespace emrkc_dev
