// manifold_jvp_kernel instantiations with side 1 = a lone integer-exponent
// superquadric (kSingleSq in the JVP dispatch, manifold_jvp.cuh jvp_kind_of).
#include "manifold_jvp.cuh"

namespace cmgb {
int launch_jvp_k1_ssq(const JvpParams& p, int threads, cudaStream_t s) {
  return launch_jvp_k2<kSingleSq>(p, threads, s);
}
#ifdef CMGB_PHASE_CLOCKS
int jvp_phase_clocks_ssq(unsigned long long* out) { return read_phase_clocks(out); }
#endif
}  // namespace cmgb
