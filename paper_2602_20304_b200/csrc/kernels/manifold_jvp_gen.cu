// manifold_jvp_kernel instantiations with side 1 = kGeneric (manifold_jvp.cuh).
#include "manifold_jvp.cuh"

namespace cmgb {
int launch_jvp_k1_gen(const JvpParams& p, int threads, cudaStream_t s) { return launch_jvp_k2<kGeneric>(p, threads, s); }
#ifdef CMGB_PHASE_CLOCKS
int jvp_phase_clocks_gen(unsigned long long* out) { return read_phase_clocks(out); }
#endif
}  // namespace cmgb
