// manifold_jvp_kernel instantiations with side 1 = kBoxCp (manifold_jvp.cuh).
#include "manifold_jvp.cuh"

namespace cmgb {
int launch_jvp_k1_cp(const JvpParams& p, int threads, cudaStream_t s) { return launch_jvp_k2<kBoxCp>(p, threads, s); }
#ifdef CMGB_PHASE_CLOCKS
int jvp_phase_clocks_cp(unsigned long long* out) { return read_phase_clocks(out); }
#endif
}  // namespace cmgb
