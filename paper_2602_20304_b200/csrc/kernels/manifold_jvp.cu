// Pose-Jacobian dispatch: the SDF kind of side 1 picks the translation unit
// (manifold_jvp_{sq,cp,gen}.cu), side 2 the instantiation inside it.
#include "manifold_jvp.cuh"

namespace cmgb {

int jvp_directions() { return 12; }
int jvp_max_threads() { return kJvpThreads; }
int jvp_smem_cap() { return CMGB_JVP_SMEM_KB * 1024; }

int launch_manifold_jvp(const JvpParams& p, int block_threads, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int threads = block_threads > 0 && block_threads <= kJvpThreads ? block_threads : kJvpThreads;
  switch (jvp_kind_of(p.m.side[0].sdf)) {
    case kSqE01: return launch_jvp_k1_sq(p, threads, s);
    case kBoxCp: return launch_jvp_k1_cp(p, threads, s);
    case kSingleSq: return launch_jvp_k1_ssq(p, threads, s);
    default: return launch_jvp_k1_gen(p, threads, s);
  }
}

}  // namespace cmgb

#ifdef CMGB_PHASE_CLOCKS
namespace cmgb {
int manifold_phase_clocks(unsigned long long* out);
}
extern "C" int cmgb_debug_manifold_phase_clocks(unsigned long long* out) { return cmgb::manifold_phase_clocks(out); }
extern "C" int cmgb_debug_jvp_phase_clocks(unsigned long long* out) {
  for (int i = 0; i < 16; ++i) out[i] = 0;
  return cmgb::jvp_phase_clocks_sq(out) | cmgb::jvp_phase_clocks_cp(out) | cmgb::jvp_phase_clocks_gen(out) |
         cmgb::jvp_phase_clocks_ssq(out);
}
#endif
