// Manifold instantiations for the compile-time-exponent superquadric kinds
// other than eps = 0.1 (common.h: kSqE02, kSqE025, kSqE05, kSqEll, kSqCyl):
// both sides of the same kind (box-box-like scenes, with the separate V-S
// launch when the vertex sets are pass-through) and each kind against the
// box_planes leaf in either order (config C's plate vs primitive). Every other
// combination runs through manifold.cu's runtime-exponent instantiations.
#include "manifold.cuh"

namespace cmgb {

namespace {

template <int K>
int launch_vs_cp(const ManifoldParams& p, int threads, int grid, size_t smem, cudaStream_t s, bool* handled) {
  const int k1 = p.side[0].sdf.kind, k2 = p.side[1].sdf.kind;
  if (k1 == K && k2 == K) {
    *handled = true;
    return launch_same_kind<K>(p, threads, grid, smem, s);
  }
  if (k1 == kBoxCp && k2 == K) {
    *handled = true;
    return launch_kind<kBoxCp, K>(p, threads, grid, smem, s);
  }
  if (k1 == K && k2 == kBoxCp) {
    *handled = true;
    return launch_kind<K, kBoxCp>(p, threads, grid, smem, s);
  }
  return 0;
}

}  // namespace

int launch_manifold_ct(const ManifoldParams& p, int threads, int grid, size_t smem, cudaStream_t s, bool* handled) {
  *handled = false;
  int rc = 0;
  for (int k : {p.side[0].sdf.kind, p.side[1].sdf.kind}) {
    switch (k) {
      case kSqE02: rc = launch_vs_cp<kSqE02>(p, threads, grid, smem, s, handled); break;
      case kSqE025: rc = launch_vs_cp<kSqE025>(p, threads, grid, smem, s, handled); break;
      case kSqE05: rc = launch_vs_cp<kSqE05>(p, threads, grid, smem, s, handled); break;
      case kSqEll: rc = launch_vs_cp<kSqEll>(p, threads, grid, smem, s, handled); break;
      case kSqCyl: rc = launch_vs_cp<kSqCyl>(p, threads, grid, smem, s, handled); break;
      case kCapsule: rc = launch_vs_cp<kCapsule>(p, threads, grid, smem, s, handled); break;
      default: break;
    }
    if (*handled) return rc;
  }
  return 0;
}

#ifdef CMGB_PHASE_CLOCKS
int manifold_ct_phase_clocks(unsigned long long* out) {
  unsigned long long h[16];
  if (cudaMemcpyFromSymbol(h, g_mf_phase, sizeof(h)) != cudaSuccess) return 1;
  for (int i = 0; i < 16; ++i) out[i] += h[i];
  return 0;
}
#endif

}  // namespace cmgb
