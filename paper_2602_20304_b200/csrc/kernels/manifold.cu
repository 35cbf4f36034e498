// Manifold launch dispatch for the base SDF kinds (kSqE01, kSingleSq,
// kSingleCp, kBoxCp, kGeneric); the other compile-time-exponent superquadric
// kinds are instantiated in manifold_ct.cu (parallel compilation).
#include "manifold.cuh"

namespace cmgb {

int launch_manifold_ct(const ManifoldParams& p, int threads, int grid, size_t smem, cudaStream_t s, bool* handled);

namespace {

// Kinds without their own instantiation here run as the runtime-exponent
// superquadric (same leaf code, exponents read from the descriptor).
constexpr int base_kind(int k) { return k == kCapsule ? (int)kGeneric : (ct_sq(k) && k != kSqE01 ? (int)kSingleSq : k); }

template <int K1>
int launch_k2(const ManifoldParams& p, int threads, int grid, size_t smem, cudaStream_t s) {
  switch (base_kind(p.side[1].sdf.kind)) {
    case kSqE01:
      if constexpr (K1 == kSqE01 || K1 == kSingleSq || K1 == kSingleCp || K1 == kBoxCp)
        return launch_kind<K1, kSqE01>(p, threads, grid, smem, s);
      else
        return launch_kind<K1, kSingleSq>(p, threads, grid, smem, s);
    case kSingleSq: return launch_kind<K1, kSingleSq>(p, threads, grid, smem, s);
    case kSingleCp: return launch_kind<K1, kSingleCp>(p, threads, grid, smem, s);
    case kBoxCp: return launch_kind<K1, kBoxCp>(p, threads, grid, smem, s);
    default: return launch_kind<K1, kGeneric>(p, threads, grid, smem, s);
  }
}

}  // namespace

int launch_manifold(const ManifoldParams& p, int block_threads, int grid, size_t smem_bytes,
                    void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t n1 = p.stride1 ? p.n_env : 1, n2 = p.stride2 ? p.n_env : 1;
  if (!p.frames_ready && launch_frames(p.poses1, p.pose_stride1, n1, const_cast<double*>(p.frames1), p.poses2,
                                       p.pose_stride2, n2, const_cast<double*>(p.frames2), s))
    return 1;
  if (p.pairs_gmem)  // the generic interpreter evaluates every SDF kind
    return launch_kind<kGeneric, kGeneric, true>(p, block_threads, grid, smem_bytes, s);
  if (p.side[0].sdf.kind == kSqE01 && p.side[1].sdf.kind == kSqE01)
    return launch_same_kind<kSqE01>(p, block_threads, grid, smem_bytes, s);
  {
    bool handled = false;
    const int rc = launch_manifold_ct(p, block_threads, grid, smem_bytes, s, &handled);
    if (handled) return rc;
  }
  switch (base_kind(p.side[0].sdf.kind)) {
    case kSqE01: return launch_k2<kSqE01>(p, block_threads, grid, smem_bytes, s);
    case kSingleSq: return launch_k2<kSingleSq>(p, block_threads, grid, smem_bytes, s);
    case kSingleCp: return launch_k2<kSingleCp>(p, block_threads, grid, smem_bytes, s);
    case kBoxCp: return launch_k2<kBoxCp>(p, block_threads, grid, smem_bytes, s);
    default: return launch_k2<kGeneric>(p, block_threads, grid, smem_bytes, s);
  }
}

int manifold_max_threads(int k1, int k2) { return max_threads(k1, k2); }

int launch_scene_frames(const double* poses, int64_t n_poses, double* frames, void* stream) {
  return launch_frames(poses, 6, n_poses, frames, nullptr, 0, 0, nullptr, static_cast<cudaStream_t>(stream));
}

#ifdef CMGB_PHASE_CLOCKS
int manifold_ct_phase_clocks(unsigned long long* out);
int manifold_phase_clocks(unsigned long long* out) {  // both translation units' counters
  if (cudaMemcpyFromSymbol(out, g_mf_phase, 16 * sizeof(unsigned long long)) != cudaSuccess) return 1;
  return manifold_ct_phase_clocks(out);
}
#endif
int manifold_min_blocks(int k1, int k2) { return min_blocks(k1, k2); }

}  // namespace cmgb
