// Active-contact compaction — an EXTRA output beside the reference's fixed
// layout (include/cmg/manifold.hpp:62-72, 303-330; SURVEY.md §7 hard part 8:
// never a replacement). For every env of a batch it keeps the contacts with
// activity > thr, in fixed-layout order, packed back to back across the whole
// batch, plus each kept contact's slot index and per-env offsets / counts.
//
// Mapping (HBM-bound: every fixed-layout byte is read once, only the kept
// contacts are written):
//   * one CTA per tile of `epb` consecutive envs; their fixed-layout contacts
//     are one contiguous block of epb x C x 32 B, staged into shared memory by
//     ONE TMA bulk copy (cp.async.bulk + mbarrier transaction count);
//   * one warp per env: __ballot_sync(activity > thr) per 32-contact chunk,
//     __popc -> the env's count;
//   * tile offset: a scan of the tile's env counts, then a decoupled look-back
//     over the preceding tiles' published aggregates / inclusive prefixes. Tiles
//     are numbered by an atomic ticket taken at CTA start, so every tile a CTA
//     waits on belongs to a CTA that is already running (forward progress);
//   * each warp writes its env's kept contacts as two float4 per contact
//     (lanes of a chunk -> consecutive 32-B slots: coalesced), their slot
//     indices and (optionally) provenance, and the env's offset / count.
// Envs too large to stage (C x 32 B beyond the shared-memory budget) read
// their contacts from global memory twice instead (kStaged = false).
#include <cstdint>
#include <cstdlib>

#include <cuda_runtime.h>

#include "../device/bulk.cuh"
#include "launch_util.cuh"

namespace cmgb {

int compact_envs_per_tile(int C);
size_t compact_workspace_bytes(int64_t n_env, int C);

namespace {

constexpr uint64_t kFlagAgg = 1ull << 62;
constexpr uint64_t kFlagIncl = 2ull << 62;
constexpr uint64_t kValMask = (1ull << 62) - 1;
constexpr int kMaskWords = 40;  // ballots kept in shared memory for C <= 1,280 contacts per env

__device__ __forceinline__ uint64_t ld_acquire(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(uint64_t* p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

struct CompactParams {
  const float* contacts;   // [n][C][8]
  const int32_t* src;      // optional [n][C][2]
  int64_t n_env;
  int32_t C;
  int32_t epb;             // envs per tile (= warps per CTA)
  float thr;
  int64_t capacity;        // rows of out_contacts / out_slot / out_src
  float* out_contacts;     // [capacity][8]
  int32_t* out_slot;       // optional [capacity]
  int32_t* out_src;        // optional [capacity][2]
  int64_t* env_offset;     // optional [n + 1] (exclusive scan; [n] = total)
  int32_t* env_count;      // optional [n]
  int64_t* total;          // optional [1]
  uint64_t* status;        // [n_tiles] zeroed
  uint32_t* ticket;        // [1] zeroed
};

template <bool kStaged>
__global__ void __launch_bounds__(256) compact_kernel(const __grid_constant__ CompactParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t s_tile;
  __shared__ int64_t s_base;
  __shared__ int32_t s_cnt[8];
  __shared__ unsigned s_mask[8][kMaskWords];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int C = p.C;
  if (threadIdx.x == 0) s_tile = atomicAdd(p.ticket, 1u);
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t env0 = tile * p.epb;
  const int64_t left = p.n_env - env0;
  const int n_here = left < p.epb ? (int)left : p.epb;
  const float4* gsrc = reinterpret_cast<const float4*>(p.contacts) + env0 * C * 2;
  const float4* tile_c = gsrc;
  if constexpr (kStaged) {
    const uint32_t bytes = (uint32_t)n_here * (uint32_t)C * 32u;
    if (threadIdx.x == 0) {
      mbar_init(&bar, 1);
      mbar_fence_init();
      mbar_arrive_expect_tx(&bar, bytes);
      bulk_g2s(smem, gsrc, bytes, &bar);
    }
    __syncthreads();
    mbar_wait(&bar, 0);
    tile_c = reinterpret_cast<const float4*>(smem);
  }

  // ---- per-env counts (one warp per env); the ballots are kept per warp for
  // the write pass (up to kMaskWords chunks, else the activities are re-read)
  int cnt = 0;
  const bool masks = C <= 32 * kMaskWords;
  if (warp < n_here) {
    const float4* ec = tile_c + (int64_t)warp * C * 2;
    const float* act = reinterpret_cast<const float*>(ec) + 7;  // activity of contact j at act[8 j]
#pragma unroll 4
    for (int j0 = 0; j0 < C; j0 += 32) {
      const int j = j0 + lane;
      const bool keep = j < C && act[8 * j] > p.thr;
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      if (masks && lane == 0) s_mask[warp][j0 >> 5] = m;
      cnt += __popc(m);
    }
    if (lane == 0) s_cnt[warp] = cnt;
  }
  __syncthreads();

  // ---- tile offset: aggregate, decoupled look-back, inclusive prefix -----------
  if (warp == 0) {
    int64_t mine = 0;
    for (int w = 0; w < n_here; ++w) mine += s_cnt[w];
    if (lane == 0) st_release(p.status + tile, (tile == 0 ? kFlagIncl : kFlagAgg) | (uint64_t)mine);
    int64_t excl = 0;
    if (tile > 0) {
      int64_t base = tile - 1;
      while (true) {
        const int64_t idx = base - lane;
        uint64_t s = idx >= 0 ? ld_acquire(p.status + idx) : kFlagIncl;
        while (__any_sync(0xffffffffu, (s >> 62) == 0)) {  // a predecessor has not published yet
          if ((s >> 62) == 0) s = ld_acquire(p.status + idx);
        }
        const unsigned incl = __ballot_sync(0xffffffffu, (s >> 62) == 2);
        const int stop = incl ? __ffs(incl) - 1 : 31;  // nearest tile with an inclusive prefix
        int64_t v = lane <= stop ? (int64_t)(s & kValMask) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        excl += v;
        if (incl) break;
        base -= 32;
      }
      if (lane == 0) st_release(p.status + tile, kFlagIncl | (uint64_t)(excl + mine));
    }
    if (lane == 0) {
      s_base = excl;
      const int64_t ntiles = (p.n_env + p.epb - 1) / p.epb;
      if (tile == ntiles - 1) {
        if (p.total) *p.total = excl + mine;
        if (p.env_offset) p.env_offset[p.n_env] = excl + mine;
      }
    }
  }
  __syncthreads();

  // ---- writes: env offset / count, then the kept contacts in layout order -----
  if (warp >= n_here) return;
  int64_t off = s_base;
  for (int w = 0; w < warp; ++w) off += s_cnt[w];
  const int64_t e = env0 + warp;
  if (lane == 0) {
    if (p.env_offset) p.env_offset[e] = off;
    if (p.env_count) p.env_count[e] = s_cnt[warp];
  }
  const float4* ec = tile_c + (int64_t)warp * C * 2;
  float4* oc = reinterpret_cast<float4*>(p.out_contacts);
  const float* act = reinterpret_cast<const float*>(ec) + 7;
  for (int j0 = 0; j0 < C; j0 += 32) {
    const int j = j0 + lane;
    const unsigned m =
        masks ? s_mask[warp][j0 >> 5] : __ballot_sync(0xffffffffu, j < C && act[8 * j] > p.thr);
    if (m == 0u) continue;
    const bool keep = (m >> lane) & 1u;
    const int64_t dst = off + __popc(m & ((1u << lane) - 1u));
    if (keep && dst < p.capacity) {  // only the kept contacts are read again (L2-resident)
      oc[2 * dst] = ec[2 * j];
      oc[2 * dst + 1] = ec[2 * j + 1];
      if (p.out_slot) p.out_slot[dst] = j;
      if (p.out_src) {
        const int2 s = reinterpret_cast<const int2*>(p.src)[e * C + j];
        reinterpret_cast<int2*>(p.out_src)[dst] = s;
      }
    }
    off += __popc(m);
  }
}

// ---- compaction from the manifold kernel's activity masks -------------------
// The fixed layout is not scanned again. Two launches: (1) an exclusive scan
// of the per-env counts, 1,024 envs per CTA (warp shuffles, decoupled
// look-back over tiles as above; few tiles, so the look-back chain stays
// short); (2) one warp per env walks the env's mask words (one lane per word)
// and copies only the kept contacts (32 B each) to their compacted rows --
// no dependency between envs, every warp of the grid in flight at once.
constexpr int kScanTile = 1024;  // envs per scan CTA (one thread each)

struct MaskedParams {
  const float* contacts;
  const int32_t* src;
  int64_t n_env;
  int32_t C, mask_words;
  const uint32_t* mask;
  const int32_t* count;
  int64_t capacity;
  float* out_contacts;
  int32_t* out_slot;
  int32_t* out_src;
  int64_t* env_offset;  // required here: the gather reads it
  int32_t* env_count;
  int64_t* total;
  uint64_t* status;
  uint32_t* ticket;
};

__global__ void __launch_bounds__(kScanTile) compact_scan_kernel(const __grid_constant__ MaskedParams p) {
  __shared__ uint32_t s_tile;
  __shared__ int64_t s_wsum[kScanTile / 32];
  __shared__ int64_t s_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) s_tile = atomicAdd(p.ticket, 1u);
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t e = tile * kScanTile + tid;
  const int64_t cnt = e < p.n_env ? p.count[e] : 0;
  int64_t incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) s_wsum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    // scan of the 32 warp sums, then the look-back
    const int64_t ws = s_wsum[lane];
    int64_t wi = ws;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t v = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += v;
    }
    s_wsum[lane] = wi - ws;  // exclusive warp offsets
    const int64_t agg = __shfl_sync(0xffffffffu, wi, 31);
    if (lane == 0) st_release(p.status + tile, (tile == 0 ? kFlagIncl : kFlagAgg) | (uint64_t)agg);
    int64_t excl = 0;
    if (tile > 0) {
      int64_t base = tile - 1;
      while (true) {
        const int64_t idx = base - lane;
        uint64_t st = idx >= 0 ? ld_acquire(p.status + idx) : kFlagIncl;
        while (__any_sync(0xffffffffu, (st >> 62) == 0)) {
          if ((st >> 62) == 0) st = ld_acquire(p.status + idx);
        }
        const unsigned inc = __ballot_sync(0xffffffffu, (st >> 62) == 2);
        const int stop = inc ? __ffs(inc) - 1 : 31;
        int64_t v = lane <= stop ? (int64_t)(st & kValMask) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        excl += v;
        if (inc) break;
        base -= 32;
      }
      if (lane == 0) st_release(p.status + tile, kFlagIncl | (uint64_t)(excl + agg));
    }
    if (lane == 0) {
      s_base = excl;
      const int64_t ntiles = (p.n_env + kScanTile - 1) / kScanTile;
      if (tile == ntiles - 1) {
        if (p.total) *p.total = excl + agg;
        p.env_offset[p.n_env] = excl + agg;
      }
    }
  }
  __syncthreads();
  if (e < p.n_env) {
    p.env_offset[e] = s_base + s_wsum[warp] + incl - cnt;
    if (p.env_count) p.env_count[e] = (int32_t)cnt;
  }
}

__global__ void __launch_bounds__(256) compact_gather_kernel(const __grid_constant__ MaskedParams p) {
  const int lane = threadIdx.x & 31;
  const int64_t ej = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (ej >= p.n_env) return;
  const int mw = p.mask_words;
  const float4* in = reinterpret_cast<const float4*>(p.contacts);
  float4* oc = reinterpret_cast<float4*>(p.out_contacts);
  int64_t run = p.env_offset[ej];
  for (int w0 = 0; w0 < mw; w0 += 32) {
    const int w = w0 + lane;
    uint32_t m = w < mw ? p.mask[ej * mw + w] : 0u;
    const int pc = __popc(m);
    int pre = pc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, pre, o);
      if (lane >= o) pre += v;
    }
    int64_t dst = run + pre - pc;  // this word's first kept row
    while (m) {
      const int b = __ffs(m) - 1;
      m &= m - 1;
      const int cidx = 32 * w + b;
      if (dst < p.capacity) {
        const int64_t srow = ej * p.C + cidx;
        oc[2 * dst] = in[2 * srow];
        oc[2 * dst + 1] = in[2 * srow + 1];
        if (p.out_slot) p.out_slot[dst] = cidx;
        if (p.out_src) reinterpret_cast<int2*>(p.out_src)[dst] = reinterpret_cast<const int2*>(p.src)[srow];
      }
      ++dst;
    }
    run += __shfl_sync(0xffffffffu, pre, 31);
  }
}

}  // namespace

size_t compact_workspace_bytes(int64_t n_env, int C) {
  const int epb = compact_envs_per_tile(C);
  const int64_t tiles = (n_env + epb - 1) / epb;
  return sizeof(uint64_t) * (size_t)(tiles + 2);
}

// A/B switch for measurement (CMGB_COMPACT_STAGED=1: TMA-staged tiles).
static bool compact_staged() {
  static const int v = [] {
    const char* e = getenv("CMGB_COMPACT_STAGED");
    return e ? atoi(e) : 0;
  }();
  return v != 0;
}

// Envs per tile: staged, up to 8 warps in <= 40 KB of shared memory (several
// CTAs per SM keep bulk copies in flight); direct, 8 warps.
int compact_envs_per_tile(int C) {
  if (!compact_staged()) return 8;
  const int per_env = C * 32;
  int epb = per_env > 0 ? (40 * 1024) / per_env : 8;
  return epb < 1 ? 1 : (epb > 8 ? 8 : epb);
}

int launch_compact(const float* contacts, const int32_t* src, int64_t n_env, int C, float thr, int64_t capacity,
                   float* out_contacts, int32_t* out_slot, int32_t* out_src, int64_t* env_offset,
                   int32_t* env_count, int64_t* total, void* workspace, cudaStream_t s) {
  CompactParams p{};
  p.contacts = contacts;
  p.src = src;
  p.n_env = n_env;
  p.C = C;
  p.epb = compact_envs_per_tile(C);
  p.thr = thr;
  p.capacity = capacity;
  p.out_contacts = out_contacts;
  p.out_slot = out_slot;
  p.out_src = out_src;
  p.env_offset = env_offset;
  p.env_count = env_count;
  p.total = total;
  const int64_t tiles = (n_env + p.epb - 1) / p.epb;
  p.ticket = static_cast<uint32_t*>(workspace);
  p.status = static_cast<uint64_t*>(workspace) + 1;
  if (cudaMemsetAsync(workspace, 0, compact_workspace_bytes(n_env, C), s) != cudaSuccess) return 1;
  const size_t stage = (size_t)p.epb * C * 32;
  static PerDeviceOnce configured;
  configured([] {
    allow_max_dynamic_smem(compact_kernel<true>);
  });
  note_launch();
  if (compact_staged() && stage <= (size_t)smem_optin_per_block())
    compact_kernel<true><<<(unsigned)tiles, 32 * p.epb, stage, s>>>(p);
  else
    compact_kernel<false><<<(unsigned)tiles, 32 * p.epb, 0, s>>>(p);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

size_t compact_masked_workspace_bytes(int64_t n_env) {
  // ticket + scan-tile status words, then (when the caller wants no offsets) env offsets
  return sizeof(uint64_t) * (size_t)((n_env + kScanTile - 1) / kScanTile + 2) + sizeof(int64_t) * (n_env + 1);
}

int launch_compact_masked(const float* contacts, const int32_t* src, int64_t n_env, int C, const uint32_t* mask,
                          const int32_t* count, int64_t capacity, float* out_contacts, int32_t* out_slot,
                          int32_t* out_src, int64_t* env_offset, int32_t* env_count, int64_t* total,
                          void* workspace, cudaStream_t s) {
  MaskedParams p{};
  p.contacts = contacts;
  p.src = src;
  p.n_env = n_env;
  p.C = C;
  p.mask_words = (C + 31) / 32;
  p.mask = mask;
  p.count = count;
  p.capacity = capacity;
  p.out_contacts = out_contacts;
  p.out_slot = out_slot;
  p.out_src = out_src;
  p.env_count = env_count;
  p.total = total;
  const int64_t tiles = (n_env + kScanTile - 1) / kScanTile;
  const size_t status_bytes = sizeof(uint64_t) * (size_t)(tiles + 2);
  p.ticket = static_cast<uint32_t*>(workspace);
  p.status = static_cast<uint64_t*>(workspace) + 1;
  p.env_offset = env_offset ? env_offset
                            : reinterpret_cast<int64_t*>(static_cast<unsigned char*>(workspace) + status_bytes);
  if (cudaMemsetAsync(workspace, 0, status_bytes, s) != cudaSuccess) return 1;
  note_launch();
  compact_scan_kernel<<<(unsigned)tiles, kScanTile, 0, s>>>(p);
  if (cudaGetLastError() != cudaSuccess) return 1;
  note_launch();
  compact_gather_kernel<<<(unsigned)((n_env * 32 + 255) / 256), 256, 0, s>>>(p);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // namespace cmgb
