// sn_far.cu -- the far half of a depth-sliced scene pass (sn_render_opts.near_slice).
//
// A sliced pass emits, sorts and streams only each env's near depth slice (z < z_cut, a sample
// quantile); its far visible splats are never emitted or sorted. Tiles whose near list runs out
// with a live (or undecided) pixel register themselves (the blend: unfinished list, bucket_of map,
// env mask). For those tiles only:
//   far_collect  -- (sn_preprocess.cu) the far items of the envs with unfinished tiles are projected
//                   again; each one reaching an unfinished tile gets a far record and one bucket
//                   item per such tile, keyed bucket | top depth bits;
//   (sort)       -- one 32-bit radix sort of the items: by bucket, then depth;
//   far_tie_fix  -- equal-key runs ordered by (float64 z, gaussian index);
//   far_ranges   -- each bucket's item range;
// and the continuation blend / the float64 fixups walk the bucket after the near list -- the
// reference's per-tile order (renderer.py:80-101: a tile's splats in (z, index) order) is the near
// list followed by the bucket, since every far z is >= every near z of the env.
#include "sn_common.cuh"
#include "sn_internal.h"

#include <algorithm>

namespace sn {

namespace {

__device__ __forceinline__ bool far_ok(const FarArgs &f) {  // no overflow: every item is valid
    return f.fctl[1] <= f.cap_b && f.fctl[4] <= f.cap_f;
}

__device__ __forceinline__ bool far_less(const FarArgs &f, uint32_t a, uint32_t c) {
    const double za = f.recs[a].z, zc = f.recs[c].z;
    if (za != zc) return za < zc;
    return f.gid[a] < f.gid[c];
}

// Runs of equal keys (same bucket, same top depth bits) -- one thread per run start -- ordered by
// (z, gaussian index): insertion sort, the runs are short.
__global__ void __launch_bounds__(kBlock) far_tie_fix_kernel(FarArgs f, const uint32_t *keys, uint32_t *vals) {
    if (!far_ok(f)) return;
    const int64_t n = (int64_t)f.fctl[1];
    const int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    if (i >= n) return;
    if (i > 0 && keys[i - 1] == keys[i]) return;
    int64_t e = i + 1;
    while (e < n && keys[e] == keys[i]) ++e;
    if (e - i < 2) return;
    uint32_t *v = vals + i;
    const int64_t L = e - i;
    for (int64_t x = 1; x < L; ++x) {
        const uint32_t cur = v[x];
        int64_t y = x - 1;
        while (y >= 0 && far_less(f, cur, v[y])) {
            v[y + 1] = v[y];
            --y;
        }
        v[y + 1] = cur;
    }
}

// Each bucket's [first, last + 1) in the sorted items (buckets without items keep the zeroed range).
__global__ void __launch_bounds__(kBlock) far_ranges_kernel(FarArgs f, const uint32_t *keys) {
    if (!far_ok(f)) return;
    const int64_t n = (int64_t)f.fctl[1];
    const int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    if (i >= n) return;
    const int sh = 32 - f.ub;
    const uint32_t b = keys[i] >> sh;
    SN_ASSERT(b < (1u << f.ub));
    if (i == 0 || (keys[i - 1] >> sh) != b) f.ranges[b].x = (uint32_t)i;
    if (i == n - 1 || (keys[i + 1] >> sh) != b) f.ranges[b].y = (uint32_t)(i + 1);
}

unsigned grid_of(uint64_t cap) { return (unsigned)std::max<uint64_t>(1, (cap + kBlock - 1) / kBlock); }

// The far pipeline runs only when the render registered an unfinished tile (a conditional graph node).
__global__ void far_cond_kernel(cudaGraphConditionalHandle h, const unsigned long long *fctl) {
    cudaGraphSetConditional(h, fctl[0] != 0ull ? 1u : 0u);
}

}  // namespace

cudaError_t launch_far_cond(cudaGraphConditionalHandle h, const unsigned long long *fctl, cudaStream_t s) {
    far_cond_kernel<<<1, 1, 0, s>>>(h, fctl);
    return cudaGetLastError();
}

cudaError_t launch_far_tie_fix(const FarArgs &f, const uint32_t *keys, uint32_t *vals, cudaStream_t s) {
    if (f.cap_b == 0) return cudaSuccess;
    far_tie_fix_kernel<<<grid_of(f.cap_b), kBlock, 0, s>>>(f, keys, vals);
    return cudaGetLastError();
}

cudaError_t launch_far_ranges(const FarArgs &f, const uint32_t *keys, cudaStream_t s) {
    if (f.cap_b == 0) return cudaSuccess;
    far_ranges_kernel<<<grid_of(f.cap_b), kBlock, 0, s>>>(f, keys);
    return cudaGetLastError();
}

}  // namespace sn
