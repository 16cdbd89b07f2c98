// sn_far.cu -- the far half of a depth-sliced scene pass (sn_render_opts.near_slice).
//
// A sliced pass sorts only each env's near depth slice (z < z_cut, a sample quantile); the far
// visible splats are written as 16-byte FarRec (gaussian, env, tight rectangle) and never sorted
// globally. Tiles whose near list runs out with a live (or undecided) pixel register themselves
// (the blend: unfinished list + bucket_of map). For those tiles only:
//   far_count   -- each far splat adds itself to the bucket of every unfinished tile of its env its
//                  rectangle covers;
//   (scan)      -- bucket offsets;
//   far_scatter -- the same walk writes the far index into the bucket;
//   far_project -- (sn_preprocess.cu) each bucket item re-projected: SplatRec + BlendGeo + z key;
//   (sort)      -- stable radix sorts by z key, then by bucket: each bucket in depth order;
//   far_tie_fix -- equal (bucket, 32-bit z key) runs ordered by (float64 z, gaussian index);
// and the continuation blend / the float64 fixups walk the bucket after the near list -- the
// reference's per-tile order (renderer.py:80-101: a tile's splats in (z, index) order) is the near
// list followed by the bucket, since every far z is >= every near z of the env.
#include "sn_common.cuh"
#include "sn_internal.h"

#include <algorithm>

namespace sn {

namespace {

__device__ __forceinline__ uint64_t n_far_of(const FarArgs &f) {
    const uint64_t n = f.env_off[2 * f.ec] - f.env_off[f.ec];
    return n < f.cap_f ? n : f.cap_f;
}

template <bool SCATTER>
__global__ void __launch_bounds__(kBlock) far_bucket_kernel(FarArgs f) {
    const uint64_t n = n_far_of(f);
    const uint64_t i = (uint64_t)blockIdx.x * kBlock + threadIdx.x;
    if (i >= n) return;
    const FarRec r = f.far[i];
    if (r.rect.x > r.rect.y) return;  // reaches no pixel
    const int32_t *bo = f.bucket_of + (int64_t)r.env * f.n_tiles;
    for (int ty = r.rect.z; ty <= r.rect.w; ++ty)
        for (int tx = r.rect.x; tx <= r.rect.y; ++tx) {
            const int32_t u = __ldg(bo + ty * f.tiles_x + tx);
            if (u < 0) continue;
            if (!SCATTER) {
                atomicAdd(f.bcount + u, 1u);
            } else {
                const uint64_t pos = f.boff[u] + atomicAdd(f.bfill + u, 1u);
                if (pos < f.cap_b) {
                    f.items[pos] = (uint32_t)i;
                    f.item_bucket[pos] = (uint32_t)u;
                }
            }
        }
}

// bucket id of each item, in the current (z-sorted) order
__global__ void __launch_bounds__(kBlock) far_bucket_keys_kernel(FarArgs f, const uint32_t *order, uint32_t *keys) {
    const uint64_t n = min(*f.n_items, f.cap_b);
    const uint64_t i = (uint64_t)blockIdx.x * kBlock + threadIdx.x;
    if (i < n) keys[i] = f.item_bucket[order[i]];
}

__device__ __forceinline__ bool far_less(const FarArgs &f, uint32_t a, uint32_t c) {
    const double za = f.brec[a].z, zc = f.brec[c].z;
    if (za != zc) return za < zc;
    return f.far[f.items[a]].gid < f.far[f.items[c]].gid;
}

// Runs of equal (bucket, 32-bit z key) -- one thread per run start -- ordered by (z, gaussian index).
__global__ void __launch_bounds__(kBlock) far_tie_fix_kernel(FarArgs f, const uint32_t *bkeys, uint32_t *order) {
    const int64_t n = (int64_t)min(*f.n_items, f.cap_b);
    const int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    if (i >= n) return;
    auto same = [&](int64_t x, int64_t y) { return bkeys[x] == bkeys[y] && f.zkey[order[x]] == f.zkey[order[y]]; };
    if (i > 0 && same(i - 1, i)) return;
    int64_t e = i + 1;
    while (e < n && same(i, e)) ++e;
    if (e - i < 2) return;
    uint32_t *v = order + i;
    const int64_t L = e - i;
    for (int64_t x = 1; x < L; ++x) {  // insertion sort (runs are short: equal 32-bit depth keys)
        const uint32_t cur = v[x];
        int64_t y = x - 1;
        while (y >= 0 && far_less(f, cur, v[y])) {
            v[y + 1] = v[y];
            --y;
        }
        v[y + 1] = cur;
    }
}

unsigned grid_of(uint64_t cap) { return (unsigned)std::max<uint64_t>(1, (cap + kBlock - 1) / kBlock); }

}  // namespace

cudaError_t launch_far_count(const FarArgs &f, cudaStream_t s) {
    if (f.cap_f == 0) return cudaSuccess;
    far_bucket_kernel<false><<<grid_of(f.cap_f), kBlock, 0, s>>>(f);
    return cudaGetLastError();
}

cudaError_t launch_far_scatter(const FarArgs &f, cudaStream_t s) {
    if (f.cap_f == 0) return cudaSuccess;
    far_bucket_kernel<true><<<grid_of(f.cap_f), kBlock, 0, s>>>(f);
    return cudaGetLastError();
}

cudaError_t launch_far_bucket_keys(const FarArgs &f, const uint32_t *order, uint32_t *keys, cudaStream_t s) {
    if (f.cap_b == 0) return cudaSuccess;
    far_bucket_keys_kernel<<<grid_of(f.cap_b), kBlock, 0, s>>>(f, order, keys);
    return cudaGetLastError();
}

cudaError_t launch_far_tie_fix(const FarArgs &f, const uint32_t *bkeys, uint32_t *order, cudaStream_t s) {
    if (f.cap_b == 0) return cudaSuccess;
    far_tie_fix_kernel<<<grid_of(f.cap_b), kBlock, 0, s>>>(f, bkeys, order);
    return cudaGetLastError();
}

}  // namespace sn
