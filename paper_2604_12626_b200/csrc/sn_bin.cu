// sn_bin.cu -- K3-K6: depth sort, permute into depth order, tile-pair duplication, pair sort,
// tile-range extraction.
//
// Order contract (renderer.py:80-101 + projection.py:184): within each (env, tile) the splats
// appear in (z, original index) order. The emit stage writes records env-major in index order;
// a stable radix sort on the 64-bit key (env | z_bits - z_base) therefore yields the exact
// lexsort order (the sort runs on the top 32 bits; tie_fix orders equal-key runs by the float64 z
// and index). Pairs are then emitted in (env, depth-rank) order and a stable sort on the tile bits
// alone keeps every (env, tile) group contiguous and in depth order -- the semantics of a 64-bit
// (env | tile | depth) key without sorting the env or depth bits again.
#include "sn_common.cuh"
#include "sn_internal.h"

#include <algorithm>


namespace sn {

namespace {

// Visible splats / tile pairs of the pass, read on the device (clamped to the host capacity: an
// overflowing pass is detected by the host afterwards and re-run with larger buffers).
__device__ __forceinline__ int64_t n_vis_of(const BinArgs &b) {
    const uint64_t n = *b.d_nvis;
    return (int64_t)(n < b.cap_v ? n : b.cap_v);
}
__device__ __forceinline__ int64_t n_pairs_of(const BinArgs &b) {
    const uint64_t n = *b.d_npairs;
    return (int64_t)(n < b.cap_p ? n : b.cap_p);
}

__device__ __forceinline__ ushort4 rect_union(ushort4 a, ushort4 c) {
    return make_ushort4(min(a.x, c.x), max(a.y, c.y), min(a.z, c.z), max(a.w, c.w));
}

__device__ __forceinline__ ushort4 warp_rect_union(ushort4 r) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        ushort4 q;
        q.x = (unsigned short)__shfl_xor_sync(0xffffffffu, (unsigned)r.x, o);
        q.y = (unsigned short)__shfl_xor_sync(0xffffffffu, (unsigned)r.y, o);
        q.z = (unsigned short)__shfl_xor_sync(0xffffffffu, (unsigned)r.z, o);
        q.w = (unsigned short)__shfl_xor_sync(0xffffffffu, (unsigned)r.w, o);
        r = rect_union(r, q);
    }
    return r;
}

// Writes each depth-sorted splat's tile rectangle and tile count and, per 256-splat batch (one
// CTA), the batch's union rectangle for the blend's cull. The 64-byte records themselves stay
// where the emit wrote them: the blend gathers them through the sort's index.
#ifndef SN_PERMUTE_MIN_BLOCKS
#define SN_PERMUTE_MIN_BLOCKS 5
#endif
__global__ void __launch_bounds__(kBlock, SN_PERMUTE_MIN_BLOCKS) permute_kernel(BinArgs b) {
    __shared__ ushort4 s_u[kBlock / 32];
    const int64_t n_vis = n_vis_of(b);
    if ((int64_t)blockIdx.x * kBlock >= n_vis) return;
    int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    ushort4 mine = make_ushort4(0xffff, 0, 0xffff, 0);  // empty
    if (i < n_vis) mine = b.rects_in[b.vals_sorted[i]];
    ushort4 u = warp_rect_union(mine);
    if ((threadIdx.x & 31) == 0) s_u[threadIdx.x >> 5] = u;
    __syncthreads();
    if (threadIdx.x == 0) {
        ushort4 t = s_u[0];
        for (int w = 1; w < kBlock / 32; ++w) t = rect_union(t, s_u[w]);
        b.batch_rects[blockIdx.x] = t;
    }
    if (i >= n_vis) return;
    ushort4 r = mine;
    b.rects_out[i] = r;
    if (b.tiles_touched)
        b.tiles_touched[i] = r.x <= r.y && r.z <= r.w ? (uint32_t)(r.y - r.x + 1) * (uint32_t)(r.w - r.z + 1) : 0u;
}

// Load-balanced pair emission: a CTA owns 256 consecutive depth-sorted splats and spreads
// their (tile) pairs evenly over its threads, so a splat covering all 1,200 tiles does not
// serialize one thread. Writes are contiguous.
__global__ void __launch_bounds__(kBlock) duplicate_kernel(BinArgs b) {
    __shared__ uint64_t s_off[kBlock + 1];
    __shared__ ushort4 s_rect[kBlock];
    __shared__ uint32_t s_env[kBlock];
    const int64_t n_vis = n_vis_of(b);
    int64_t i0 = (int64_t)blockIdx.x * kBlock;
    if (i0 >= n_vis) return;
    int t = threadIdx.x;
    int64_t i = i0 + t;
    int cnt = (int)min((int64_t)kBlock, n_vis - i0);
    if (t < cnt) {
        s_off[t] = b.pair_off[i];
        s_rect[t] = b.rects_out[i];
        uint32_t e = 0;
        while (e + 1 < (uint32_t)b.ec && b.env_off[e + 1] <= (uint64_t)i) ++e;
        s_env[t] = e;
    }
    if (t == 0) s_off[cnt] = b.pair_off[i0 + cnt];
    __syncthreads();
    uint64_t base = s_off[0];
    uint64_t total = s_off[cnt] - base;
    if (base + total > b.cap_p) total = base < b.cap_p ? b.cap_p - base : 0;  // overflow: re-run later
    for (uint64_t k = t; k < total; k += kBlock) {
        uint64_t gk = base + k;
        int lo = 0, hi = cnt - 1;  // last splat with s_off <= gk
        while (lo < hi) {
            int mid = (lo + hi + 1) >> 1;
            if (s_off[mid] <= gk)
                lo = mid;
            else
                hi = mid - 1;
        }
        ushort4 r = s_rect[lo];
        uint32_t local = (uint32_t)(gk - s_off[lo]);
        uint32_t span = (uint32_t)(r.y - r.x + 1);
        uint32_t tx = r.x + local % span, ty = r.z + local / span;
        uint32_t tile = ty * (uint32_t)b.tiles_x + tx;
        SN_ASSERT(gk < b.cap_p && tile < (uint32_t)(b.tiles_x * b.tiles_y));
        b.pair_keys[gk] = (s_env[lo] << b.tile_bits) | tile;
        b.pair_vals[gk] = b.vals_sorted[i0 + lo];  // the record slot: the blend gathers it directly
    }
}

__global__ void __launch_bounds__(kBlock) ranges_kernel(BinArgs b, const uint32_t *keys) {
    const int64_t n = n_pairs_of(b);
    int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    if (i >= n) return;
    uint2 *ranges = b.ranges;
    uint32_t k = keys[i];
    if (i == 0 || keys[i - 1] != k) {
        ranges[k].x = (uint32_t)i;
        if (b.tile_list) b.tile_list[atomicAdd(b.n_list, 1u)] = k;  // a non-empty (env, tile)
    }
    if (i == n - 1 || keys[i + 1] != k) ranges[k].y = (uint32_t)(i + 1);
}

__global__ void __launch_bounds__(kBlock) super_rects_kernel(BinArgs b, ushort4 *super_rects) {
    const ushort4 *batch_rects = b.batch_rects;
    const int64_t n_batches = (n_vis_of(b) + kBlock - 1) / kBlock;
    int64_t sb = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    int64_t b0 = sb * kSuperBatch;
    if (b0 >= n_batches) return;
    ushort4 t = batch_rects[b0];
    for (int64_t k = b0 + 1; k < min(n_batches, b0 + kSuperBatch); ++k) t = rect_union(t, batch_rects[k]);
    super_rects[sb] = t;
}

// The depth sort ran on 32-bit keys (env + top bits of z). Splats whose 32-bit keys tie are
// re-ordered here by the full float64 z, then by slot (= original index, the emit writes in index
// order): the exact np.lexsort((idx, z)) order. Runs are almost always 1-3 long; long runs
// (pathological exact-depth planes) fall back to an in-place heap sort.
// (a spatially reordered scene, sn_cloud.index: the slot order is not the original order -- ties
// compare the original ids the emit wrote, gid)
__device__ __forceinline__ bool z_less(const SplatRec *recs, const uint32_t *gid, uint32_t a, uint32_t c) {
    double za = recs[a].z, zc = recs[c].z;
    return za < zc || (za == zc && (gid ? gid[a] < gid[c] : a < c));
}

// Sorts the run of equal 32-bit keys starting at i by (exact z, index).
__device__ __forceinline__ void tie_fix_run(const BinArgs &b, int64_t i, int64_t n_vis) {
    const uint32_t k = b.keys_sorted[i];
    int64_t e = i + 1;
    while (e < n_vis && b.keys_sorted[e] == k) ++e;
    const int64_t L = e - i;
    if (L < 2) return;
    uint32_t *v = b.vals_sorted + i;
    if (L <= 32) {
        for (int64_t x = 1; x < L; ++x) {  // insertion sort
            uint32_t cur = v[x];
            int64_t y = x - 1;
            while (y >= 0 && z_less(b.recs_un, b.gid_un, cur, v[y])) {
                v[y + 1] = v[y];
                --y;
            }
            v[y + 1] = cur;
        }
        return;
    }
    // heap sort (max-heap by z_less)
    auto sift = [&](int64_t root, int64_t end) {
        while (2 * root + 1 < end) {
            int64_t c = 2 * root + 1;
            if (c + 1 < end && z_less(b.recs_un, b.gid_un, v[c], v[c + 1])) ++c;
            if (!z_less(b.recs_un, b.gid_un, v[root], v[c])) return;
            uint32_t t = v[root];
            v[root] = v[c];
            v[c] = t;
            root = c;
        }
    };
    for (int64_t r = L / 2 - 1; r >= 0; --r) sift(r, L);
    for (int64_t end = L - 1; end > 0; --end) {
        uint32_t t = v[0];
        v[0] = v[end];
        v[end] = t;
        sift(0, end);
    }
}


__global__ void __launch_bounds__(kBlock) tie_fix_kernel(BinArgs b) {
    const int64_t n_vis = n_vis_of(b);
    int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    if (i >= n_vis) return;
    const uint32_t k = b.keys_sorted[i];
    if (i > 0 && b.keys_sorted[i - 1] == k) return;  // not a run start
    tie_fix_run(b, i, n_vis);
}

}  // namespace

// One (chunk, pass)'s sizes into mapped host memory: visible (near) splats, tile pairs and, for a
// depth-sliced pass, far splats (f_hi - f_lo), unfinished tiles and far bucket items.
__global__ void publish_counts_kernel(const uint64_t *v, const uint64_t *p, const unsigned long long *fctl,
                                      volatile uint64_t *dst) {
    dst[0] = *v;
    dst[1] = *p;
    // a sliced scene pass (control words, kFarCtl): far records, unfinished tiles, bucket items, far-short
    dst[2] = fctl ? fctl[4] : 0ull;
    dst[3] = fctl ? fctl[0] : 0ull;
    dst[4] = fctl ? fctl[1] : 0ull;
    dst[5] = fctl ? fctl[3] : 0ull;
}

cudaError_t launch_publish_counts(const uint64_t *v, const uint64_t *p, const unsigned long long *fctl,
                                  uint64_t *mapped_dst, cudaStream_t s) {
    publish_counts_kernel<<<1, 1, 0, s>>>(v, p, fctl, mapped_dst);
    return cudaGetLastError();
}

static unsigned grid_of(uint64_t cap) { return (unsigned)std::max<uint64_t>(1, (cap + kBlock - 1) / kBlock); }

cudaError_t launch_depth_tie_fix(const BinArgs &b, cudaStream_t s) {
    if (b.cap_v == 0) return cudaSuccess;
    tie_fix_kernel<<<grid_of(b.cap_v), kBlock, 0, s>>>(b);
    return cudaGetLastError();
}

cudaError_t launch_super_rects(const BinArgs &b, ushort4 *super_rects, cudaStream_t s) {
    if (b.cap_v == 0) return cudaSuccess;
    const uint64_t n_super = (b.cap_v + (uint64_t)kBlock * kSuperBatch - 1) / ((uint64_t)kBlock * kSuperBatch);
    super_rects_kernel<<<grid_of(n_super), kBlock, 0, s>>>(b, super_rects);
    return cudaGetLastError();
}

cudaError_t launch_permute(const BinArgs &b, cudaStream_t s) {
    if (b.cap_v == 0) return cudaSuccess;
    permute_kernel<<<grid_of(b.cap_v), kBlock, 0, s>>>(b);
    return cudaGetLastError();
}

cudaError_t launch_duplicate(const BinArgs &b, cudaStream_t s) {
    if (b.cap_v == 0) return cudaSuccess;
    duplicate_kernel<<<grid_of(b.cap_v), kBlock, 0, s>>>(b);
    return cudaGetLastError();
}

cudaError_t launch_ranges(const BinArgs &b, const uint32_t *keys_sorted, cudaStream_t s) {
    if (b.cap_p == 0) return cudaSuccess;
    ranges_kernel<<<grid_of(b.cap_p), kBlock, 0, s>>>(b, keys_sorted);
    return cudaGetLastError();
}

}  // namespace sn
