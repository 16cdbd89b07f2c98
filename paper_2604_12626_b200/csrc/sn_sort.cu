// sn_sort.cu -- device-wide LSD radix sort (u32 keys + u32 values) and an exclusive scan whose
// item counts live in DEVICE memory, so a render pass queues its whole sequence of kernels without
// a host round trip (grids are sized by the host-side capacity; blocks past the count exit).
//
// Sort, per digit pass (digit width <= 8 bits, passes = ceil(bits / 8)):
//   upsweep   -- each 2048-item tile builds its digit histogram (per-warp shared-memory counters);
//   rowscan   -- one CTA per digit scans that digit's per-tile counts (exclusive) and its total;
//   downsweep -- each tile ranks its items stably (warp peers from one ballot per digit bit, the
//                warp's running count per digit from a returning shared atomic by each peer
//                group's first lane, then a prefix over the tile's warps), stages them in digit
//                order in shared memory and writes each digit's run to digit base + tile offset,
//                coalesced.
// Stable at every level (lane order within a round, round order within a warp's 256-item segment,
// warp order within a tile, tile order in the scan), hence a stable LSD sort. Traffic per pass:
// 4 B/item read (upsweep) + 8 B read + 8 B written (downsweep).
#include "sn_common.cuh"
#include "sn_internal.h"

#include <algorithm>

namespace sn {

namespace {

constexpr int kSortThreads = 256;
#ifndef SN_SORT_ROUNDS
#define SN_SORT_ROUNDS 8
#endif
constexpr int kSortRounds = SN_SORT_ROUNDS;  // items per thread
#ifndef SN_SORT_MATCH
#define SN_SORT_MATCH 0  // downsweep ranks: __match_any_sync peers (1) or digit-bit ballots (0)
#endif
constexpr int kSortTile = kSortThreads * kSortRounds;
constexpr int kRowThreads = 1024;
constexpr unsigned kAll = 0xffffffffu;

__device__ __forceinline__ uint64_t clamp_n(const uint64_t *d_n, uint64_t cap) {
    const uint64_t n = *d_n;
    return n < cap ? n : cap;
}

__global__ void __launch_bounds__(kSortThreads) sort_upsweep(const uint32_t *keys, const uint64_t *d_n, uint64_t cap,
                                                             int shift, int dbits, uint32_t *hist, int n_tiles) {
    __shared__ uint32_t h[kSortThreads / 32][256];
    const int warp = threadIdx.x >> 5;
    const int bins = 1 << dbits;
    for (int i = threadIdx.x; i < (kSortThreads / 32) * 256; i += kSortThreads) (&h[0][0])[i] = 0;
    __syncthreads();
    const uint64_t n = clamp_n(d_n, cap);
    const uint64_t base = (uint64_t)blockIdx.x * kSortTile;
    const uint32_t mask = (uint32_t)bins - 1u;
    if (base < n) {
#pragma unroll
        for (int r = 0; r < kSortRounds; ++r) {
            const uint64_t i = base + (uint64_t)r * kSortThreads + threadIdx.x;
            if (i < n) atomicAdd(&h[warp][(__ldg(keys + i) >> shift) & mask], 1u);
        }
    }
    __syncthreads();
    for (int d = threadIdx.x; d < bins; d += kSortThreads) {
        uint32_t s = 0;
#pragma unroll
        for (int w = 0; w < kSortThreads / 32; ++w) s += h[w][d];
        hist[(int64_t)d * n_tiles + blockIdx.x] = s;
    }
}

// Block-wide exclusive scan of one value per thread (kRowThreads threads); returns the block total.
template <int NT>
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t &excl, uint32_t *s_w) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kAll, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t t = lane < NT / 32 ? s_w[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kAll, t, o);
            if (lane >= o) t += y;
        }
        if (lane < NT / 32) s_w[lane] = t;  // inclusive warp totals
    }
    __syncthreads();
    const uint32_t warp_base = warp > 0 ? s_w[warp - 1] : 0u;
    const uint32_t total = s_w[NT / 32 - 1];
    excl = warp_base + x - v;
    __syncthreads();
    return total;
}

__global__ void __launch_bounds__(kRowThreads) sort_rowscan(uint32_t *hist, int n_tiles, uint32_t *totals) {
    __shared__ uint32_t s_w[32];
    uint32_t *row = hist + (int64_t)blockIdx.x * n_tiles;
    uint32_t run = 0;
    for (int b0 = 0; b0 < n_tiles; b0 += kRowThreads) {
        const int i = b0 + threadIdx.x;
        const uint32_t v = i < n_tiles ? row[i] : 0u;
        uint32_t ex;
        const uint32_t tot = block_exclusive_scan<kRowThreads>(v, ex, s_w);
        if (i < n_tiles) row[i] = run + ex;
        run += tot;
    }
    if (threadIdx.x == 0) totals[blockIdx.x] = run;
}

#ifndef SN_SORT_MIN_BLOCKS
#define SN_SORT_MIN_BLOCKS 5
#endif
__global__ void __launch_bounds__(kSortThreads, SN_SORT_MIN_BLOCKS) sort_downsweep(const uint32_t *kin, const uint32_t *vin, uint32_t *kout,
                                                               uint32_t *vout, const uint64_t *d_n, uint64_t cap,
                                                               int shift, int dbits, const uint32_t *hist,
                                                               const uint32_t *totals, int n_tiles) {
    __shared__ uint32_t s_base[256];
    __shared__ uint32_t s_tstart[256];
    __shared__ uint32_t s_cnt[kSortThreads / 32][256];
    __shared__ uint32_t s_w[kSortThreads / 32];
    __shared__ uint32_t s_k[kSortTile], s_v[kSortTile];
    const uint64_t n = clamp_n(d_n, cap);
    const uint64_t base = (uint64_t)blockIdx.x * kSortTile;
    if (base >= n) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int bins = 1 << dbits;
    const uint32_t mask = (uint32_t)bins - 1u;
    // digit bases: exclusive scan of the digit totals + this tile's offset within each digit
    {
        const uint32_t v = threadIdx.x < bins ? totals[threadIdx.x] : 0u;
        uint32_t ex;
        block_exclusive_scan<kSortThreads>(v, ex, s_w);
        if (threadIdx.x < bins) s_base[threadIdx.x] = ex + hist[(int64_t)threadIdx.x * n_tiles + blockIdx.x];
    }
    for (int i = threadIdx.x; i < (kSortThreads / 32) * 256; i += kSortThreads) (&s_cnt[0][0])[i] = 0;
    __syncthreads();
    uint32_t k[kSortRounds], v[kSortRounds], pos[kSortRounds];
    const uint64_t seg = base + (uint64_t)warp * (32 * kSortRounds);
#pragma unroll
    for (int r = 0; r < kSortRounds; ++r) {
        const uint64_t i = seg + (uint64_t)r * 32 + lane;
        const bool valid = i < n;
        k[r] = valid ? __ldg(kin + i) : 0u;
        v[r] = valid ? (vin ? __ldg(vin + i) : (uint32_t)i) : 0u;  // vin null: identity values
    }
#if SN_SORT_MATCH
#pragma unroll
    for (int r = 0; r < kSortRounds; ++r) {
        const uint64_t i = seg + (uint64_t)r * 32 + lane;
        const bool valid = i < n;
        const uint32_t d = valid ? (k[r] >> shift) & mask : 0xffffu;  // invalid lanes: own peer group
        const unsigned peers = __match_any_sync(kAll, d);
        const uint32_t rank = __popc(peers & ((1u << lane) - 1u));
        const uint32_t before = valid ? s_cnt[warp][d] : 0u;
        __syncwarp();
        if (valid && rank == 0) s_cnt[warp][d] = before + __popc(peers);
        __syncwarp();
        pos[r] = before + rank;
    }
#else
    // Peers (lanes with the same digit) from one ballot per digit bit, and the warp's running count
    // per digit from a returning shared atomic by each peer group's first lane, broadcast by a
    // shuffle: no shared-memory read-modify-write chain between rounds, so they pipeline.
#pragma unroll
    for (int r = 0; r < kSortRounds; ++r) {
        const uint64_t i = seg + (uint64_t)r * 32 + lane;
        const bool valid = i < n;
        const uint32_t d = (k[r] >> shift) & mask;
        unsigned peers = __ballot_sync(kAll, valid);
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            if (b < dbits) {
                const unsigned bal = __ballot_sync(kAll, (d >> b) & 1u);
                peers &= ((d >> b) & 1u) ? bal : ~bal;
            }
        }
        const int leader = __ffs(peers) - 1;  // (invalid lanes: any; their result is unused)
        uint32_t before = 0u;
        if (valid && lane == leader) before = atomicAdd(&s_cnt[warp][d], (uint32_t)__popc(peers));
        before = __shfl_sync(kAll, before, leader < 0 ? lane : leader);
        pos[r] = before + __popc(peers & ((1u << lane) - 1u));
    }
#endif
    __syncthreads();
    uint32_t tile_cnt = 0;
    if (threadIdx.x < bins) {  // per digit: prefix over the tile's warps, and the tile's count
#pragma unroll
        for (int w = 0; w < kSortThreads / 32; ++w) {
            const uint32_t c = s_cnt[w][threadIdx.x];
            s_cnt[w][threadIdx.x] = tile_cnt;
            tile_cnt += c;
        }
    }
    __syncthreads();
    {  // where each digit's run starts inside the tile
        uint32_t ex;
        block_exclusive_scan<kSortThreads>(threadIdx.x < bins ? tile_cnt : 0u, ex, s_w);
        if (threadIdx.x < bins) s_tstart[threadIdx.x] = ex;
    }
    __syncthreads();
    // stage the tile in digit order in shared memory, then write each digit's run out with
    // consecutive threads on consecutive addresses (coalesced)
#pragma unroll
    for (int r = 0; r < kSortRounds; ++r) {
        const uint64_t i = seg + (uint64_t)r * 32 + lane;
        if (i >= n) continue;
        const uint32_t d = (k[r] >> shift) & mask;
        const uint32_t l = s_tstart[d] + s_cnt[warp][d] + pos[r];
        s_k[l] = k[r];
        s_v[l] = v[r];
    }
    __syncthreads();
    const int tile_n = (int)min((uint64_t)kSortTile, n - base);
    for (int l = threadIdx.x; l < tile_n; l += kSortThreads) {
        const uint32_t key = s_k[l];
        const uint32_t d = (key >> shift) & mask;
        const uint32_t g = s_base[d] + (uint32_t)l - s_tstart[d];
        kout[g] = key;
        vout[g] = s_v[l];
    }
}

// ---- exclusive scan u32 -> u64 over n (device) items, n + 1 outputs (out[n] = total) ----
constexpr int kScanChunk = 4096;  // items per CTA (256 threads x 16)

__global__ void __launch_bounds__(256) scan_reduce(const uint32_t *in, const uint64_t *d_n, uint64_t cap,
                                                   uint64_t *sums) {
    __shared__ uint64_t s_w[8];
    const uint64_t n = clamp_n(d_n, cap);
    const uint64_t base = (uint64_t)blockIdx.x * kScanChunk;
    uint64_t s = 0;
    if (base < n) {
        for (int r = 0; r < kScanChunk / 256; ++r) {
            const uint64_t i = base + (uint64_t)r * 256 + threadIdx.x;
            if (i < n) s += __ldg(in + i);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kAll, s, o);
    if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t t = 0;
        for (int w = 0; w < 8; ++w) t += s_w[w];
        sums[blockIdx.x] = t;
    }
}

// one CTA: chunk sums -> exclusive chunk bases (in place), total -> *total
__global__ void __launch_bounds__(1024) scan_chunks(uint64_t *sums, int n_chunks, uint64_t *total) {
    __shared__ uint64_t s_w[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint64_t run = 0;
    for (int b0 = 0; b0 < n_chunks; b0 += 1024) {
        const int i = b0 + threadIdx.x;
        const uint64_t v = i < n_chunks ? sums[i] : 0ull;
        uint64_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t y = __shfl_up_sync(kAll, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_w[warp] = x;
        __syncthreads();
        if (warp == 0) {
            uint64_t t = s_w[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint64_t y = __shfl_up_sync(kAll, t, o);
                if (lane >= o) t += y;
            }
            s_w[lane] = t;
        }
        __syncthreads();
        const uint64_t wb = warp > 0 ? s_w[warp - 1] : 0ull;
        if (i < n_chunks) sums[i] = run + wb + x - v;
        run += s_w[31];
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = run;
}

__global__ void __launch_bounds__(256) scan_down(const uint32_t *in, const uint64_t *d_n, uint64_t cap,
                                                 const uint64_t *bases, const uint64_t *total, uint64_t *out) {
    __shared__ uint64_t s_w[8];
    const uint64_t n = clamp_n(d_n, cap);
    const uint64_t base = (uint64_t)blockIdx.x * kScanChunk;
    if (base > n) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // each thread owns 16 consecutive items
    const uint64_t t0 = base + (uint64_t)threadIdx.x * (kScanChunk / 256);
    uint32_t v[kScanChunk / 256];
    uint64_t s = 0;
#pragma unroll
    for (int r = 0; r < kScanChunk / 256; ++r) {
        const uint64_t i = t0 + r;
        v[r] = i < n ? __ldg(in + i) : 0u;
        s += v[r];
    }
    uint64_t x = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(kAll, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    uint64_t wb = 0;
    for (int w = 0; w < warp; ++w) wb += s_w[w];
    uint64_t run = bases[blockIdx.x] + wb + x - s;
#pragma unroll
    for (int r = 0; r < kScanChunk / 256; ++r) {
        const uint64_t i = t0 + r;
        if (i < n) out[i] = run;
        run += v[r];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) out[n] = *total;
}

}  // namespace

// ---- host wrappers ----

size_t sort_temp_bytes(uint64_t cap) {
    const uint64_t tiles = (cap + kSortTile - 1) / kSortTile;
    return sizeof(uint32_t) * (256 * std::max<uint64_t>(tiles, 1) + 256);
}

// Sorts (keys, values) by the low `bits` key bits, stably; n = min(*d_n, cap) (identity_values: the
// values are the positions 0..n-1 and v0 is never read; k_in: pass 0 reads the keys there and k0 is
// scratch). Passes alternate
// between the two buffer pairs starting with (k0, v0) -> (k1, v1); returns true when the sorted
// result ends in (k1, v1) (odd pass count), false when it is back in (k0, v0).
bool radix_sort_pairs(void *temp, uint32_t *k0, uint32_t *v0, uint32_t *k1, uint32_t *v1, const uint64_t *d_n,
                      uint64_t cap, int bits, cudaStream_t s, int64_t *launches, bool identity_values,
                      const uint32_t *k_in) {
    if (cap == 0 || bits <= 0) return false;
    const int passes = (bits + 7) / 8;
    const int dbits = (bits + passes - 1) / passes;
    const int n_tiles = (int)((cap + kSortTile - 1) / kSortTile);
    uint32_t *hist = static_cast<uint32_t *>(temp);
    uint32_t *totals = hist + (size_t)256 * n_tiles;
    uint32_t *ks = k0, *vs = v0, *kd = k1, *vd = v1;
    for (int p = 0; p < passes; ++p) {
        const uint32_t *vin = (p == 0 && identity_values) ? nullptr : vs;  // pass 0: values = positions
        const uint32_t *kin = (p == 0 && k_in) ? k_in : ks;  // pass 0 may read the keys from elsewhere
        const int shift = p * dbits;
        const int db = std::min(dbits, bits - shift);
        sort_upsweep<<<n_tiles, kSortThreads, 0, s>>>(kin, d_n, cap, shift, db, hist, n_tiles);
        sort_rowscan<<<1 << db, kRowThreads, 0, s>>>(hist, n_tiles, totals);
        sort_downsweep<<<n_tiles, kSortThreads, 0, s>>>(kin, vin, kd, vd, d_n, cap, shift, db, hist, totals, n_tiles);
        if (launches) *launches += 3;
        std::swap(ks, kd);
        std::swap(vs, vd);
    }
    return passes % 2 == 1;
}

size_t scan_temp_bytes_dev(uint64_t cap) {
    return sizeof(uint64_t) * ((cap + kScanChunk) / kScanChunk + 2);
}

// out[i] = sum_{j < i} in[j] for i <= n (n + 1 outputs), n = min(*d_n, cap); *total_out = out[n].
cudaError_t scan_u32_to_u64(void *temp, const uint32_t *in, const uint64_t *d_n, uint64_t cap, uint64_t *out,
                            uint64_t *total_out, cudaStream_t s, int64_t *launches) {
    const int n_chunks = (int)(cap / kScanChunk + 1);
    uint64_t *sums = static_cast<uint64_t *>(temp);
    scan_reduce<<<n_chunks, 256, 0, s>>>(in, d_n, cap, sums);
    scan_chunks<<<1, 1024, 0, s>>>(sums, n_chunks, total_out);
    scan_down<<<n_chunks, 256, 0, s>>>(in, d_n, cap, sums, total_out, out);
    if (launches) *launches += 3;
    return cudaGetLastError();
}

}  // namespace sn
