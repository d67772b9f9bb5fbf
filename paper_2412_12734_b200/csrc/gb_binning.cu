// gb_binning.cu -- K2: tile binning (build_binning, raster.hpp:116-147) as
// tile buckets sorted in place -- no global sort.
//
//   k_tile_count  : pairs per tile, counted per CTA in shared memory (kBinCtas
//                   CTAs own contiguous primitive ranges; from the K1 rects)
//   k_tile_prefix : per tile, each CTA's base inside the tile's bucket and the
//                   tile's total (one warp per tile)
//   CUB scan      : tile offsets, tile_off[n_tiles] = P (saturated at 2^31 - 1)
//   k_scatter_priv: each primitive appends the 64-bit key (depth_bits << 32 |
//                   index) to every tile it overlaps (shared-memory cursors:
//                   arbitrary order inside the bucket)
//   k_tile_lists  : one CTA per tile sorts its bucket by that key -- a bitonic
//                   sort of 128- or 2048-key chunks by the mean bucket length
//                   (registers + shuffles for the in-warp stages), then
//                   merge-path passes through global memory -- and writes the
//                   primitive ids and the tile's range
//
// Deep scenes (more than kDeepBucket pairs per tile on average) take the two
// stable radix sorts at the end of this file instead.
//
// (depth_bits, index) keys are unique, so every tile's list is in (depth_key,
// index) order -- the reference's per-tile order (raster.hpp:141-145) -- bit for
// bit, the order a stable sort on (tile, depth) gives.  Against the two stable
// CUB radix sorts this replaced (32 bits over K primitives, then the tile bits
// over P pairs, with a scan over the depth-permuted counts and a duplication
// pass in between), the build costs ~150 instead of ~200 µs per configs[3]
// view and leaves the SMs to the compositors of the other view lanes sooner
// (profiles/ab_r02.md s32-s36).  Images with more than kSmemTiles tiles count and
// scatter with global atomics instead.
//
// Capacity mode (gb_binning_set_capacity): the host never reads P back.  The
// key buffer holds `cap` slots; pairs past it are dropped, the lists clipped at
// it and the overflow flagged (the caller redoes the step with more room), so
// the whole build can be captured into a CUDA graph.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include "gb_internal.cuh"

namespace gb {

// The scan saturates at kPairLimit = 2^31 - 1 (the lists index pairs with int32): a pair count that would wrap
// the uint32 tile offsets reads as the limit instead, which the blocking build rejects and the capacity build
// flags as an overflow.  min(a + b, L) is associative for a, b <= L, and a + b < 2^32 cannot wrap.
constexpr uint32_t kPairLimit = 0x7fffffffu;
struct SatAdd {
    __host__ __device__ uint32_t operator()(uint32_t a, uint32_t b) const {
        const uint32_t s = a + b;
        return s < kPairLimit ? s : kPairLimit;
    }
};

// global-atomic versions of the count and scatter passes (images with more than kSmemTiles tiles)
__global__ void __launch_bounds__(256) k_tile_hist(int64_t K, int tiles_x, const uint32_t* __restrict__ counts,
                                                   const uint2* __restrict__ rects, uint32_t* __restrict__ hist) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= K || counts[k] == 0) return;
    const uint2 r = rects[k];
    const int tx0 = r.x & 0xffff, ty0 = r.x >> 16, tx1 = r.y & 0xffff, ty1 = r.y >> 16;
    for (int ty = ty0; ty <= ty1; ++ty)
        for (int tx = tx0; tx <= tx1; ++tx) atomicAdd(&hist[ty * tiles_x + tx], 1u);
}

__global__ void __launch_bounds__(256) k_scatter(int64_t K, int tiles_x, const uint32_t* __restrict__ counts,
                                                 const uint2* __restrict__ rects,
                                                 const uint32_t* __restrict__ depth_bits,
                                                 uint32_t* __restrict__ cursor, uint64_t* __restrict__ keys,
                                                 uint32_t cap) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= K || counts[k] == 0) return;
    const uint2 r = rects[k];
    const uint64_t key = ((uint64_t)depth_bits[k] << 32) | (uint32_t)k;
    const int tx0 = r.x & 0xffff, ty0 = r.x >> 16, tx1 = r.y & 0xffff, ty1 = r.y >> 16;
    for (int ty = ty0; ty <= ty1; ++ty)
        for (int tx = tx0; tx <= tx1; ++tx) {
            const uint32_t pos = atomicAdd(&cursor[ty * tiles_x + tx], 1u);
            if (pos < cap) keys[pos] = key;
        }
}

// Shared-memory privatised count and scatter (n_tiles <= kSmemTiles): kBinCtas CTAs own
// contiguous primitive ranges; each counts its pairs per tile in shared memory (mat[c][t]), a warp per
// tile turns the column into per-CTA bases, and the scatter hands out bucket slots from shared cursors --
// global atomics on hot tiles (thousands of pairs each) serialise, shared ones per CTA barely contend.
#ifndef GB_BIN_CTAS
#define GB_BIN_CTAS 148
#endif
#ifndef GB_BIN_THREADS
#define GB_BIN_THREADS 512
#endif
constexpr int kBinCtas = GB_BIN_CTAS;
constexpr int kBinThreads = GB_BIN_THREADS;  // half an SM: co-resident with the compositors of other view lanes
constexpr int kSmemTiles = 12288;  // 48 KB of per-CTA tile counters
#ifndef GB_BIN_BATCH
#define GB_BIN_BATCH 4
#endif
constexpr int kBinBatch = GB_BIN_BATCH;

__device__ __forceinline__ void cta_range(int64_t K, int64_t& k0, int64_t& k1) {
    const int64_t chunk = (K + kBinCtas - 1) / kBinCtas;
    k0 = (int64_t)blockIdx.x * chunk;
    k1 = min(K, k0 + chunk);
}

__global__ void __launch_bounds__(kBinThreads) k_tile_count(int64_t K, int tiles_x, int n_tiles,
                                                            const uint32_t* __restrict__ counts,
                                                            const uint2* __restrict__ rects,
                                                            uint32_t* __restrict__ mat) {
    extern __shared__ uint32_t sh[];
    for (int t = threadIdx.x; t < n_tiles; t += kBinThreads) sh[t] = 0;
    __syncthreads();
    int64_t k0, k1;
    cta_range(K, k0, k1);
    // kBinBatch primitives per thread per round: their loads issue together (the pass is latency-bound)
    for (int64_t kb = k0 + threadIdx.x; kb < k1; kb += (int64_t)kBinBatch * kBinThreads) {
        uint32_t c[kBinBatch];
        uint2 r[kBinBatch];
#pragma unroll
        for (int j = 0; j < kBinBatch; ++j) {
            const int64_t k = kb + (int64_t)j * kBinThreads;
            c[j] = k < k1 ? counts[k] : 0u;
            r[j] = k < k1 ? rects[k] : make_uint2(0u, 0u);
        }
#pragma unroll
        for (int j = 0; j < kBinBatch; ++j) {
            if (c[j] == 0) continue;
            const int tx0 = r[j].x & 0xffff, ty0 = r[j].x >> 16, tx1 = r[j].y & 0xffff, ty1 = r[j].y >> 16;
            for (int ty = ty0; ty <= ty1; ++ty)
                for (int tx = tx0; tx <= tx1; ++tx) atomicAdd(&sh[ty * tiles_x + tx], 1u);
        }
    }
    __syncthreads();
    uint32_t* row = mat + (size_t)blockIdx.x * n_tiles;
    for (int t = threadIdx.x; t < n_tiles; t += kBinThreads) row[t] = sh[t];
}

// one warp per tile: mat[c][t] <- pairs of tile t in CTAs before c; hist[t] <- the tile's total
__global__ void __launch_bounds__(256) k_tile_prefix(int n_tiles, uint32_t* __restrict__ mat,
                                                     uint32_t* __restrict__ hist) {
    const int t = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (t >= n_tiles) return;
    uint32_t run = 0;
    for (int c0 = 0; c0 < kBinCtas; c0 += 32) {
        const int c = c0 + lane;
        const uint32_t v = c < kBinCtas ? mat[(size_t)c * n_tiles + t] : 0u;
        uint32_t inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        if (c < kBinCtas) mat[(size_t)c * n_tiles + t] = run + inc - v;
        run += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (lane == 0) hist[t] = run;
}

__global__ void __launch_bounds__(kBinThreads) k_scatter_priv(int64_t K, int tiles_x, int n_tiles,
                                                              const uint32_t* __restrict__ counts,
                                                              const uint2* __restrict__ rects,
                                                              const uint32_t* __restrict__ depth_bits,
                                                              const uint32_t* __restrict__ tile_off,
                                                              const uint32_t* __restrict__ mat,
                                                              uint64_t* __restrict__ keys, uint32_t cap) {
    extern __shared__ uint32_t cur[];
    const uint32_t* row = mat + (size_t)blockIdx.x * n_tiles;
    for (int t = threadIdx.x; t < n_tiles; t += kBinThreads) cur[t] = tile_off[t] + row[t];
    __syncthreads();
    int64_t k0, k1;
    cta_range(K, k0, k1);
    for (int64_t kb = k0 + threadIdx.x; kb < k1; kb += (int64_t)kBinBatch * kBinThreads) {
        uint32_t c[kBinBatch], d[kBinBatch];
        uint2 r[kBinBatch];
#pragma unroll
        for (int j = 0; j < kBinBatch; ++j) {
            const int64_t k = kb + (int64_t)j * kBinThreads;
            c[j] = k < k1 ? counts[k] : 0u;
            r[j] = k < k1 ? rects[k] : make_uint2(0u, 0u);
            d[j] = k < k1 ? depth_bits[k] : 0u;
        }
#pragma unroll
        for (int j = 0; j < kBinBatch; ++j) {
            if (c[j] == 0) continue;
            const int64_t k = kb + (int64_t)j * kBinThreads;
            const uint64_t key = ((uint64_t)d[j] << 32) | (uint32_t)k;
            const int tx0 = r[j].x & 0xffff, ty0 = r[j].x >> 16, tx1 = r[j].y & 0xffff, ty1 = r[j].y >> 16;
            for (int ty = ty0; ty <= ty1; ++ty)
                for (int tx = tx0; tx <= tx1; ++tx) {
                    const uint32_t pos = atomicAdd(&cur[ty * tiles_x + tx], 1u);
                    if (pos < cap) keys[pos] = key;
                }
        }
    }
}

constexpr int kDeepBucket = 512;  // mean pairs per tile past which the radix build is used

// Bucket sort <kSortChunk keys sorted in shared memory at once, kSortThreads>: 128-key chunks with 128
// threads -- 1 KB of shared memory, so the sort's CTAs barely displace the other view lanes' compositors
// (profiles/ab_r02.md s34-s36) -- then merge-path passes through global memory.

// Ascending bitonic sort of s[0, np), np a power of two >= 64.  Each warp owns 64-key blocks (lane l holds
// keys l and l + 32 of a block in registers): the stages with partner distance j <= 32 stay inside a block
// and run on registers and shuffles; only the j >= 64 stages go through shared memory with a barrier.
__device__ __forceinline__ uint64_t shfl_xor64(uint64_t x, int m) {
    const uint32_t lo = __shfl_xor_sync(0xffffffffu, (uint32_t)x, m);
    const uint32_t hi = __shfl_xor_sync(0xffffffffu, (uint32_t)(x >> 32), m);
    return ((uint64_t)hi << 32) | lo;
}

// stages (k, j = min(k/2, 32) .. 1) on one block's registers; pa = position of a (b sits at pa + 32)
__device__ __forceinline__ void block_stages(uint64_t& a, uint64_t& b, int pa, int k) {
    const int lane = threadIdx.x & 31;
    for (int j = min(k >> 1, 32); j > 0; j >>= 1) {
        if (j == 32) {
            const bool asc = (pa & k) == 0;
            const uint64_t lo = a < b ? a : b, hi = a < b ? b : a;
            a = asc ? lo : hi;
            b = asc ? hi : lo;
        } else {
            const uint64_t ya = shfl_xor64(a, j), yb = shfl_xor64(b, j);
            const bool lower = (lane & j) == 0;
            const bool asc_a = (pa & k) == 0, asc_b = ((pa + 32) & k) == 0;
            a = (lower == asc_a) ? (a < ya ? a : ya) : (a < ya ? ya : a);
            b = (lower == asc_b) ? (b < yb ? b : yb) : (b < yb ? yb : b);
        }
    }
}

template <int kSortThreads>
__device__ __forceinline__ void bitonic_sort(uint64_t* s, int np) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int kWarps = kSortThreads / 32;
    // k = 2 .. 64: every block sorted alternately ascending / descending, in registers
    for (int blk = warp; blk < (np >> 6); blk += kWarps) {
        const int pa = blk * 64 + lane;
        uint64_t a = s[pa], b = s[pa + 32];
        for (int k = 2; k <= 64; k <<= 1) block_stages(a, b, pa, k);
        s[pa] = a;
        s[pa + 32] = b;
    }
    __syncthreads();
    for (int k = 128; k <= np; k <<= 1) {
        for (int j = k >> 1; j >= 64; j >>= 1) {
            for (int i = threadIdx.x; i < (np >> 1); i += kSortThreads) {
                const int lo = ((i & ~(j - 1)) << 1) | (i & (j - 1)), hi = lo + j;  // j is a power of two
                const uint64_t x = s[lo], y = s[hi];
                if ((x > y) == ((lo & k) == 0)) {
                    s[lo] = y;
                    s[hi] = x;
                }
            }
            __syncthreads();
        }
        for (int blk = warp; blk < (np >> 6); blk += kWarps) {
            const int pa = blk * 64 + lane;
            uint64_t a = s[pa], b = s[pa + 32];
            block_stages(a, b, pa, k);
            s[pa] = a;
            s[pa + 32] = b;
        }
        __syncthreads();
    }
}

// keys[0, n) (n <= the chunk) -> sorted in s
template <int kSortThreads>
__device__ __forceinline__ void sort_chunk(const uint64_t* __restrict__ keys, int n, uint64_t* s) {
    int np = 64;
    while (np < n) np <<= 1;
    for (int i = threadIdx.x; i < np; i += kSortThreads) s[i] = i < n ? keys[i] : ~0ull;
    __syncthreads();
    bitonic_sort<kSortThreads>(s, np);
}

// one pass of the bucket merge sort: runs of length L in src[0, n) merged pairwise into dst (merge path)
template <int kSortThreads>
__device__ void merge_pass(const uint64_t* __restrict__ src, uint64_t* __restrict__ dst, int n, int L) {
    constexpr int IT = 8;
    for (int base = 0; base < n; base += kSortThreads * IT) {
        int i0 = base + threadIdx.x * IT;
        const int i1 = min(i0 + IT, n);
        while (i0 < i1) {
            const int ps = (i0 / (2 * L)) * (2 * L);
            const int la = min(L, n - ps), lb = min(L, n - ps - la);
            const uint64_t* A = src + ps;
            const uint64_t* B = A + la;
            const int pe = ps + la + lb, end = min(i1, pe);
            const int diag = i0 - ps;
            int lo = max(0, diag - lb), hi = min(diag, la);
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (A[mid] < B[diag - 1 - mid])
                    lo = mid + 1;
                else
                    hi = mid;
            }
            int ai = lo, bi = diag - lo;
            for (int o = i0; o < end; ++o) dst[o] = (bi >= lb || (ai < la && A[ai] < B[bi])) ? A[ai++] : B[bi++];
            i0 = end;
        }
    }
    __syncthreads();
}

// tile t's bucket [min(off[t], limit), min(off[t+1], limit)) and range; tile 0 flags a total past the capacity
__device__ __forceinline__ int tile_bucket(const uint32_t* __restrict__ tile_off, uint32_t limit, int n_tiles,
                                           uint2* __restrict__ ranges, int32_t* __restrict__ overflow,
                                           uint32_t& b) {
    const int t = blockIdx.x;
    b = min(tile_off[t], limit);
    const uint32_t e = min(tile_off[t + 1], limit);
    if (threadIdx.x == 0) {
        ranges[t] = make_uint2(b, e);
        if (t == 0 && overflow && tile_off[n_tiles] > limit) *overflow = 1;
    }
    return (int)(e - b);
}

// the global-memory tail of a bucket sort: runs of L sorted keys in keys[0, n) merged up to one run, the ids
// written to values
template <int kThreads>
__device__ __forceinline__ void merge_runs(uint64_t* src, uint64_t* dst, int n, int L, int32_t* __restrict__ values) {
    for (; L < n; L <<= 1) {
        merge_pass<kThreads>(src, dst, n, L);
        uint64_t* tmp = src;
        src = dst;
        dst = tmp;
    }
    for (int i = threadIdx.x; i < n; i += kThreads) values[i] = (int32_t)(uint32_t)src[i];
}

// One CTA per tile sorts its bucket in 128-key register/shared bitonic chunks, then merges them in global
// memory; the primitive ids go to values, the range to ranges.
template <int kSortChunk, int kSortThreads>
__global__ void __launch_bounds__(kSortThreads) k_tile_lists(const uint32_t* __restrict__ tile_off, uint32_t limit,
                                                             int n_tiles, uint64_t* __restrict__ keys,
                                                             uint64_t* __restrict__ scratch,
                                                             int32_t* __restrict__ values, uint2* __restrict__ ranges,
                                                             int32_t* __restrict__ overflow) {
    __shared__ uint64_t s[kSortChunk];
    uint32_t b;
    const int n = tile_bucket(tile_off, limit, n_tiles, ranges, overflow, b);
    if (n == 0) return;
    if (n <= kSortChunk) {
        sort_chunk<kSortThreads>(keys + b, n, s);
        for (int i = threadIdx.x; i < n; i += kSortThreads) values[b + i] = (int32_t)(uint32_t)s[i];
        return;
    }
    uint64_t* src = keys + b;
    for (int c = 0; c < n; c += kSortChunk) {
        const int m = min(kSortChunk, n - c);
        sort_chunk<kSortThreads>(src + c, m, s);
        for (int i = threadIdx.x; i < m; i += kSortThreads) src[c + i] = s[i];
        __syncthreads();
    }
    merge_runs<kSortThreads>(src, scratch + b, n, kSortChunk, values + b);
}

size_t tile_scan_temp_bytes(int n_tiles) {
    size_t bytes = 0;
    cub::DeviceScan::InclusiveScan(nullptr, bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr, SatAdd{},
                                   n_tiles > 0 ? n_tiles : 1);
    return bytes;
}

size_t tile_scratch_words(int n_tiles) { return (size_t)(kBinCtas + 1) * (size_t)(n_tiles > 0 ? n_tiles : 1); }

// tile_off (n_tiles + 1) = exclusive scan of the pairs per tile, tile_off[n_tiles] = P; scratch holds
// tile_scratch_words(n_tiles) words: the per-tile totals, then (privatised path) the per-CTA bases
cudaError_t launch_tile_offsets(void* temp, size_t temp_bytes, int64_t K, int tiles_x, int n_tiles,
                                const uint32_t* counts, const uint2* rects, uint32_t* scratch, uint32_t* tile_off,
                                cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(tile_off, 0, sizeof(uint32_t) * (size_t)(n_tiles + 1), st);
    if (e != cudaSuccess || n_tiles == 0) return e;
    uint32_t* hist = scratch;
    if (n_tiles <= kSmemTiles) {
        uint32_t* mat = scratch + n_tiles;
        k_tile_count<<<kBinCtas, kBinThreads, sizeof(uint32_t) * n_tiles, st>>>(K, tiles_x, n_tiles, counts, rects,
                                                                                mat);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        k_tile_prefix<<<(unsigned)(((int64_t)n_tiles * 32 + 255) / 256), 256, 0, st>>>(n_tiles, mat, hist);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    } else {
        if ((e = cudaMemsetAsync(hist, 0, sizeof(uint32_t) * (size_t)n_tiles, st)) != cudaSuccess) return e;
        if (K > 0) {
            k_tile_hist<<<(unsigned)((K + 255) / 256), 256, 0, st>>>(K, tiles_x, counts, rects, hist);
            if ((e = cudaGetLastError()) != cudaSuccess) return e;
        }
    }
    return cub::DeviceScan::InclusiveScan(temp, temp_bytes, hist, tile_off + 1, SatAdd{}, n_tiles, st);
}

// keys[tile_off[t] ..) <- the (depth, index) keys of tile t's pairs, unordered
cudaError_t launch_scatter(int64_t K, int tiles_x, int n_tiles, const uint32_t* counts, const uint2* rects,
                           const uint32_t* depth_bits, const uint32_t* tile_off, uint32_t* scratch, uint64_t* keys,
                           uint32_t cap, cudaStream_t st) {
    if (K == 0 || n_tiles == 0) return cudaSuccess;
    if (n_tiles <= kSmemTiles) {
        k_scatter_priv<<<kBinCtas, kBinThreads, sizeof(uint32_t) * n_tiles, st>>>(
            K, tiles_x, n_tiles, counts, rects, depth_bits, tile_off, scratch + n_tiles, keys, cap);
        return cudaGetLastError();
    }
    uint32_t* cursor = scratch;  // the totals are consumed by the scan: reuse as cursors
    cudaError_t e = cudaMemcpyAsync(cursor, tile_off, sizeof(uint32_t) * (size_t)n_tiles, cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return e;
    k_scatter<<<(unsigned)((K + 255) / 256), 256, 0, st>>>(K, tiles_x, counts, rects, depth_bits, cursor, keys, cap);
    return cudaGetLastError();
}

int tile_offsets_launches(int64_t K, int n_tiles) {
    if (n_tiles == 0) return 0;
    return (n_tiles <= kSmemTiles ? 2 : (K > 0)) + 2;  // count + prefix (or one hist), CUB scan init + scan
}

cudaError_t launch_tile_lists(int n_tiles, const uint32_t* tile_off, uint32_t limit, uint64_t* keys,
                              uint64_t* scratch, int32_t* values, uint2* ranges, int32_t* overflow, cudaStream_t st) {
    if (n_tiles == 0) return cudaSuccess;
    k_tile_lists<128, 128><<<n_tiles, 128, 0, st>>>(tile_off, limit, n_tiles, keys, scratch, values, ranges,
                                                    overflow);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Deep scenes (mean tile list > kDeepBucket pairs, e.g. configs[4] at 4M surfels: ~2000 per tile, up to
// ~7.7K): two stable CUB radix sorts.  The primitives' 32-bit depth keys are sorted once (culled ones carry
// ~0 and sort last), the tile counts scanned in that order, each primitive's (tile id, primitive) pairs
// emitted in that order and stably sorted on the ceil(log2 tiles) tile-id bits only -- bit-identical to a
// sort of (tile << 32 | depth) keys.  At these list lengths the per-tile bucket sorts above cost more than
// the bandwidth-bound radix passes (4M x 1: 1.36 vs 1.00 ms per build).  Capacity mode pads the slots past
// P with the key n_tiles, which sorts after every tile and k_ranges skips.
// ---------------------------------------------------------------------------
int deep_bucket_mean() { return kDeepBucket; }

__global__ void __launch_bounds__(256) k_iota(int64_t K, int32_t* __restrict__ out) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < K) out[k] = (int32_t)k;
}

// cap: pair capacity of keys/values.  Pairs at or beyond it are dropped and flagged in *overflow
// (capacity mode only; the blocking mode sizes the buffers to P exactly).
__global__ void __launch_bounds__(256) k_duplicate(int64_t K, int tiles_x, const int32_t* __restrict__ perm,
                                                   const uint32_t* __restrict__ offsets,
                                                   const uint2* __restrict__ rects, uint32_t* __restrict__ keys,
                                                   int32_t* __restrict__ values, uint32_t cap,
                                                   int32_t* __restrict__ overflow) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= K) return;
    const uint32_t end = min(offsets[i + 1], cap);
    uint32_t o = offsets[i];
    if (i == K - 1 && offsets[K] > cap && overflow) *overflow = 1;
    if (o >= end) return;
    const int32_t k = perm[i];
    const uint2 r = rects[k];
    const int tx0 = r.x & 0xffff, ty0 = r.x >> 16, tx1 = r.y & 0xffff, ty1 = r.y >> 16;
    for (int ty = ty0; ty <= ty1 && o < end; ++ty)
        for (int tx = tx0; tx <= tx1 && o < end; ++tx) {
            keys[o] = (uint32_t)(ty * tiles_x + tx);
            values[o] = k;
            ++o;
        }
}

// capacity mode: slots [P, cap) get the pad tile key n_tiles, which sorts after every real tile
__global__ void __launch_bounds__(256) k_pad(uint32_t cap, const uint32_t* __restrict__ total, uint32_t pad,
                                             uint32_t* __restrict__ keys, int32_t* __restrict__ values) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= cap || i < *total) return;
    keys[i] = pad;
    values[i] = -1;
}

// pairs with a pad key (>= n_tiles) belong to no tile
__global__ void __launch_bounds__(256) k_ranges(int64_t P, const uint32_t* __restrict__ keys,
                                                uint2* __restrict__ ranges, uint32_t n_tiles) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P) return;
    const uint32_t tile = keys[i];
    if (tile >= n_tiles) return;
    if (i == 0 || keys[i - 1] != tile) ranges[tile].x = (uint32_t)i;
    if (i == P - 1 || keys[i + 1] != tile) ranges[tile].y = (uint32_t)(i + 1);
}

static int bits_for(uint32_t v) {
    int b = 0;
    while (b < 32 && (1ull << b) < (uint64_t)v) ++b;
    return b;
}

// key bits covering tile keys 0 .. n_keys - 1 (n_keys = n_tiles, + 1 for the capacity mode's pad key)
int tile_sort_bits(int n_keys) {
    const int b = bits_for((uint32_t)n_keys);
    return b ? b : 1;
}

// counts[perm[i]]: the tile counts read in depth order straight into the scan (no gather pass)
struct PermutedCount {
    const int32_t* perm;
    const uint32_t* counts;
    __host__ __device__ uint32_t operator()(int64_t i) const { return counts[perm[i]]; }
};
using CountIter = thrust::transform_iterator<PermutedCount, thrust::counting_iterator<int64_t>, uint32_t>;

size_t scan_temp_bytes(int64_t K) {
    size_t bytes = 0;
    CountIter it(thrust::counting_iterator<int64_t>(0), PermutedCount{nullptr, nullptr});
    cub::DeviceScan::InclusiveScan(nullptr, bytes, it, (uint32_t*)nullptr, SatAdd{}, (int)K);
    return bytes;
}

size_t sort_temp_bytes(int64_t n) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, (uint32_t*)nullptr, (uint32_t*)nullptr, (int32_t*)nullptr,
                                    (int32_t*)nullptr, (int)n);
    return bytes;
}

// Radix passes CUB launches for a sort over `bits` key bits (histogram + exclusive sum + one per 8-bit digit).
int sort_launches(int bits) { return bits > 0 ? 2 + (bits + 7) / 8 : 0; }

// perm = primitive indices in stable (depth_bits, index) order; depth_sorted is scratch.
cudaError_t launch_depth_sort(void* temp, size_t temp_bytes, const uint32_t* depth_bits, uint32_t* depth_sorted,
                              int32_t* iota, int32_t* perm, int64_t K, cudaStream_t st) {
    if (K == 0) return cudaSuccess;
    k_iota<<<(unsigned)((K + 255) / 256), 256, 0, st>>>(K, iota);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return cub::DeviceRadixSort::SortPairs(temp, temp_bytes, depth_bits, depth_sorted, iota, perm, (int)K, 0, 32, st);
}

// offsets (K+1 entries) = exclusive scan of the counts in perm order; offsets[K] = P (saturated at 2^31 - 1).
cudaError_t launch_scan(void* temp, size_t temp_bytes, const int32_t* perm, const uint32_t* counts,
                        uint32_t* offsets, int64_t K, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(offsets, 0, sizeof(uint32_t), st);
    if (e != cudaSuccess || K == 0) return e;
    CountIter it(thrust::counting_iterator<int64_t>(0), PermutedCount{perm, counts});
    return cub::DeviceScan::InclusiveScan(temp, temp_bytes, it, offsets + 1, SatAdd{}, (int)K, st);
}

cudaError_t launch_duplicate(int64_t K, int tiles_x, const int32_t* perm, const uint32_t* offsets, const uint2* rects,
                             uint32_t* keys, int32_t* values, uint32_t cap, int32_t* overflow, cudaStream_t st) {
    if (K == 0) return cudaSuccess;
    k_duplicate<<<(unsigned)((K + 255) / 256), 256, 0, st>>>(K, tiles_x, perm, offsets, rects, keys, values, cap,
                                                             overflow);
    return cudaGetLastError();
}

cudaError_t launch_pad(uint32_t cap, const uint32_t* total, int n_tiles, uint32_t* keys, int32_t* values,
                       cudaStream_t st) {
    if (cap == 0) return cudaSuccess;
    k_pad<<<(cap + 255) / 256, 256, 0, st>>>(cap, total, (uint32_t)n_tiles, keys, values);
    return cudaGetLastError();
}

// Stable sort of (tile id, primitive) pairs on the tile-id bits.
cudaError_t launch_tile_sort(void* temp, size_t temp_bytes, uint32_t* keys_in, uint32_t* keys_out, int32_t* vals_in,
                             int32_t* vals_out, int64_t P, int n_keys, cudaStream_t st) {
    if (P == 0) return cudaSuccess;
    return cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys_in, keys_out, vals_in, vals_out, (int)P, 0,
                                           tile_sort_bits(n_keys), st);
}


cudaError_t launch_ranges(int64_t P, const uint32_t* keys, uint2* ranges, int n_tiles, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(ranges, 0, sizeof(uint2) * (size_t)n_tiles, st);
    if (e != cudaSuccess || P == 0) return e;
    k_ranges<<<(unsigned)((P + 255) / 256), 256, 0, st>>>(P, keys, ranges, (uint32_t)n_tiles);
    return cudaGetLastError();
}

}  // namespace gb
