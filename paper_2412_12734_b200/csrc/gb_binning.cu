// gb_binning.cu -- K2: tile binning (build_binning, raster.hpp:116-147) as a
// two-level stable sort.
//
//   depth_bits (K1) --CUB stable radix sort, 32 bits--> perm  (primitives in
//                      (depth, index) order; culled ones carry ~0 and sort last)
//   CUB inclusive scan of the counts read in that order -> offsets
//   k_duplicate      : one (tile id, primitive) pair per overlapped tile,
//                      emitted in (depth, index) order
//   CUB stable radix sort on the ceil(log2 tiles) tile-id bits only
//   k_ranges         : per-tile [start, end) into the sorted values
//
// Both sorts are stable, so inside every tile the pairs stay in (depth_key,
// index) order -- the reference's per-tile order (raster.hpp:141-145) -- and the
// result equals one sort of 64-bit (tile << 32 | depth) keys, bit for bit.  It
// replaces that 45-bit sort over P pairs (6 radix passes of 12 B records) with
// a 32-bit sort over K primitives plus 2 passes of 8 B records over P pairs.
//
// Capacity mode (gb_binning_set_capacity): the host never reads P back.  The
// pair buffers hold `cap` slots, k_pad fills slots [P, cap) with the pad key
// n_tiles (one more key bit at most), the tile sort runs over all cap slots
// and k_ranges ignores pad keys -- so the per-tile ranges are identical and
// the whole build can be captured into a CUDA graph.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include "gb_internal.cuh"

namespace gb {

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

// The scan saturates at kPairLimit = 2^31 - 1 (the sorts index pairs with int): a pair count that would wrap
// the uint32 offsets reads as the limit instead, which the blocking build rejects and the capacity build
// flags as an overflow.  min(a + b, L) is associative for a, b <= L, and a + b < 2^32 cannot wrap.
constexpr uint32_t kPairLimit = 0x7fffffffu;
struct SatAdd {
    __host__ __device__ uint32_t operator()(uint32_t a, uint32_t b) const {
        const uint32_t s = a + b;
        return s < kPairLimit ? s : kPairLimit;
    }
};

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
