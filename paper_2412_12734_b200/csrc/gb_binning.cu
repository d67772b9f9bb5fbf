// gb_binning.cu -- K2: tile binning (build_binning, raster.hpp:116-147).
//
//   counts (K1) --CUB inclusive scan--> offsets
//   k_duplicate : one (tile << 32 | depth_bits, k) pair per overlapped tile,
//                 emitted in primitive-index order
//   CUB stable radix sort on the low 32 + ceil(log2 tiles) key bits
//   k_ranges    : per-tile [start, end) into the sorted values
//
// Stability + index-ordered emission reproduce the reference's per-tile
// order "ascending depth_key, ties by index" (raster.hpp:141-145) exactly.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "gb_internal.cuh"

namespace gb {

__global__ void __launch_bounds__(256) k_duplicate(int64_t K, int tiles_x, const uint32_t* __restrict__ offsets,
                                                   const uint2* __restrict__ rects,
                                                   const uint32_t* __restrict__ depth_bits,
                                                   uint64_t* __restrict__ keys, int32_t* __restrict__ values) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= K) return;
    const uint32_t end = offsets[k + 1];
    uint32_t o = offsets[k];
    if (o == end) return;
    const uint2 r = rects[k];
    const int tx0 = r.x & 0xffff, ty0 = r.x >> 16, tx1 = r.y & 0xffff, ty1 = r.y >> 16;
    const uint64_t lo = depth_bits[k];
    for (int ty = ty0; ty <= ty1; ++ty)
        for (int tx = tx0; tx <= tx1; ++tx) {
            keys[o] = ((uint64_t)(ty * tiles_x + tx) << 32) | lo;
            values[o] = (int32_t)k;
            ++o;
        }
}

__global__ void __launch_bounds__(256) k_ranges(int64_t P, const uint64_t* __restrict__ keys,
                                                uint2* __restrict__ ranges) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P) return;
    const uint32_t tile = (uint32_t)(keys[i] >> 32);
    if (i == 0 || (uint32_t)(keys[i - 1] >> 32) != tile) ranges[tile].x = (uint32_t)i;
    if (i == P - 1 || (uint32_t)(keys[i + 1] >> 32) != tile) ranges[tile].y = (uint32_t)(i + 1);
}

size_t scan_temp_bytes(int64_t K) {
    size_t bytes = 0;
    cub::DeviceScan::InclusiveSum(nullptr, bytes, (uint32_t*)nullptr, (uint32_t*)nullptr, (int)K);
    return bytes;
}

size_t sort_temp_bytes(int64_t P) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, (uint64_t*)nullptr, (uint64_t*)nullptr, (int32_t*)nullptr,
                                    (int32_t*)nullptr, (int)P);
    return bytes;
}

// offsets must have K+1 entries; offsets[0] is zeroed here.
cudaError_t launch_scan(void* temp, size_t temp_bytes, const uint32_t* counts, uint32_t* offsets, int64_t K,
                        cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(offsets, 0, sizeof(uint32_t), st);
    if (e != cudaSuccess || K == 0) return e;
    return cub::DeviceScan::InclusiveSum(temp, temp_bytes, counts, offsets + 1, (int)K, st);
}

cudaError_t launch_duplicate(int64_t K, int tiles_x, const uint32_t* offsets, const uint2* rects,
                             const uint32_t* depth_bits, uint64_t* keys, int32_t* values, cudaStream_t st) {
    if (K == 0) return cudaSuccess;
    k_duplicate<<<(unsigned)((K + 255) / 256), 256, 0, st>>>(K, tiles_x, offsets, rects, depth_bits, keys, values);
    return cudaGetLastError();
}

static int bits_for(uint32_t v) {
    int b = 0;
    while (b < 32 && (1ull << b) < (uint64_t)v) ++b;
    return b;
}

// Sorts (keys_in, vals_in) into (keys_out, vals_out).
cudaError_t launch_sort(void* temp, size_t temp_bytes, uint64_t* keys_in, uint64_t* keys_out, int32_t* vals_in,
                        int32_t* vals_out, int64_t P, int n_tiles, cudaStream_t st) {
    if (P == 0) return cudaSuccess;
    const int end_bit = 32 + bits_for((uint32_t)n_tiles);
    return cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys_in, keys_out, vals_in, vals_out, (int)P, 0,
                                           end_bit, st);
}

cudaError_t launch_ranges(int64_t P, const uint64_t* keys, uint2* ranges, int n_tiles, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(ranges, 0, sizeof(uint2) * (size_t)n_tiles, st);
    if (e != cudaSuccess || P == 0) return e;
    k_ranges<<<(unsigned)((P + 255) / 256), 256, 0, st>>>(P, keys, ranges);
    return cudaGetLastError();
}

}  // namespace gb
