// gb_io.cu -- the GBIL splat file (serialize.hpp:15-124) between device SoA
// buffers and disk.
//
// The file is a header plus K little-endian fp32 records, one per primitive
// (array-of-structures); the device SplatSet is structure-of-arrays.  The
// transpose runs on the GPU: k_pack_records gathers the SoA fields into
// record order in HBM, then the records stream to disk through a pinned
// staging buffer in fixed-size chunks; loading is the reverse (pinned chunk
// -> H2D -> k_unpack_records scatter).  Every byte is written by exactly one
// thread with coalesced record-side accesses, so both kernels are HBM-bound.
//
//   version 1 (the reference's, ortho):  x, y, depth_key, theta, log_su, log_sv,
//                                        opacity_logit, n*n*3 grid
//   version 2 (this build's pinhole extension): mx, my, mz, qw, qx, qy, qz,
//                                        log_su, log_sv, opacity_logit, grid
// Header: "GBIL", u32 version, u32 K, u32 N, f32 sigma (serialize.hpp:17-21).
// Error messages follow serialize.hpp:90-124 word for word.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <string>

#include "gb_io.cuh"

namespace gb {

__global__ void __launch_bounds__(256) k_pack_records(int64_t K, RecordMap m, const float* __restrict__ grid,
                                                      float* __restrict__ rec) {
    const int R = m.fields + m.F;
    const int64_t total = K * R;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
        const int64_t k = i / R;
        const int f = (int)(i - k * R);
        float v;
        if (f < m.fields) {
            v = m.src[f][k * m.stride[f] + m.offset[f]];
        } else {
            v = grid[k * m.F + (f - m.fields)];
        }
        rec[i] = v;
    }
}

__global__ void __launch_bounds__(256) k_unpack_records(int64_t K, RecordMap m, float* __restrict__ grid,
                                                        const float* __restrict__ rec) {
    const int R = m.fields + m.F;
    const int64_t total = K * R;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
        const int64_t k = i / R;
        const int f = (int)(i - k * R);
        const float v = rec[i];
        if (f < m.fields) {
            const_cast<float*>(m.src[f])[k * m.stride[f] + m.offset[f]] = v;
        } else {
            grid[k * m.F + (f - m.fields)] = v;
        }
    }
}

RecordMap record_map(int version, const gb_splats* s) {
    RecordMap m;
    std::memset(&m, 0, sizeof(m));
    m.F = 3 * s->grid.n * s->grid.n;
    auto put = [&](const float* p, int stride, int off) {
        m.src[m.fields] = p;
        m.stride[m.fields] = stride;
        m.offset[m.fields] = off;
        ++m.fields;
    };
    if (version == 1) {
        put(s->position, 2, 0);
        put(s->position, 2, 1);
        put(s->depth_key, 1, 0);
        put(s->theta, 1, 0);
    } else {
        for (int j = 0; j < 3; ++j) put(s->position, 3, j);
        for (int j = 0; j < 4; ++j) put(s->quat, 4, j);
    }
    put(s->log_scale, 2, 0);
    put(s->log_scale, 2, 1);
    put(s->opacity_logit, 1, 0);
    return m;
}

cudaError_t launch_pack(int64_t K, const RecordMap& m, const float* grid, float* rec, int sm_count, cudaStream_t st) {
    if (K == 0) return cudaSuccess;
    const int64_t total = K * (m.fields + m.F);
    int64_t blocks = (total + 255) / 256;
    if (blocks > (int64_t)sm_count * 8) blocks = (int64_t)sm_count * 8;
    k_pack_records<<<(unsigned)blocks, 256, 0, st>>>(K, m, grid, rec);
    return cudaGetLastError();
}

cudaError_t launch_unpack(int64_t K, const RecordMap& m, float* grid, const float* rec, int sm_count,
                          cudaStream_t st) {
    if (K == 0) return cudaSuccess;
    const int64_t total = K * (m.fields + m.F);
    int64_t blocks = (total + 255) / 256;
    if (blocks > (int64_t)sm_count * 8) blocks = (int64_t)sm_count * 8;
    k_unpack_records<<<(unsigned)blocks, 256, 0, st>>>(K, m, grid, rec);
    return cudaGetLastError();
}

}  // namespace gb
