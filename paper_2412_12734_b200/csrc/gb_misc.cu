// gb_misc.cu -- K6 (photometric loss -> dL/dC) and K7 (fused Adam).
//
// K6: L1 (the BASELINE configs' loss) and MSE (train.hpp:120-133), one pass:
//     reads color + target, writes the image cotangent, block-reduces the loss.
// K7: adam_step (optim.hpp:96-117) per parameter group, fp32 state; a
//     finite-check pass runs first and, if any gradient is non-finite, the
//     update pass becomes a no-op (the reference throws, optim.hpp:81-83).
#include "gb_internal.cuh"

namespace gb {

template <int KIND>  // 0 = L1, 1 = MSE
__global__ void __launch_bounds__(256) k_loss(const float* __restrict__ color, const float* __restrict__ target,
                                              int64_t n, float scale, float* __restrict__ grad,
                                              float* __restrict__ loss) {
    float acc = 0.0f;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const float d = color[i] - target[i];
        if (KIND == 0) {
            acc += fabsf(d);
            grad[i] = scale * (float)((d > 0.0f) - (d < 0.0f));
        } else {
            acc = fmaf(d, d, acc);
            grad[i] = 2.0f * scale * d;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    __shared__ float s[8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) s[warp] = acc;
    __syncthreads();
    if (warp == 0) {
        acc = lane < (int)(blockDim.x >> 5) ? s[lane] : 0.0f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0 && loss) atomicAdd(loss, acc * scale);
    }
}

cudaError_t launch_loss(int kind, const float* color, const float* target, int64_t n, float scale, float* grad,
                        float* loss, int sm_count, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    int64_t blocks = (n + 255) / 256;
    const int64_t cap = (int64_t)sm_count * 8;
    if (blocks > cap) blocks = cap;
    if (kind == 0)
        k_loss<0><<<(unsigned)blocks, 256, 0, st>>>(color, target, n, scale, grad, loss);
    else
        k_loss<1><<<(unsigned)blocks, 256, 0, st>>>(color, target, n, scale, grad, loss);
    return cudaGetLastError();
}

// first non-finite gradient, encoded (group << 48) | index; ~0 (or INT64_MAX, gb_adam_segments) = none
__global__ void __launch_bounds__(256) k_adam_check(const float* __restrict__ g, int64_t n, int group,
                                                    unsigned long long* __restrict__ bad) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t n4 = ((reinterpret_cast<uintptr_t>(g) & 15) == 0) ? n / 4 : 0;
    const float4* g4 = reinterpret_cast<const float4*>(g);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
        const float4 q = g4[i];
        if (!(isfinite(q.x) && isfinite(q.y) && isfinite(q.z) && isfinite(q.w))) {
            for (int j = 0; j < 4; ++j)
                if (!isfinite(g[4 * i + j]))
                    atomicMin(bad, ((unsigned long long)group << 48) | (unsigned long long)(4 * i + j));
        }
    }
    for (int64_t i = 4 * n4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        if (!isfinite(g[i])) atomicMin(bad, ((unsigned long long)group << 48) | (unsigned long long)i);
    }
}

// optim.hpp:84-88 for one element
// (1 - beta) arrive from the host rounded once from double: 1 - 0.999f in fp32 is 1.3e-5 off.
__device__ __forceinline__ void adam_one(float& p, float gi, float& m, float& v, float lr, float b1, float b2,
                                         float omb1, float omb2, float eps, float inv_bias1, float inv_bias2) {
    const float mi = b1 * m + omb1 * gi;
    const float vi = b2 * v + omb2 * gi * gi;
    m = mi;
    v = vi;
    p -= lr * (mi * inv_bias1) / (sqrtf(vi * inv_bias2) + eps);
}

// HBM-bound: 16-byte vector loads/stores when all four arrays are 16-B aligned (the flat gradient / state
// buffers keep every group 16-B aligned), scalar tail.
__global__ void __launch_bounds__(256) k_adam_update(float* __restrict__ p, const float* __restrict__ g,
                                                     float* __restrict__ m, float* __restrict__ v, int64_t n, float lr,
                                                     float b1, float b2, float omb1, float omb2, float eps,
                                                     float inv_bias1, float inv_bias2,
                                                     const unsigned long long* __restrict__ bad) {
    if (*bad < (1ull << 62)) return;  // a non-finite gradient was found (clear values: ~0 or INT64_MAX)
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const bool vec = ((reinterpret_cast<uintptr_t>(p) | reinterpret_cast<uintptr_t>(g) |
                       reinterpret_cast<uintptr_t>(m) | reinterpret_cast<uintptr_t>(v)) & 15) == 0;
    const int64_t n4 = vec ? n / 4 : 0;
    float4* p4 = reinterpret_cast<float4*>(p);
    const float4* g4 = reinterpret_cast<const float4*>(g);
    float4* m4 = reinterpret_cast<float4*>(m);
    float4* v4 = reinterpret_cast<float4*>(v);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
        float4 pp = p4[i], mm = m4[i], vv = v4[i];
        const float4 gg = g4[i];
        adam_one(pp.x, gg.x, mm.x, vv.x, lr, b1, b2, omb1, omb2, eps, inv_bias1, inv_bias2);
        adam_one(pp.y, gg.y, mm.y, vv.y, lr, b1, b2, omb1, omb2, eps, inv_bias1, inv_bias2);
        adam_one(pp.z, gg.z, mm.z, vv.z, lr, b1, b2, omb1, omb2, eps, inv_bias1, inv_bias2);
        adam_one(pp.w, gg.w, mm.w, vv.w, lr, b1, b2, omb1, omb2, eps, inv_bias1, inv_bias2);
        p4[i] = pp;
        m4[i] = mm;
        v4[i] = vv;
    }
    for (int64_t i = 4 * n4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        adam_one(p[i], g[i], m[i], v[i], lr, b1, b2, omb1, omb2, eps, inv_bias1, inv_bias2);
}

// RGBA-padded texel gradients (K4 with gb_context_set_texel_grad_stride(4)) into the reference layout
__global__ void __launch_bounds__(256) k_texel_unpad(const float4* __restrict__ padded, float* __restrict__ dst,
                                                     int64_t texels, bool accumulate) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < texels; t += (int64_t)gridDim.x * blockDim.x) {
        const float4 g = padded[t];
        float* d = dst + 3 * t;
        if (accumulate) {
            d[0] += g.x;
            d[1] += g.y;
            d[2] += g.z;
        } else {
            d[0] = g.x;
            d[1] = g.y;
            d[2] = g.z;
        }
    }
}

cudaError_t launch_texel_unpad(const float* padded, float* dst, int64_t texels, bool accumulate, int sm_count,
                               cudaStream_t st) {
    if (texels <= 0) return cudaSuccess;
    int64_t blocks = (texels + 255) / 256;
    if (blocks > (int64_t)sm_count * 16) blocks = (int64_t)sm_count * 16;
    k_texel_unpad<<<(unsigned)blocks, 256, 0, st>>>(reinterpret_cast<const float4*>(padded), dst, texels, accumulate);
    return cudaGetLastError();
}

__global__ void __launch_bounds__(256) k_texel_pad(const float* __restrict__ src, float4* __restrict__ dst,
                                                   int64_t texels) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < texels; t += (int64_t)gridDim.x * blockDim.x)
        dst[t] = make_float4(src[3 * t], src[3 * t + 1], src[3 * t + 2], 0.0f);
}

cudaError_t launch_texel_pad(const float* src, float* dst, int64_t texels, int sm_count, cudaStream_t st) {
    if (texels <= 0) return cudaSuccess;
    int64_t blocks = (texels + 255) / 256;
    if (blocks > (int64_t)sm_count * 16) blocks = (int64_t)sm_count * 16;
    k_texel_pad<<<(unsigned)blocks, 256, 0, st>>>(src, reinterpret_cast<float4*>(dst), texels);
    return cudaGetLastError();
}

__global__ void k_adam_flag_init(long long* __restrict__ flag, const int* __restrict__ veto) {
    *flag = (veto && *veto) ? GB_ADAM_FLAG_VETO : GB_ADAM_FLAG_CLEAR;
}

cudaError_t launch_adam_flag_init(int64_t* flag, const int32_t* veto, cudaStream_t st) {
    k_adam_flag_init<<<1, 1, 0, st>>>(reinterpret_cast<long long*>(flag), veto);
    return cudaGetLastError();
}

static unsigned grid_for(int64_t n, int sm_count) {
    int64_t blocks = (n + 255) / 256;
    const int64_t cap = (int64_t)sm_count * 8;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    return (unsigned)blocks;
}

cudaError_t launch_adam_check(const float* g, int64_t n, int group, unsigned long long* bad, int sm_count,
                              cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    k_adam_check<<<grid_for(n, sm_count), 256, 0, st>>>(g, n, group, bad);
    return cudaGetLastError();
}

cudaError_t launch_adam_update(float* p, const float* g, float* m, float* v, int64_t n, float lr, float b1, float b2,
                               float omb1, float omb2, float eps, float inv_bias1, float inv_bias2,
                               const unsigned long long* bad, int sm_count, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    k_adam_update<<<grid_for(n, sm_count), 256, 0, st>>>(p, g, m, v, n, lr, b1, b2, omb1, omb2, eps, inv_bias1,
                                                          inv_bias2, bad);
    return cudaGetLastError();
}

#ifdef GB_PARITY_F64
// parity build: dst += (float)src, one rounding of the fp64 texel-gradient sums
__global__ void __launch_bounds__(256) k_add_f64(const double* __restrict__ src, float* __restrict__ dst, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        if (src[i] != 0.0) dst[i] = (float)((double)dst[i] + src[i]);
}

cudaError_t launch_add_f64(const double* src, float* dst, int64_t n, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    k_add_f64<<<1184, 256, 0, st>>>(src, dst, n);
    return cudaGetLastError();
}
#endif

}  // namespace gb
