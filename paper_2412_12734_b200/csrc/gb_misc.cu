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

// first non-finite gradient, encoded (group << 48) | index; ~0 = none
__global__ void __launch_bounds__(256) k_adam_check(const float* __restrict__ g, int64_t n, int group,
                                                    unsigned long long* __restrict__ bad) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        if (!isfinite(g[i])) atomicMin(bad, ((unsigned long long)group << 48) | (unsigned long long)i);
    }
}

__global__ void __launch_bounds__(256) k_adam_update(float* __restrict__ p, const float* __restrict__ g,
                                                     float* __restrict__ m, float* __restrict__ v, int64_t n, float lr,
                                                     float b1, float b2, float eps, float inv_bias1, float inv_bias2,
                                                     const unsigned long long* __restrict__ bad) {
    if (*bad != ~0ull) return;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const float gi = g[i];
        const float mi = b1 * m[i] + (1.0f - b1) * gi;
        const float vi = b2 * v[i] + (1.0f - b2) * gi * gi;
        m[i] = mi;
        v[i] = vi;
        const float m_hat = mi * inv_bias1;
        const float v_hat = vi * inv_bias2;
        p[i] -= lr * m_hat / (sqrtf(v_hat) + eps);
    }
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
                               float eps, float inv_bias1, float inv_bias2, const unsigned long long* bad,
                               int sm_count, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    k_adam_update<<<grid_for(n, sm_count), 256, 0, st>>>(p, g, m, v, n, lr, b1, b2, eps, inv_bias1, inv_bias2, bad);
    return cudaGetLastError();
}

}  // namespace gb
