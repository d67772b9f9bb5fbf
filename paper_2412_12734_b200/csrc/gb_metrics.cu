// gb_metrics.cu -- image metrics of the training loop on the GPU:
// SSIM with its gradient (metrics.hpp:98-163, 183-191) and the PSNR sum
// (metrics.hpp:169-179).
//
// SSIM is the Wang 2004 definition the reference uses: 11-tap Gaussian window
// (sigma 1.5, normalised), K1 = 0.01, K2 = 0.03, dynamic range 1,
// valid-region windows only, mean over positions and the three channels.
// Images are HWC fp32 (RenderOutput.color / the target).
//
//   k_ssim_fwd : one CTA per (32 x 16 valid positions, channel).  The
//                (32+10) x (16+10) halo of a and b is staged in shared
//                memory, the five moments (a, b, a^2, b^2, ab) are filtered
//                separably (horizontal pass into shared memory, vertical
//                pass in registers), and each position yields its SSIM term
//                plus, when a gradient is wanted, the three coefficients
//                d/d(mu_a), d/d(E[a^2]), d/d(E[ab]) (metrics.hpp:141-147).
//   k_ssim_bwd : the adjoint of the valid filter (metrics.hpp:66-84
//                scatter_valid) as a tiled "full" correlation of the three
//                coefficient maps, combined per pixel as
//                grad = norm * (S_mu + 2 a S_xx + b S_xy) (metrics.hpp:153-155)
//                and ADDED (times a scale) to the caller's gradient image.
// Both are bandwidth/L1 bound: each input pixel is read by ~1.6 CTAs.
#include <cuda_runtime.h>

#include "gb_internal.cuh"

namespace gb {

constexpr int kSsimTX = 32, kSsimTY = 16, kSsimR = 10;  // window 11 = 1 + 2*5; valid region shrinks by 10

__constant__ float c_ssim_k[11];

static bool g_kernel_ready = false;

static cudaError_t ensure_kernel() {
    if (g_kernel_ready) return cudaSuccess;
    // metrics.hpp:27-40: exp(-d^2 / (2 * 1.5^2)), d = i - 5, normalised (fp64 then rounded)
    double k[11], sum = 0.0;
    for (int i = 0; i < 11; ++i) {
        const double d = i - 5.0;
        k[i] = std::exp(-d * d / (2.0 * 1.5 * 1.5));
        sum += k[i];
    }
    float kf[11];
    for (int i = 0; i < 11; ++i) kf[i] = (float)(k[i] / sum);
    cudaError_t e = cudaMemcpyToSymbol(c_ssim_k, kf, sizeof(kf));
    if (e == cudaSuccess) g_kernel_ready = true;
    return e;
}

__device__ __forceinline__ float clamp01(float v) { return fminf(fmaxf(v, 0.0f), 1.0f); }

__device__ __forceinline__ void block_add_double(double v, double* out) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __shared__ double s[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) s[warp] = v;
    __syncthreads();
    if (warp == 0) {
        v = lane < (int)(blockDim.x >> 5) ? s[lane] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) atomicAdd(out, v);
    }
}

// grid (ceil(OW/TX), ceil(OH/TY), 3), 256 threads
__global__ void __launch_bounds__(256) k_ssim_fwd(const float* __restrict__ a, const float* __restrict__ b, int W,
                                                  int H, int clamp, double inv_count, double* __restrict__ sum,
                                                  float* __restrict__ dcoef) {
    constexpr int IW = kSsimTX + kSsimR, IH = kSsimTY + kSsimR;
    __shared__ float sa[IH][IW], sb[IH][IW];
    __shared__ float hm[5][IH][kSsimTX];
    const int OW = W - kSsimR, OH = H - kSsimR;
    const int c = blockIdx.z;
    const int ox0 = blockIdx.x * kSsimTX, oy0 = blockIdx.y * kSsimTY;
    for (int i = threadIdx.x; i < IW * IH; i += blockDim.x) {
        const int ly = i / IW, lx = i - ly * IW;
        const int x = ox0 + lx, y = oy0 + ly;
        float va = 0.0f, vb = 0.0f;
        if (x < W && y < H) {
            const size_t p = ((size_t)y * W + x) * 3 + c;
            va = a[p];
            vb = b[p];
            if (clamp) {
                va = clamp01(va);
                vb = clamp01(vb);
            }
        }
        sa[ly][lx] = va;
        sb[ly][lx] = vb;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < IH * kSsimTX; i += blockDim.x) {  // horizontal pass
        const int ly = i / kSsimTX, lx = i - ly * kSsimTX;
        float m0 = 0.f, m1 = 0.f, m2 = 0.f, m3 = 0.f, m4 = 0.f;
#pragma unroll
        for (int t = 0; t < 11; ++t) {
            const float k = c_ssim_k[t], x = sa[ly][lx + t], y = sb[ly][lx + t];
            m0 = fmaf(k, x, m0);
            m1 = fmaf(k, y, m1);
            m2 = fmaf(k, x * x, m2);
            m3 = fmaf(k, y * y, m3);
            m4 = fmaf(k, x * y, m4);
        }
        hm[0][ly][lx] = m0;
        hm[1][ly][lx] = m1;
        hm[2][ly][lx] = m2;
        hm[3][ly][lx] = m3;
        hm[4][ly][lx] = m4;
    }
    __syncthreads();
    constexpr float kC1 = 0.01f * 0.01f, kC2 = 0.03f * 0.03f;
    double acc = 0.0;
    for (int i = threadIdx.x; i < kSsimTY * kSsimTX; i += blockDim.x) {  // vertical pass + SSIM terms
        const int ly = i / kSsimTX, lx = i - ly * kSsimTX;
        const int ox = ox0 + lx, oy = oy0 + ly;
        if (ox >= OW || oy >= OH) continue;
        float mx = 0.f, my = 0.f, fxx = 0.f, fyy = 0.f, fxy = 0.f;
#pragma unroll
        for (int t = 0; t < 11; ++t) {
            const float k = c_ssim_k[t];
            mx = fmaf(k, hm[0][ly + t][lx], mx);
            my = fmaf(k, hm[1][ly + t][lx], my);
            fxx = fmaf(k, hm[2][ly + t][lx], fxx);
            fyy = fmaf(k, hm[3][ly + t][lx], fyy);
            fxy = fmaf(k, hm[4][ly + t][lx], fxy);
        }
        // metrics.hpp:130-140
        const float sx = fxx - mx * mx, sy = fyy - my * my, sxy = fxy - mx * my;
        const float a1 = 2.0f * mx * my + kC1, a2 = 2.0f * sxy + kC2;
        const float b1 = mx * mx + my * my + kC1, b2 = sx + sy + kC2;
        const float ib = 1.0f / (b1 * b2);
        const float s = a1 * a2 * ib;
        acc += (double)s;
        if (dcoef) {  // metrics.hpp:141-147
            const size_t q = ((size_t)c * OH + oy) * OW + ox;
            const size_t plane = (size_t)3 * OH * OW;
            dcoef[q] = 2.0f * my * (a2 - a1) * ib + 2.0f * mx * s * (1.0f / b2 - 1.0f / b1);
            dcoef[plane + q] = -s / b2;
            dcoef[2 * plane + q] = 2.0f * a1 * ib;
        }
    }
    block_add_double(acc * inv_count, sum);
}

// grid (ceil(W/TX), ceil(H/TY), 3), 256 threads
__global__ void __launch_bounds__(256) k_ssim_bwd(const float* __restrict__ a, const float* __restrict__ b, int W,
                                                  int H, const float* __restrict__ dcoef, float scale,
                                                  float* __restrict__ grad) {
    constexpr int IW = kSsimTX + kSsimR, IH = kSsimTY + kSsimR;
    __shared__ float sd[3][IH][IW];
    __shared__ float hs[3][IH][kSsimTX];
    const int OW = W - kSsimR, OH = H - kSsimR;
    const size_t plane = (size_t)3 * OH * OW;
    const int c = blockIdx.z;
    const int x0 = blockIdx.x * kSsimTX, y0 = blockIdx.y * kSsimTY;
    // coefficient positions q = p - t, t in [0, 10]: the staged window starts 10 before the tile
    for (int i = threadIdx.x; i < IW * IH; i += blockDim.x) {
        const int ly = i / IW, lx = i - ly * IW;
        const int qx = x0 - kSsimR + lx, qy = y0 - kSsimR + ly;
        float d0 = 0.f, d1 = 0.f, d2 = 0.f;
        if (qx >= 0 && qy >= 0 && qx < OW && qy < OH) {
            const size_t q = ((size_t)c * OH + qy) * OW + qx;
            d0 = dcoef[q];
            d1 = dcoef[plane + q];
            d2 = dcoef[2 * plane + q];
        }
        sd[0][ly][lx] = d0;
        sd[1][ly][lx] = d1;
        sd[2][ly][lx] = d2;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < IH * kSsimTX; i += blockDim.x) {  // horizontal: sum_t k[t] d[px - t]
        const int ly = i / kSsimTX, lx = i - ly * kSsimTX;
        float s0 = 0.f, s1 = 0.f, s2 = 0.f;
#pragma unroll
        for (int t = 0; t < 11; ++t) {
            const float k = c_ssim_k[t];
            s0 = fmaf(k, sd[0][ly][lx + kSsimR - t], s0);
            s1 = fmaf(k, sd[1][ly][lx + kSsimR - t], s1);
            s2 = fmaf(k, sd[2][ly][lx + kSsimR - t], s2);
        }
        hs[0][ly][lx] = s0;
        hs[1][ly][lx] = s1;
        hs[2][ly][lx] = s2;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kSsimTY * kSsimTX; i += blockDim.x) {
        const int ly = i / kSsimTX, lx = i - ly * kSsimTX;
        const int x = x0 + lx, y = y0 + ly;
        if (x >= W || y >= H) continue;
        float s0 = 0.f, s1 = 0.f, s2 = 0.f;
#pragma unroll
        for (int t = 0; t < 11; ++t) {
            const float k = c_ssim_k[t];
            s0 = fmaf(k, hs[0][ly + kSsimR - t][lx], s0);
            s1 = fmaf(k, hs[1][ly + kSsimR - t][lx], s1);
            s2 = fmaf(k, hs[2][ly + kSsimR - t][lx], s2);
        }
        const size_t p = ((size_t)y * W + x) * 3 + c;
        grad[p] += scale * (s0 + 2.0f * a[p] * s1 + b[p] * s2);
    }
}

__global__ void __launch_bounds__(256) k_psnr_sum(const float* __restrict__ a, const float* __restrict__ b, int64_t n,
                                                  double* __restrict__ sum) {
    double acc = 0.0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const double d = (double)clamp01(a[i]) - (double)clamp01(b[i]);  // metrics.hpp:172-173
        acc += d * d;
    }
    block_add_double(acc, sum);
}

// *sum += mean SSIM (channels and valid positions); when grad != nullptr,
// grad += grad_scale * d(mean SSIM)/d(a).  dcoef: 9 * (W-10) * (H-10) floats of scratch.
cudaError_t launch_ssim(const float* a, const float* b, int W, int H, int clamp, double* sum, float* grad,
                        float grad_scale, float* dcoef, cudaStream_t st) {
    cudaError_t e = ensure_kernel();
    if (e != cudaSuccess) return e;
    const int OW = W - kSsimR, OH = H - kSsimR;
    const double inv = 1.0 / (3.0 * (double)OW * (double)OH);
    dim3 g1((OW + kSsimTX - 1) / kSsimTX, (OH + kSsimTY - 1) / kSsimTY, 3);
    k_ssim_fwd<<<g1, 256, 0, st>>>(a, b, W, H, clamp, inv, sum, grad ? dcoef : nullptr);
    e = cudaGetLastError();
    if (e != cudaSuccess || !grad) return e;
    dim3 g2((W + kSsimTX - 1) / kSsimTX, (H + kSsimTY - 1) / kSsimTY, 3);
    k_ssim_bwd<<<g2, 256, 0, st>>>(a, b, W, H, dcoef, (float)(grad_scale * inv), grad);
    return cudaGetLastError();
}

cudaError_t launch_psnr_sum(const float* a, const float* b, int64_t n, double* sum, int sm_count, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    int64_t blocks = (n + 255) / 256;
    if (blocks > (int64_t)sm_count * 4) blocks = (int64_t)sm_count * 4;
    k_psnr_sum<<<(unsigned)blocks, 256, 0, st>>>(a, b, n, sum);
    return cudaGetLastError();
}

}  // namespace gb
