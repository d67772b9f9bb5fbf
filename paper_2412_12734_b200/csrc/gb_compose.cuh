// gb_compose.cuh -- device helpers shared by the K3/K4 compositor variants
// (gb_raster.cu: staged + direct one-pixel-per-thread; gb_composite.cu:
// multi-pixel-per-thread): bilinear set-up (texture.hpp:27-66), warp
// reductions and the global red helpers of the backward.
#pragma once

#include "gb_internal.cuh"

namespace gb {

constexpr unsigned kFull = 0xffffffffu;

template <int NT>
__device__ __forceinline__ int tex_n(int n_rt) {
    return NT ? NT : n_rt;
}

struct Bilin {
    int t00;  // texel index of (i_u, i_v)
    int o00;  // offset of texel (i_u, i_v) channel 0
    real fu, fv;
    real w00, w10, w01, w11;
};

__device__ __forceinline__ void bilin_setup(real u, real v, int N, const RasterConst& rc, Bilin& b) {
    int iu, iv;
    real s = fma_rn(u, rc.tex_scale, rc.tex_offset);
    s = rmin(rmax(s, (real)0), (real)(N - 1));
    iu = min((int)rfloor(s), N - 2);
    b.fu = sub_rn(s, (real)iu);
    real t = fma_rn(v, rc.tex_scale, rc.tex_offset);
    t = rmin(rmax(t, (real)0), (real)(N - 1));
    iv = min((int)rfloor(t), N - 2);
    b.fv = sub_rn(t, (real)iv);
    b.t00 = iu * N + iv;
    b.o00 = b.t00 * 3;
    GB_CHECK(N >= 2 && b.t00 >= 0 && b.t00 + N + 1 < N * N);
    const real gu = (real)1 - b.fu, gv = (real)1 - b.fv;
    b.w00 = gu * gv;
    b.w10 = b.fu * gv;
    b.w01 = gu * b.fv;
    b.w11 = b.fu * b.fv;
}

// Warp sum of NV <= 16 per-lane values through a per-warp shared-memory
// transpose (scratch: kRedRows x kRedStride floats): lane l writes value i
// to row i, column l; lane l then sums half (l & 1) of row l >> 1 with four
// conflict-free 128-bit loads and one shuffle.  ~NV + 22 instructions
// versus ~4 NV for a shuffle butterfly.  Returns the row l >> 1 total.
constexpr int kRedRows = 16;
constexpr int kRedStride = 36;  // 32 lanes + 4 pad: rows land in distinct bank quads

template <int NV>
__device__ __forceinline__ float smem_reduce(const float (&v)[NV], float* scratch, int lane) {
    __syncwarp();  // previous readers of the scratch are done
#pragma unroll
    for (int i = 0; i < NV; ++i) scratch[i * kRedStride + lane] = v[i];
    __syncwarp();
    const int row = lane >> 1;
    float acc = 0.0f;
    if (row < NV) {
        const float4* q = reinterpret_cast<const float4*>(scratch + row * kRedStride + (lane & 1) * 16);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float4 a = q[k];
            acc += (a.x + a.y) + (a.z + a.w);
        }
    }
    return acc + __shfl_xor_sync(kFull, acc, 1);
}

// fp64 (parity build): the same transpose, scalar loads
template <int NV>
__device__ __forceinline__ double smem_reduce(const double (&v)[NV], double* scratch, int lane) {
    __syncwarp();
#pragma unroll
    for (int i = 0; i < NV; ++i) scratch[i * kRedStride + lane] = v[i];
    __syncwarp();
    const int row = lane >> 1;
    double acc = 0.0;
    if (row < NV) {
        const double* q = scratch + row * kRedStride + (lane & 1) * 16;
#pragma unroll
        for (int k = 0; k < 16; ++k) acc += q[k];
    }
    return acc + __shfl_xor_sync(kFull, acc, 1);
}

__device__ __forceinline__ void red_add(real* p, real v) {
    if (v != (real)0) atomicAdd(p, v);
}

#ifdef GB_PARITY_F64
__device__ __forceinline__ void red3(double* p, double a, double b, double c) {
    atomicAdd(p, a);
    atomicAdd(p + 1, b);
    atomicAdd(p + 2, c);
}
__device__ __forceinline__ void red4(double* p, double a, double b, double c, double d) {
    red3(p, a, b, c);
    atomicAdd(p + 3, d);
}
__device__ __forceinline__ void red2(double* p, double a, double b) {
    atomicAdd(p, a);
    atomicAdd(p + 1, b);
}
#else
// p[0..2] += (a, b, c): one 8-byte vector red and one scalar red (branch-free on alignment)
__device__ __forceinline__ void red3(float* p, float a, float b, float c) {
    const bool even = (reinterpret_cast<uintptr_t>(p) & 7) == 0;
    float2* pv = reinterpret_cast<float2*>(even ? p : p + 1);
    atomicAdd(pv, even ? make_float2(a, b) : make_float2(b, c));
    atomicAdd(even ? p + 2 : p, even ? c : a);
}

// p[0..3] += (a, b, c, d) with one 16-byte vector red (p 16-B aligned)
__device__ __forceinline__ void red4(float* p, float a, float b, float c, float d) {
    atomicAdd(reinterpret_cast<float4*>(p), make_float4(a, b, c, d));
}

// p[0..1] += (a, b) with one 8-byte vector red (p 8-B aligned)
__device__ __forceinline__ void red2(float* p, float a, float b) {
    atomicAdd(reinterpret_cast<float2*>(p), make_float2(a, b));
}
#endif

// texel corner k (0..3 = 00, 10, 01, 11) channel c -> float offset from the base texel
__device__ __forceinline__ int corner_offset(int i, int N) {
    const int k = i / 3, c = i - 3 * (i / 3);
    return ((k & 1) ? 3 * N : 0) + ((k & 2) ? 3 : 0) + c;
}

// true when the entry's alpha-box misses the warp's pixel block for certain
__device__ __forceinline__ bool box_miss(const float4& box, float bx0, float bx1, float by0, float by1) {
    return box.y < bx0 || box.x > bx1 || box.w < by0 || box.z > by1;
}

// True unless the entry's alpha-skip ellipse (K1 alpha_ellipse) certainly
// misses the pixel-index rectangle [x0, x1] x [y0, y1].  Exact for an
// ellipse: the minimum of the quadratic form over the rectangle is at the
// centre when the centre is inside, else on a rectangle edge that faces the
// centre; each candidate edge is minimised in closed form.
__device__ __forceinline__ bool ellipse_meets_rect(const float4 a, const float4 b, float x0, float x1, float y0,
                                                   float y1) {
    const float ax = x0 - a.x, bx = x1 - a.x, ay = y0 - a.y, by = y1 - a.y;
    const bool inx = ax <= 0.0f && bx >= 0.0f;
    const bool iny = ay <= 0.0f && by >= 0.0f;
    const float xe = ax > 0.0f ? ax : bx;  // facing vertical edge
    const float ye = ay > 0.0f ? ay : by;  // facing horizontal edge
    const float dy1 = fminf(fmaxf(-b.y * xe, ay), by);
    const float dx2 = fminf(fmaxf(-b.z * ye, ax), bx);
    const float q1 = a.z * xe * xe + 2.0f * b.x * xe * dy1 + a.w * dy1 * dy1;
    const float q2 = a.z * dx2 * dx2 + 2.0f * b.x * dx2 * ye + a.w * ye * ye;
    return (inx && iny) || (!inx && q1 <= 1.0f) || (!iny && q2 <= 1.0f);
}

}  // namespace gb
