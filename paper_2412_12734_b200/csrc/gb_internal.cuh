// gb_internal.cuh -- shared device-side definitions for the sm_100a kernels.
//
// Data layout in HBM (all fp32 unless noted):
//   params   : the caller's SplatSet SoA (gb_splats)                       40 B + 12n^2 B / primitive
//   headers  : ScreenHeader[K], 48 B, written by K1 for binned primitives
//   rects    : uint2[K] packed tile rectangle (tx0|ty0<<16, tx1|ty1<<16)
//   counts   : uint32[K] tiles per primitive
//   depth    : uint32[K] orderable fp32 depth bits (~0 when culled)
//   perm     : int32[K] primitives in stable (depth, index) order
//   offsets  : uint32[K+1] exclusive scan of the counts in perm order
//   keys     : uint32[P] tile id per (tile, primitive) pair, stably sorted
//   values   : int32[P] primitive index per pair (per tile: depth, index order)
//   ranges   : uint2[tiles] [start, end) into values per tile
//   accum    : real[K*12] per-primitive screen-space gradient sums (K4 -> K5)
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/gb_raster.h"

namespace gb {

// The compositors' arithmetic type.  The product is fp32 throughout.  The test-only parity build
// (-DGB_PARITY_F64, libgb_raster_f64.so, never loaded by the product) runs the same K3/K4/K5 code in fp64
// -- headers, evaluation, compositing, rewind, adjoint and every accumulation -- so the parity tests can
// hold each gradient entry to rtol 1e-4 / atol 1e-5 with no cancellation exemption: that build differs
// from the reference's fp64 path (raster.hpp:198-387) only in summation order.
#ifdef GB_PARITY_F64
typedef double real;
typedef double4 real4;
#else
typedef float real;
typedef float4 real4;
#endif

// Debug build (-DGB_DEBUG_CHECKS, libgb_raster_debug.so; tests/test_gpu_debug_checks.py): bounds checks on
// list entries, primitive ids, tile keys and texel indices that trap (a launch error) instead of reading or
// writing out of range.  compute-sanitizer is closed on the GPU pool, so this is the memory-safety net.
#ifdef GB_DEBUG_CHECKS
#define GB_CHECK(c)          \
    do {                     \
        if (!(c)) __trap();  \
    } while (0)
#else
#define GB_CHECK(c) \
    do {            \
    } while (0)
#endif

constexpr int kAccumStride = 12;  // values per primitive in the K4 -> K5 accumulator
constexpr real kMaxAlpha = (real)0.999;  // core.hpp:16

// Per-primitive screen header (three real4 + the alpha-box; 64 B in the product).
//   ortho  : h0 = (x, y, cos t, sin t)   h1 = (1/s_u, 1/s_v, alpha_k, 0)   h2 = 0
//   pinhole: the ray-splat intersection as a linear-fractional map of the
//            pixel offset (dx, dy) from the projected centre:
//              (u, v, 1) ~ (X.x dx + Y.x dy,  X.y dx + Y.y dy,  1 + X.z dx + Y.z dy)
//            with X = Cx/(E_z fx), Y = Cy/(E_z fy) precomputed in fp64 (K1):
//            h0 = (X.x, X.y, X.z, Y.x)  h1 = (Y.y, Y.z, alpha_k, hx)
//            h2 = (hy, int cxi, int cyi, 0); dx = (x - cxi) + hx, dy = (y - cyi) + hy.
//   both   : h3 = (x0, x1, y0, y1) the inclusive pixel box outside which
//            alpha < alpha_skip for certain (fp64 AABB of the alpha-skip
//            ellipse, enlarged by a safety margin) -- filled only in the
//            -DGB_CULL_BOX variant, whose compositors test it; the product
//            tests the alpha-skip ellipse of the cull record instead.
struct __align__(16) ScreenHeader {
    real4 h0, h1, h2;
    float4 h3;
};

// integers stored in header slots (pinhole centre): bit-cast in fp32, exact values in fp64
__device__ __forceinline__ int hdr_int(float v) { return __float_as_int(v); }
__device__ __forceinline__ int hdr_int(double v) { return (int)v; }
__device__ __forceinline__ real hdr_from_int(int i) {
#ifdef GB_PARITY_F64
    return (double)i;
#else
    return __int_as_float(i);
#endif
}

// vector header loads through the read-only path
__device__ __forceinline__ float4 ld_real4(const float4* p) { return __ldg(p); }
__device__ __forceinline__ double4 ld_real4(const double4* p) {
    const double2 a = __ldg(reinterpret_cast<const double2*>(p)), b = __ldg(reinterpret_cast<const double2*>(p) + 1);
    return make_double4(a.x, a.y, b.x, b.y);
}

// pinned-rounding arithmetic for both precisions
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float fma_rn(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double fma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float rmin(float a, float b) { return fminf(a, b); }
__device__ __forceinline__ double rmin(double a, double b) { return fmin(a, b); }
__device__ __forceinline__ float rmax(float a, float b) { return fmaxf(a, b); }
__device__ __forceinline__ double rmax(double a, double b) { return fmax(a, b); }
__device__ __forceinline__ float rabs(float a) { return fabsf(a); }
__device__ __forceinline__ double rabs(double a) { return fabs(a); }
__device__ __forceinline__ float rfloor(float a) { return floorf(a); }
__device__ __forceinline__ double rfloor(double a) { return floor(a); }

// Per-primitive alpha-skip ellipse in pixel-index coordinates (K1, alpha_ellipse):
// a = (e_x, e_y, Q11, Q22), b = (Q12, Q12/Q22, Q12/Q11, 0).
struct __align__(16) CullRec {
    float4 a, b;
};

// Per-launch camera constants for the compositor.
struct CamConst {
    int width, height;
    float inv_fx, inv_fy;
    real bg[3];
};

// Raster constants shared by K3/K4.
struct RasterConst {
    int tile_size;
    int tiles_x, tiles_y;
    real alpha_skip;      // <= 0 disables
    real early_stop;      // the early-termination threshold, or -1 when disabled (T >= 0 never falls below it)
    real tex_scale;       // (n-1)/(2 sigma)
    real tex_offset;      // (n-1)/2
    real sigma;
    int tgs;  // K4 texel-gradient stride: 3 = the reference layout, 4 = RGBA-padded (one 16-B red per texel)
    const float4* tex4;  // non-null: K3/K4 read the texels from this RGBA-padded copy (gb_context_set_texel_rgba)
#ifdef GB_DEBUG_CHECKS
    int64_t dbg_K;  // primitives: every list entry must be in [0, K)
#endif
#ifdef GB_PARITY_F64
    double* trans64;  // parity build: K3 stores the fp64 final transmittance here, K4 rewinds from it
#endif
};

// Thread -> pixel mapping inside a tile.  For tile sizes that are multiples
// of 8 with ts*ts a multiple of 32, each warp covers an 8x4 pixel block
// (better texel/activity coherence); otherwise row-major.
__device__ __forceinline__ void tile_pixel(int tid, int ts, int& lx, int& ly) {
    if ((ts & 7) == 0) {
        const int warp = tid >> 5, lane = tid & 31;
        const int wx = ts >> 3;  // warps per row of 8-wide blocks
        lx = (warp % wx) * 8 + (lane & 7);
        ly = (warp / wx) * 4 + (lane >> 3);
    } else {
        lx = tid % ts;
        ly = tid / ts;
    }
}

// ---- the per-(pixel, entry) evaluation shared bit-for-bit by K3 and K4 ------
// Explicit _rn intrinsics pin the rounding sequence so forward and backward
// make identical alpha-skip decisions (the reference needs
// -ffp-contract=off for the same reason, CMakeLists.txt:12-15).

struct PinholeTerms {  // kept for the backward chain
    real dx, dy, cz, iz;
};

// Approximate reciprocal (one MUFU.RCP, ~1 ulp).  It is deterministic, so K3
// and K4 still see identical bits; only the oracle comparison is
// tolerance-based, and 1 ulp is far inside it.
__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ double rcp_approx(double x) { return __drcp_rn(x); }

// raster.hpp:36-42 (ortho) -- returns true (always a hit).
__device__ __forceinline__ bool eval_uv_ortho(const ScreenHeader& h, int x, int y, real& u, real& v) {
    const real dx = sub_rn(add_rn((real)x, (real)0.5), h.h0.x);
    const real dy = sub_rn(add_rn((real)y, (real)0.5), h.h0.y);
    const real c = h.h0.z, s = h.h0.w;
    u = mul_rn(fma_rn(c, dx, mul_rn(s, dy)), h.h1.x);
    v = mul_rn(fma_rn(-s, dx, mul_rn(c, dy)), h.h1.y);
    return true;
}

// Pinhole 2DGS ray-splat intersection in the centred
// linear-fractional form above.  A miss (ray parallel to the plane, or the
// plane hit behind the camera: c_z <= 0 after the K1 normalisation) is skipped;
// c_z below FLT_MIN (a hit at ~infinity, G = 0 anyway) counts as a miss so the
// flush-to-zero reciprocal never sees a denormal.
__device__ __forceinline__ bool eval_uv_pinhole(const ScreenHeader& h, int x, int y, real& u, real& v,
                                                PinholeTerms& p) {
    const int cxi = hdr_int(h.h2.y), cyi = hdr_int(h.h2.z);
    p.dx = add_rn((real)(x - cxi), h.h1.w);
    p.dy = add_rn((real)(y - cyi), h.h2.x);
    const real cx = fma_rn(p.dx, h.h0.x, mul_rn(p.dy, h.h0.w));
    const real cy = fma_rn(p.dx, h.h0.y, mul_rn(p.dy, h.h1.x));
    p.cz = fma_rn(p.dx, h.h0.z, fma_rn(p.dy, h.h1.y, (real)1));
    p.iz = rcp_approx(p.cz);
    u = mul_rn(cx, p.iz);
    v = mul_rn(cy, p.iz);
    return p.cz > (real)1.17549435e-38f;
}

// G = exp(-(u^2+v^2)/2)  (raster.hpp:52) as one MUFU.EX2 of -(u^2+v^2) log2(e)/2
// (ftz: G underflows to 0 far outside the splat, where alpha < alpha_skip anyway).
__device__ __forceinline__ float gauss_weight(float u, float v) {
    const float x = __fmul_rn(-0.72134752044448170368f, __fmaf_rn(u, u, __fmul_rn(v, v)));
    float g;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(g) : "f"(x));
    return g;
}
__device__ __forceinline__ double gauss_weight(double u, double v) { return exp(-0.5 * (u * u + v * v)); }

// K1/K5 parameters (fp64 camera and config), passed by value.
struct ProjParams {
    int mode;
    int n;
    int64_t K;
    const float* position;
    const float* depth_key;
    const float* theta;
    const float* quat;
    const float* log_scale;
    const float* opacity;
    int W, H;
    double fx, fy, cx, cy;
    double inv_fx, inv_fy;  // 1/fx, 1/fy (K5)
    double R[9];
    double t[3];
    double near_plane;
    int ts, tiles_x, tiles_y;
    double cutoff, alpha_skip;
};

ProjParams make_proj_params(const gb_splats* s, const gb_camera* cam, const gb_raster_config* cfg, int tiles_x,
                            int tiles_y);
cudaError_t launch_project(const ProjParams& p, ScreenHeader* hdr, CullRec* cull, uint2* rects, uint32_t* counts,
                           uint32_t* depth_bits, cudaStream_t st);
cudaError_t launch_chain(const ProjParams& p, const uint32_t* counts, const real* accum, const gb_grads& g,
                         cudaStream_t st);

// gb_raster.cu: K3 with the photometric loss in its epilogue (K3 + K6); the single fused K3+K6+K4 kernel
// exists only in the -DGB_FUSED_SINGLE_KERNEL variant build
cudaError_t launch_forward_loss(int mode, int n, int tiles, int ts, const uint2* ranges, const int32_t* values,
                                const ScreenHeader* hdr, const CullRec* cull, const float* tex, const CamConst& cc,
                                const RasterConst& rc, int kind, const float* target, float scale, float* color,
                                float* trans, int32_t* last, float* image_grad, float* loss, cudaStream_t st);
#ifdef GB_FUSED_SINGLE_KERNEL
cudaError_t launch_fused(int mode, int n, int tiles, int ts, const uint2* ranges, const int32_t* values,
                         const ScreenHeader* hdr, const CullRec* cull, const float* tex, const CamConst& cc,
                         const RasterConst& rc, int kind, const float* target, float scale, float* color, float* trans,
                         int32_t* last, float* image_grad, float* loss, real* accum, real* grid_grad,
                         cudaStream_t st);
#endif

__device__ __forceinline__ uint32_t float_order_key(float d) {
    uint32_t b = __float_as_uint(d == 0.0f ? 0.0f : d);  // -0 sorts as +0 (double compare)
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

}  // namespace gb
