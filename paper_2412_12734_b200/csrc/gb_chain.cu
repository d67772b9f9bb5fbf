// gb_chain.cu -- K5: the per-primitive gradient chain from K4's screen-space sums to the raw parameters.
//
// Gradients are compared with the oracle under a tolerance (no binning decision depends on them), so this
// translation unit, unlike K1's, keeps FMA contraction and replaces fp64 divisions by reciprocals (one per
// quaternion norm, camera focal length and plane depth): fewer DDIV sequences in an issue-bound kernel.
#include "gb_geom.cuh"

namespace gb {

// K5: chain the K4 screen-space sums to the raw parameters and ADD into the
// gradient buffer with reds (red.global.add): several views' K5s run on
// different streams into one buffer (the trainer's view lanes), so a plain
// read-modify-write could lose updates.  Ortho: raster.hpp:350-360 with the per-eval products
// (u_hat*u, ...) summed by K4.  Pinhole: dL/dM from (S_A, S_B, S_D) then the
// camera/quaternion chain (oracle pinhole_chain()).
// 8 CTAs of 128 threads per SM (64 registers, with spills): fp64 latency hides better with more warps
// (+0.9 % end to end over 96-104 registers at 4-5 CTAs)
#ifndef GB_K5_MINB
#define GB_K5_MINB 8
#endif
__global__ void __launch_bounds__(128, GB_K5_MINB) k_chain(const ProjParams p, const uint32_t* __restrict__ counts,
                                               const real* __restrict__ accum, gb_grads g_out) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= p.K) return;
    if (counts[k] == 0) return;
    const real4* a4 = reinterpret_cast<const real4*>(accum + k * kAccumStride);
    const real4 A = a4[0], B = a4[1], C = a4[2];
    Geom g;
    build_geom<true>(p, k, g);
    if (p.mode == GB_MODE_ORTHO) {
        const double su = A.x, sv = A.y, suv = A.z, svu = A.w, suu = B.x, svv = B.y, sop = B.z;
        const double inv_su = 1.0 / g.s_u, inv_sv = 1.0 / g.s_v;
        atomicAdd(reinterpret_cast<float2*>(g_out.position) + k,
                  make_float2((float)(su * (-g.cos_t * inv_su) + sv * (g.sin_t * inv_sv)),
                              (float)(su * (-g.sin_t * inv_su) + sv * (-g.cos_t * inv_sv))));
        atomicAdd(g_out.theta + k, (float)(suv * (g.s_v * inv_su) - svu * (g.s_u * inv_sv)));
        atomicAdd(reinterpret_cast<float2*>(g_out.log_scale) + k,
                  make_float2(g.su_clamped ? 0.0f : (float)(-suu), g.sv_clamped ? 0.0f : (float)(-svv)));
        atomicAdd(g_out.opacity_logit + k, (float)(sop * (g.alpha_k * (1.0 - g.alpha_k))));
        return;
    }
    if (!g.valid) return;
    int cxi, cyi;
    real hx, hy;
    double dxe, dye;
    pinhole_centre<true>(p, g, cxi, cyi, hx, hy, dxe, dye);
    // K4 sums over pixels of gc' = dL/dc' (c' = c / E_z):  S_E = sum gc', S_X = sum dx gc', S_Y = sum dy gc'
    PinholeCoeffs pc;
    pinhole_coeffs(g, dxe, dye, pc);
    if (!(pc.E[2] != 0.0)) return;
    const double iez = 1.0 / pc.E[2];
    const double SE[3] = {A.x, A.y, A.z}, SX[3] = {A.w, B.x, B.y}, SY[3] = {B.z, B.w, C.x};
    const double sop = C.y;
    double gC0[3], gCx[3], gCy[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        const double gE = SE[j] * iez;  // dL/dc = dL/dc' / E_z (u, v are scale invariant)
        gC0[j] = gE;
        gCx[j] = SX[j] * iez * p.inv_fx + dxe * gE;
        gCy[j] = SY[j] * iez * p.inv_fy + dye * gE;
    }
    // C0 = M0 x M1, Cx = M1 x M2, Cy = M2 x M0  ->  dL/dM (rows)
    const double* M0 = g.M;
    const double* M1 = g.M + 3;
    const double* M2 = g.M + 6;
    double t0[3], t1[3], dM[9];
    cross3(M1, gC0, t0);
    cross3(gCy, M2, t1);
    for (int j = 0; j < 3; ++j) dM[j] = t0[j] + t1[j];
    cross3(gC0, M0, t0);
    cross3(M2, gCx, t1);
    for (int j = 0; j < 3; ++j) dM[3 + j] = t0[j] + t1[j];
    cross3(gCx, M1, t0);
    cross3(M0, gCy, t1);
    for (int j = 0; j < 3; ++j) dM[6 + j] = t0[j] + t1[j];
    double g_col0[3], g_col1[3], g_pc[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        g_col0[r] = dM[3 * r + 0];
        g_col1[r] = dM[3 * r + 1];
        g_pc[r] = dM[3 * r + 2];
    }
    double g_su = 0.0, g_sv = 0.0, g_tu[3], g_tv[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        g_su += g_col0[r] * g.tuc[r];
        g_sv += g_col1[r] * g.tvc[r];
    }
    const double* R = p.R;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        atomicAdd(g_out.position + 3 * k + j, (float)(R[0 + j] * g_pc[0] + R[3 + j] * g_pc[1] + R[6 + j] * g_pc[2]));
        g_tu[j] = g.s_u * (R[0 + j] * g_col0[0] + R[3 + j] * g_col0[1] + R[6 + j] * g_col0[2]);
        g_tv[j] = g.s_v * (R[0 + j] * g_col1[0] + R[3 + j] * g_col1[1] + R[6 + j] * g_col1[2]);
    }
    atomicAdd(reinterpret_cast<float2*>(g_out.log_scale) + k,
              make_float2(g.su_clamped ? 0.0f : (float)(g_su * g.s_u), g.sv_clamped ? 0.0f : (float)(g_sv * g.s_v)));
    const double w = g.qn[0], x = g.qn[1], y = g.qn[2], z = g.qn[3];
    double gq[4];
    gq[0] = g_tu[1] * 2 * z - g_tu[2] * 2 * y - g_tv[0] * 2 * z + g_tv[2] * 2 * x;
    gq[1] = g_tu[1] * 2 * y + g_tu[2] * 2 * z + g_tv[0] * 2 * y - g_tv[1] * 4 * x + g_tv[2] * 2 * w;
    gq[2] = -g_tu[0] * 4 * y + g_tu[1] * 2 * x - g_tu[2] * 2 * w + g_tv[0] * 2 * x + g_tv[2] * 2 * z;
    gq[3] = -g_tu[0] * 4 * z + g_tu[1] * 2 * w + g_tu[2] * 2 * x - g_tv[0] * 2 * w - g_tv[1] * 4 * z + g_tv[2] * 2 * y;
    const double dot = w * gq[0] + x * gq[1] + y * gq[2] + z * gq[3];
    const double iqn = 1.0 / g.qnorm;
    atomicAdd(reinterpret_cast<float4*>(g_out.quat) + k,
              make_float4((float)((gq[0] - g.qn[0] * dot) * iqn), (float)((gq[1] - g.qn[1] * dot) * iqn),
                          (float)((gq[2] - g.qn[2] * dot) * iqn), (float)((gq[3] - g.qn[3] * dot) * iqn)));
    atomicAdd(g_out.opacity_logit + k, (float)(sop * (g.alpha_k * (1.0 - g.alpha_k))));
}

cudaError_t launch_chain(const ProjParams& p, const uint32_t* counts, const real* accum, const gb_grads& g,
                         cudaStream_t st) {
    if (p.K == 0) return cudaSuccess;
    const int threads = 128;  // 96 fp64-heavy registers per thread: finer blocks fill the SMs better (+1 %)
    const unsigned blocks = (unsigned)((p.K + threads - 1) / threads);
    k_chain<<<blocks, threads, 0, st>>>(p, counts, accum, g);
    return cudaGetLastError();
}

}  // namespace gb
