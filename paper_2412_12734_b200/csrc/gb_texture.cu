// gb_texture.cu -- the mip diagnostic of the texture grids (texture.hpp:128-188):
// downsample_grid / downsample_set on the device.
//
// The reference halves a grid level by level, each output texel being
// (c00 + c10 + c01 + c11) * 0.25 of its 2x2 parent block, and, once an odd
// size is reached with enough levels left, collapses the grid to the 1x1 mean
// (texture.hpp:136-147).  k_downsample gives every (primitive, output texel,
// channel) one thread that evaluates exactly that tree -- same operand order,
// same 0.25 scaling per level -- in registers, reading the source texels it
// covers once (the grid is HBM-resident; each source texel is read by one
// thread per output texel that covers it).
#include "gb_internal.cuh"

namespace gb {

// value of texel (iu, iv) channel ch after `h` halvings of an n x n grid
__device__ float halved(const float* __restrict__ g, int n, int h, int iu, int iv, int ch) {
    if (h == 0) return g[((size_t)iu * n + iv) * 3 + ch];
    // texture.hpp:152-156, operand order (2iu,2iv), (2iu+1,2iv), (2iu,2iv+1), (2iu+1,2iv+1)
    const float a = halved(g, n, h - 1, 2 * iu, 2 * iv, ch);
    const float b = halved(g, n, h - 1, 2 * iu + 1, 2 * iv, ch);
    const float c = halved(g, n, h - 1, 2 * iu, 2 * iv + 1, ch);
    const float d = halved(g, n, h - 1, 2 * iu + 1, 2 * iv + 1, ch);
    return (((a + b) + c) + d) * 0.25f;
}

__global__ void __launch_bounds__(256) k_downsample(int64_t K, int n, int halvings, int collapse,
                                                    const float* __restrict__ src, float* __restrict__ dst) {
    const int cur = n >> halvings;               // size after the halvings
    const int out_n = collapse ? 1 : cur;
    const int Fo = 3 * out_n * out_n, Fi = 3 * n * n;
    const int64_t total = K * Fo;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
        const int64_t k = i / Fo;
        const int r = (int)(i - k * Fo);
        const int t = r / 3, ch = r - 3 * t;
        const float* g = src + k * Fi;
        float v;
        if (!collapse) {
            v = halved(g, n, halvings, t / out_n, t % out_n, ch);
        } else {  // texture.hpp:140-145: mean over the cur x cur grid, texel order
            float s = 0.0f;
            for (int j = 0; j < cur * cur; ++j) s += halved(g, n, halvings, j / cur, j % cur, ch);
            v = s / (float)(cur * cur);
        }
        dst[i] = v;
    }
}

// texture.hpp:132-147 shape rules: returns false (too few levels for an odd size) or the plan.
bool downsample_plan(int n, int levels, int& halvings, int& collapse, int& n_out) {
    int cur = n;
    halvings = 0;
    collapse = 0;
    for (int level = 0; level < levels && cur > 1; ++level) {
        if (cur % 2 != 0) {
            if ((1 << (levels - level)) < cur) return false;
            collapse = 1;
            break;
        }
        cur /= 2;
        ++halvings;
    }
    n_out = collapse ? 1 : cur;
    return true;
}

cudaError_t launch_downsample(int64_t K, int n, int halvings, int collapse, const float* src, float* dst,
                              int sm_count, cudaStream_t st) {
    const int out_n = collapse ? 1 : (n >> halvings);
    const int64_t total = K * 3 * out_n * out_n;
    if (total == 0) return cudaSuccess;
    int64_t blocks = (total + 255) / 256;
    if (blocks > (int64_t)sm_count * 8) blocks = (int64_t)sm_count * 8;
    k_downsample<<<(unsigned)blocks, 256, 0, st>>>(K, n, halvings, collapse, src, dst);
    return cudaGetLastError();
}

}  // namespace gb
