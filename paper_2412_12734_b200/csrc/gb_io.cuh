// gb_io.cuh -- GBIL record <-> SplatSet SoA mapping and the pack/unpack
// kernels (gb_io.cu), used by gb_splats_save / gb_splats_load (gb_capi.cu).
#pragma once

#include "gb_internal.cuh"

namespace gb {

// field f of a record <-> (SoA array, floats per primitive, component); the
// grid (F floats) follows the scalar fields.
struct RecordMap {
    int fields;
    int F;
    const float* src[10];
    int stride[10];
    int offset[10];
};

inline int record_fields_of(const RecordMap& m) { return m.fields + m.F; }

RecordMap record_map(int version, const gb_splats* s);
cudaError_t launch_pack(int64_t K, const RecordMap& m, const float* grid, float* rec, int sm_count, cudaStream_t st);
cudaError_t launch_unpack(int64_t K, const RecordMap& m, float* grid, const float* rec, int sm_count,
                          cudaStream_t st);

}  // namespace gb
