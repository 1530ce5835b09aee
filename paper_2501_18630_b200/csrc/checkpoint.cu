// Checkpoint records <-> device parameter buffer (sceneio.py:467-564,
// docs/formats.md "Checkpoints").
//
// The reference's checkpoint is a binary little-endian PLY whose vertex element is an
// array of N records of P doubles (x y z opacity_raw log_scale_* rot_* shape base_* and
// per-lobe axis / colour).  The host reads the file into (pinned) memory, copies the
// record block to the device once, and bsr_checkpoint_unpack scatters it into the flat
// group-major fp32 buffer (primitive.group_layout); bsr_checkpoint_pack is the inverse
// (fp32 -> fp64 is exact, so a saved state reloads bit-identically).  One thread per
// record scalar: record reads are coalesced, each property's writes stride through its
// group.
#include "common.cuh"

namespace bsr {

constexpr int kMaxProps = 64;

struct CkptMap {
    int64_t start[kMaxProps];  // flat element offset of primitive 0's value
    int32_t stride[kMaxProps];  // floats per primitive in its group
};

__global__ void ckpt_unpack_kernel(const double *__restrict__ rec, int64_t n, int p, CkptMap m, float *flat) {
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= n * p) return;
    const int64_t i = idx / p;
    const int q = (int)(idx - i * p);
    flat[m.start[q] + (int64_t)m.stride[q] * i] = (float)rec[idx];
}

__global__ void ckpt_pack_kernel(const float *__restrict__ flat, int64_t n, int p, CkptMap m, double *rec) {
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= n * p) return;
    const int64_t i = idx / p;
    const int q = (int)(idx - i * p);
    rec[idx] = (double)flat[m.start[q] + (int64_t)m.stride[q] * i];
}

static bool make_map(int32_t n_props, const int64_t *start, const int32_t *stride, CkptMap &m) {
    if (n_props < 1 || n_props > kMaxProps || !start || !stride) return false;
    for (int q = 0; q < n_props; ++q) {
        if (start[q] < 0 || stride[q] < 1) return false;
        m.start[q] = start[q];
        m.stride[q] = stride[q];
    }
    return true;
}

}  // namespace bsr

using namespace bsr;

extern "C" int bsr_checkpoint_unpack(const double *records, int64_t n, int32_t n_props, const int64_t *prop_start,
                                     const int32_t *prop_stride, float *flat, void *stream) {
    CkptMap m;
    if (n < 0 || !make_map(n_props, prop_start, prop_stride, m) || (n > 0 && (!records || !flat)))
        return BSR_ERR_BAD_ARG;
    if (n == 0) return BSR_OK;
    const int64_t total = n * n_props;
    ckpt_unpack_kernel<<<(unsigned)div_up(total, BSR_BLOCK), BSR_BLOCK, 0, (cudaStream_t)stream>>>(records, n, n_props,
                                                                                                  m, flat);
    BSR_LAUNCH_CHECK();
    return BSR_OK;
}

extern "C" int bsr_checkpoint_pack(const float *flat, int64_t n, int32_t n_props, const int64_t *prop_start,
                                   const int32_t *prop_stride, double *records, void *stream) {
    CkptMap m;
    if (n < 0 || !make_map(n_props, prop_start, prop_stride, m) || (n > 0 && (!records || !flat)))
        return BSR_ERR_BAD_ARG;
    if (n == 0) return BSR_OK;
    const int64_t total = n * n_props;
    ckpt_pack_kernel<<<(unsigned)div_up(total, BSR_BLOCK), BSR_BLOCK, 0, (cudaStream_t)stream>>>(flat, n, n_props, m,
                                                                                                records);
    BSR_LAUNCH_CHECK();
    return BSR_OK;
}
