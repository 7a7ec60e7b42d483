// project_tc.cu -- tcgen05 (5th-gen tensor core) TF32 grouped projection.
#include "project.cuh"

namespace hf {

hifuse_status project_tc_launch(const LayerMeta& m, const ProjMeta& pm, int K, int D,
                                const hifuse_csr* csr, const float* X, const int* gather_ids,
                                const float* W_rel, const float* W_root, float* Y, float* R0,
                                cudaStream_t s) {
  (void)m; (void)pm; (void)K; (void)D; (void)csr; (void)X; (void)gather_ids; (void)W_rel;
  (void)W_root; (void)Y; (void)R0; (void)s;
  return HIFUSE_ERR_UNSUPPORTED;
}

}  // namespace hf
