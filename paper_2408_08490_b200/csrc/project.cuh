// project.cuh -- shared declarations of the projection kernels.
#pragma once
#include "common.cuh"

#define HIFUSE_MAX_HEADS 16

namespace hf {

static constexpr int kBM = 64;     // SIMT forward / dgrad tile rows
static constexpr int kCH = 256;    // wgrad chunk rows

struct ProjMeta {
  int R, T, rows, has_root;
  int rel_src[HF_MAX_R];
  int rel_dst[HF_MAX_R];
  int rel_row_off[HF_MAX_R + 1];
  int n_dst[HF_MAX_T];
  int type_src_off[HF_MAX_T + 1];
  int type_dst_off[HF_MAX_T + 1];
};

struct DgradMeta {
  int T, has_root, bm;
  int tile_off[HF_MAX_T + 1];      // kBM-row tiles of each type's source rows
  int n_src[HF_MAX_T];
  int n_dst[HF_MAX_T];
  int type_src_off[HF_MAX_T + 1];
  int type_dst_off[HF_MAX_T + 1];
  int slot_off[HF_MAX_R + 1];
  int rel_row_off[HF_MAX_R + 1];
  int out_off[HF_MAX_T + 1];       // relations out of type s: out_rel[out_off[s]..]
  int out_rel[HF_MAX_R];
  int in_off[HF_MAX_T + 1];        // relations into type t: in_rel[in_off[t]..]
  int in_rel[HF_MAX_R];
};

void make_proj_meta(const LayerMeta& m, bool has_root, ProjMeta* pm);
void make_dgrad_meta(const LayerMeta& m, bool has_root, DgradMeta* dm, int bm = kBM);
long long proj_max_tiles(const LayerMeta& m, int step);

// tcgen05 TF32 forward projection (project_tc.cu).
// tcgen05 TF32 forward projection (persistent, warp-specialised; project_tc.cu)
// Xm != NULL: aggregate-first input layer -- message groups read the
// aggregated rows rel_off[r] + j of Xm (rel_off = rel_row_off) and write Z.
hifuse_status project_tcp_launch(const LayerMeta& m, const ProjMeta& pm, int K, int D,
                                 const int* rel_off, const int* y_src, const float* X,
                                 const float* Xm, const int* gather_ids, const float* W_rel,
                                 const float* W_root, float* Y, float* R0, const float* att,
                                 float* s_src, int H, cudaStream_t s,
                                 uint16_t* Wt_bf16 = nullptr,    // non-NULL: BF16 operands
                                 uint16_t* Yb = nullptr);        // non-NULL: Y stored bf16
// tcgen05 TF32 fused fusion GEMM of the aggregate-first input layer (NEXT(3)):
// H_t = act([X_t | Xagg_r...] [W_root,t; W_r...] + b_t), one launch.
hifuse_status fuse_gemm_launch(const LayerMeta& m, bool has_root, int K, int D, bool relu,
                               const int* gid, const float* X, const float* Xm,
                               const float* W_rel, const float* W_root, const float* bias,
                               float* H, cudaStream_t s);
// tcgen05 TF32 dgrad: dX[type s rows] = sum_terms A_term W_term^T (A = dYt rows
// through slot_y, or G for the root term).  dm built with bm = 128.
hifuse_status dgrad_tc_launch(const DgradMeta& dm, int K, int D, const int* slot_y,
                              const float* dY, const float* G, const float* W_rel,
                              const float* W_root, float* dX, cudaStream_t s, long long dy_rows,
                              int R);
// tcgen05 TF32 wgrad partials: P[c] = sum_{rows of chunk c} X_row^T dYt_row
// (chunks of CH rows per group from chunk_off; wgrad_chunk_rows() picks CH so
// that small layers still spread over every SM).
static constexpr int kCHT = 1024;
inline int wgrad_chunk_rows(const LayerMeta& m) {
  long long rows = (long long)(m.N < m.S ? m.N : m.S) + m.dst_rows;
  long long ch = rows / (2 * sm_count());
  ch = (ch + 31) / 32 * 32;
  return (int)(ch < 128 ? 128 : (ch > kCHT ? kCHT : ch));
}
hifuse_status wgrad_tc_launch(const LayerMeta& m, const ProjMeta& pm, int K, int D, int CH,
                              const int* chunk_off, const int* rel_y_off, const int* y_src,
                              const int* gather_ids, const float* X, const float* dY,
                              const float* G, float* partial, unsigned grid, cudaStream_t s,
                              const float* Xm = nullptr);
}  // namespace hf
