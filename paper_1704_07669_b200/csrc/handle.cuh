// handle.cuh — the state behind an spca_handle_t (one GPU, one consumer).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "../../include/spca.h"

namespace spca {
struct Timer {
  cudaEvent_t start = nullptr, stop = nullptr;
};
}  // namespace spca

struct spca_sketch {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaStream_t copy_stream = nullptr;
  int dtype = SPCA_F32;
  int precision = SPCA_PREC_SIMT;
  size_t ds = 4;
  int64_t n = 0, l = 0, lpad = 0;
  int bl = 64;
  bool compensated = false;

  void *omega_dev = nullptr;     // n x lpad compute precision
  double *omega64_dev = nullptr; // n x l fp64, exactly the values used
  void *tc_omega = nullptr;      // Omega^T hi | lo (2 x lpad x n fp32, sketch_tc.cuh)
  CUtensorMap tm_whi, tm_wlo;    // TMA maps over Omega^T hi / lo
  CUtensorMap tm_gT;             // TMA map over the G^T hi / lo slots (sketch_fused.cuh)

  void *g_dev = nullptr;         // cap x lpad compute precision
  int64_t g_cap = 0;
  double *g64_dev = nullptr;     // rows x l after finish
  int64_t g64_cap = 0;
  double *hcs_dev = nullptr;     // n*l H then n colsum
  double *carry_dev = nullptr;   // Kahan carry (n)
  void *hpart = nullptr;         // [hsplit][n][lpad]
  int hsplit = 1;
  double *cspart = nullptr;      // [hsplit][n]
  void *gpart = nullptr;         // P1 split-K partials
  int64_t gpart_elems = 0;
  void *tc_ws = nullptr;         // tensor-core G^T slots [kSlots][2][lpad][R0]
  size_t tc_ws_bytes = 0;
  int tc_gt_kparts = 2;          // G^T parts per slot (hi / lo, or 1 raw)
  int *tc_ctr = nullptr;         // per-launch ordering counters of the pass kernel
  int tc_lp = 64;                // l_pad of one pass-kernel launch (64 or 128)
  int tc_groups = 1;             // column groups of 128 (l > 128): one launch each
  int *order_dev = nullptr;      // unit order table of the last launch shape (tc_unit_order)
  int64_t order_cap = 0;
  int order_C = -1, order_TS = -1, order_TlS = -1, order_XR = -1;
  double order_lag = -1.0;
  int64_t tc_ctr_chunks = 0;     // chunks one launch may cover
  // row normalisation (spca_sketch_set_normalize)
  bool normalize = false;
  void *norm_ws = nullptr;       // SIMT path: normalized copy of one chunk
  double *rstat_part = nullptr;  // TC: [kSlots][2T][S][128][2] per-segment sums of d, d^2
  float *row_a0 = nullptr;       // TC: [kSlots][R0] row shifts of the chunks in flight
  float *row_inv = nullptr;      // TC: [kSlots][R0] 1 / row norms
  double *row_coef = nullptr;    // TC: [rows] (mean - a0) / norm of every row pushed
  int64_t row_coef_cap = 0;
  float *wsum = nullptr;         // TC: [lpad] column sums of Omega (as used)
  // co-sketch operand (spca_sketch_set_left): H += A_i^T L_i instead of A_i^T G_i
  void *left_dev = nullptr;      // rows x lpad compute precision (zero padded)
  double *left64_dev = nullptr;  // rows x l fp64, exactly the values used
  int64_t left_rows = 0;         // 0 = no left operand (the plain sketch)
  // column shift (spca_sketch_set_shift): the pass sketches A - 1 c^T, c = its first row
  bool shift_on = false;
  bool shift_set = false;        // c captured for this pass
  float *cshift = nullptr;       // round_up(n, 128) fp32, zero padded
  int num_sms = 148;
  int max_pairs = 74;             // co-resident CTA pairs of the pass kernel
  unsigned long long *bad_dev = nullptr;
  unsigned long long bad_seen = 0;  // first non-finite row, read back at finish

  int64_t chunk_rows = 0;        // canonical chunk (R0)
  int64_t ldp = 0;               // row stride of the library's own row buffers (tail, staging):
                                 // n, or n rounded up to 4 on the tensor-core path (16-byte TMA rows)
  void *tail = nullptr;          // R0 x n staging for the partial chunk
  int64_t tail_rows = 0;
  int64_t rows_seen = 0;         // accepted
  int64_t rows_done = 0;         // processed
  int chunks_since_flush = 0;
  int flush_every = 64;
  int tc_debug = 0;              // SPCA_TC_DEBUG bitmask (profiling experiments only)
  int tc_coop = 1;               // cooperative pass launches (SPCA_TC_COOP=0: plain launch, A/B only)
  unsigned long long *trace = nullptr;  // SPCA_TC_TRACE per-CTA timeline
  bool finished = false;
  bool final_pushed = false;     // spca_sketch_push_final was called (no more rows)

  // host staging (pinned double buffer)
  void *pinned[2] = {nullptr, nullptr};
  void *dstage[2] = {nullptr, nullptr};
  int64_t stage_rows = 0;
  cudaEvent_t copy_done[2] = {nullptr, nullptr};
  cudaEvent_t comp_done[2] = {nullptr, nullptr};
  cudaEvent_t src_ready = nullptr;  // device rows re-strided on the copy stream: producer done
  bool stage_used[2] = {false, false};
  int stage_idx = 0;

  int64_t launches = 0;
  bool timing = false;
  std::vector<spca::Timer> timers;     // unused (kept for layout stability)
  cudaEvent_t t_start = nullptr, t_stop = nullptr;  // kernel-group timing window
  bool t_open = false;
  int64_t t_chunks = 0;

  // TMA descriptors cached per pushed source buffer (encoding is a driver
  // call of several microseconds; a full-matrix push encodes once)
  const void *src_ptr = nullptr;
  int64_t src_rows = 0, src_lda = 0;
  CUtensorMap src_tg, src_th;
  CUtensorMap src_tg3, src_th2;  // paired A slots: 3-D box of two K blocks / 64-row box
  double kernel_ms = 0.0;
  int64_t timed_chunks = 0;

  int last_code = SPCA_OK;
  int64_t last_bad_row = -1;
  char last_msg[512] = {0};
};
