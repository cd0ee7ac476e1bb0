// tc_host.cuh — host side of the tensor-core path: capability checks, TMA
// descriptor encoding (driver entry point, no libcuda link), workspace and
// per-chunk launches. Included by spca_capi.cu after the error helpers.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

namespace {

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                  const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                  const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// Resolved once per process (thread-safe function-local static): two threads
// creating handles at once must both see the entry point.
EncodeTiledFn tma_encoder() {
  static const EncodeTiledFn fn = []() -> EncodeTiledFn {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return (EncodeTiledFn)p;
    return nullptr;
  }();
  return fn;
}

bool tc_available(int device) {
  int major = 0, minor = 0;
  if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device) != cudaSuccess) return false;
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device);
  return major == 10 && minor == 0 && tma_encoder() != nullptr;
}

// l <= 128: wider sketches (config 5's l = 250) use the SIMT kernels until the
// promoted accumulators of an N = 256 tile fit the register budget.
// l > 128 runs as column groups of 128 (one launch per group over the same
// rows): H[:, J] = A^T (A Omega[:, J]) needs only G[:, J].
constexpr int kTcMaxL = 4096;  // column groups of 128: one launch (one read of A) per group
// any n >= 32: rows whose stride is not a multiple of 16 bytes are re-strided
// through a padded buffer before the pass (push_device_rows)
bool tc_supported_shape(int64_t n, int64_t l) { return n >= 32 && l >= 1 && l <= kTcMaxL; }

// l_pad of the whole sketch (accumulator layouts) and of one launch
int tc_lpad(int64_t l) { return l <= 64 ? 64 : (int)(128 * ceil_div(l, 128)); }
int tc_launch_lpad(int64_t l) { return l <= 64 ? 64 : 128; }

// Canonical chunk of the single-read pass: A_c is read from HBM by the G
// units and again from L2 by the H units one stage later, so about two
// chunks must stay resident in the 126 MB L2: R0 * n * 4 B ~ 40 MB by default
// (SPCA_TC_CHUNK_MB). Whole 256-row tile pairs, at most 8192 rows.
int64_t tc_chunk_rows(int64_t n, int64_t l) {
  // l_pad 128 sketches carry twice the MMA work per K block, so the chunk's
  // DRAM re-read weighs less than per-chunk fixed costs: 80 MB measured best
  // at config 3 (10.5 vs 11.2 ms at 40 MB; 120-240 MB slower again), 40 MB at
  // config 2 (round-2 sweeps, profiles/r5_chunk_unit_sweep.txt)
  int64_t mb = l > 64 ? 80 : 40;
  if (const char *e = getenv("SPCA_TC_CHUNK_MB")) mb = std::max<int64_t>(1, atoll(e));  // tuning knob
  int64_t r = (int64_t)(mb << 20) / (4 * n);
  // wide rows: at least 1024 rows (H units of a full 32 K blocks; config 5,
  // n = 200 000: 60 ms per pass vs 127 ms at 256 rows) while a chunk stays <= 1 GB
  int64_t fl = 1024;
  if (const char *e = getenv("SPCA_TC_MIN_ROWS")) fl = std::max<int64_t>(256, atoll(e));  // tuning knob
  const int64_t floor_rows = std::max<int64_t>(256, std::min<int64_t>(fl, (int64_t)(1ll << 30) / (4 * n)));
  r = std::max<int64_t>(floor_rows, std::min<int64_t>(8192, r));
  return (r / 256) * 256;
}

// K blocks (32 deep) per work unit: the G units split n, the H units split a
// chunk's rows, both into pieces of about this size.
// (40 for l_pad 64 - config 2: eight K segments of 40 / 34 blocks instead of ten
// of 32 / 26 - measured 0.8% faster in three alternating runs, 1.681 -> 1.668 ms,
// but with 7.58 instead of 6.98 GB of DRAM reads per pass: not taken,
// profiles/r6_unit40.txt)
int tc_unit_kb(int lp) {
  (void)lp;
  int u = 32;
  if (const char *e = getenv("SPCA_TC_UNIT_KB")) u = std::max(1, atoi(e));  // tuning knob
  return u;
}

// l > 128: the column groups of 128 run in ONE launch (units of every group
// of a tile / column stripe dealt side by side, so each A tile is read from
// DRAM once for all groups) unless fused row normalisation is on (its row
// statistics are written by group 0's reductions) or SPCA_TC_SEQ_GROUPS is set
// (one launch per group, each reading A).
bool tc_merged_groups(const spca_sketch *h) {
  static const bool seq = getenv("SPCA_TC_SEQ_GROUPS") != nullptr;
  return h->tc_groups > 1 && !h->normalize && !seq;
}
int tc_max_quads();
// Two column groups of 128 (l_pad 256, config 5) as one launch of clusters of
// four, a CTA pair per group, each A tile fetched once and multicast to both
// pairs (tc_pass_kernel<.., DUAL>). Opt-in (SPCA_TC_DUAL=1): bitwise equal to
// the default, but measured slower — config 5 63.4 vs 55.7 ms, 20 000 rows
// 24.1 vs 20.6 ms: only 33 clusters of four fit (132 SMs instead of 148) and
// the two pairs run in lockstep (pair 0 refills a slot only after both pairs
// consumed it), which costs more than the halved A traffic saves
// (profiles/r5_dual_groups.txt). Fused normalisation keeps one launch per group.
bool tc_dual_groups(const spca_sketch *h) {
  static const bool on = getenv("SPCA_TC_DUAL") != nullptr && atoi(getenv("SPCA_TC_DUAL")) != 0;
  return on && h->tc_groups == 2 && h->tc_lp == 128 && tc_merged_groups(h) && tc_max_quads() >= 1;
}

FusedSched tc_base_sched(const spca_sketch *h) {
  FusedSched s{};
  s.Gr = 1;
  const int U = tc_unit_kb(h->tc_lp);
  s.R0 = (int)h->chunk_rows;
  s.nt = s.R0 / 128;
  s.T = s.nt / 2;
  s.nkb = (int)ceil_div(h->n, 32);
  // A G unit's epilogue waits for every K segment of its tile, and the
  // segments are dealt to consecutive pairs: S must not exceed the pairs of
  // the grid (else a pair would wait on its own later unit). Wide n gets
  // longer segments instead (S <= max_pairs / 2).
  // (merged column groups deal a tile's segments of every group side by side:
  // the span S * groups keeps the same bound)
  // (sized for every group whether or not this launch merges them, so the
  // buffers allocated at setup fit either way)
  const int gcap = std::max(1, h->tc_groups);
  const int max_seg = std::max(1, h->max_pairs / (2 * gcap));
  s.kp = h->tc_lp == 64 ? TcCfg<64>::KP : TcCfg<128>::KP;  // K blocks per MMA-warp iteration
  s.S = (int)std::min<int64_t>(ceil_div(s.nkb, U), max_seg);
  s.kseg = (int)(ceil_div(ceil_div(s.nkb, s.S), s.kp) * s.kp);
  s.S = (int)ceil_div(s.nkb, s.kseg);
  s.nx = (int)ceil_div(h->n, 128);
  s.X = (int)ceil_div(s.nx, 2);
  const int rkb = s.R0 / 32;
  // H units: row segments of up to 48 K blocks (config 3, 80-block chunks:
  // two segments of 40 ran 17% faster than three of 27)
  int hu = std::max(U, 48);
  if (const char *e = getenv("SPCA_TC_HSEG")) hu = std::max(1, atoi(e));  // tuning knob: K blocks per H unit
  s.RS = (int)ceil_div(rkb, hu);
  s.hseg = (int)(ceil_div(ceil_div(rkb, s.RS), s.kp) * s.kp);
  s.RS = (int)ceil_div(rkb, s.hseg);
  s.D = 2;  // measured: one extra stage of slack removes the H units' waits for G^T
  if (const char *e = getenv("SPCA_TC_LAG")) s.D = std::max(1, std::min(kMaxLag, atoi(e)));  // tuning knob
  return s;
}

int encode_2d(spca_sketch *h, CUtensorMap *map, const void *ptr, uint64_t inner, uint64_t outer,
              uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer, bool swizzle = true) {
  EncodeTiledFn enc = tma_encoder();
  if (!enc) return set_err(h, SPCA_ERR_CUDA, -1, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void *>(ptr), dims, strides, box,
                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_err(h, SPCA_ERR_CUDA, -1, "tensor map encode failed (%d): dims %llu x %llu stride %llu",
                   (int)r, (unsigned long long)inner, (unsigned long long)outer,
                   (unsigned long long)row_bytes);
  return SPCA_OK;
}

// A as K-block tiles for the G units' paired loads: dims {32, rows, n/32},
// box {32, 128, 2} = two consecutive swizzled 128 x 32 tiles (n % 32 == 0)
int encode_a3d(spca_sketch *h, CUtensorMap *map, const void *ptr, uint64_t rows, uint64_t row_bytes) {
  EncodeTiledFn enc = tma_encoder();
  if (!enc) return set_err(h, SPCA_ERR_CUDA, -1, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {32, rows, (cuuint64_t)(h->n / 32)};
  cuuint64_t strides[2] = {row_bytes, 128};
  cuuint32_t box[3] = {32, 128, 2};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void *>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_err(h, SPCA_ERR_CUDA, -1, "3-d tensor map encode failed (%d)", (int)r);
  return SPCA_OK;
}

// every A map of one source buffer: G tiles (2-D, and 3-D pairs when n % 32 == 0),
// H tiles of 32 and 64 rows
int encode_a_maps(spca_sketch *h, const void *a, uint64_t rows, uint64_t row_bytes, CUtensorMap *tg,
                  CUtensorMap *th, CUtensorMap *tg3, CUtensorMap *th2) {
  int rc = encode_2d(h, tg, a, (uint64_t)h->n, rows, row_bytes, 32, 128);
  if (rc) return rc;
  rc = encode_2d(h, th, a, (uint64_t)h->n, rows, row_bytes, 128, 32, false);
  if (rc) return rc;
  rc = encode_2d(h, th2, a, (uint64_t)h->n, rows, row_bytes, 128, 64, false);
  if (rc) return rc;
  if (h->n % 32 == 0) return encode_a3d(h, tg3, a, rows, row_bytes);
  *tg3 = *tg;  // unused (args.g3d = 0)
  return SPCA_OK;
}

// The attribute takes effect on the current device only: set it on every
// handle's setup (cheap, once per handle), never cached process-wide.
template <int LPAD>
int tc_set_smem_attrs() {
  for (auto k : {tc_pass_kernel<LPAD, false>, tc_pass_kernel<LPAD, true>, tc_pass_kernel<LPAD, false, true>})
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TcCfg<LPAD>::SMEM) !=
        cudaSuccess)
      return 1;
  if (LPAD == 128)
    for (auto k : {tc_pass_kernel<128, false, false, true>, tc_pass_kernel<128, false, true, true>})
      if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TcCfg<128>::SMEM) !=
          cudaSuccess)
        return 1;
  return 0;
}

// Clusters of four (two CTA pairs, DUAL) that can be resident at once
int tc_max_quads() {
  static int cached[64];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && cached[dev] > 0) return cached[dev];
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(4, 1, 1);
  cfg.blockDim = dim3(TcCfg<128>::THREADS, 1, 1);
  cfg.dynamicSmemBytes = TcCfg<128>::SMEM;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 4;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int nc = 0;
  if (cudaOccupancyMaxActiveClusters(&nc, tc_pass_kernel<128, false, false, true>, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  if (dev >= 0 && dev < 64) cached[dev] = nc;
  return nc;
}

// CTA pairs that can be resident at once: the persistent pass needs every
// CTA of its grid co-resident (its inter-CTA waits assume it).
template <int LPAD>
int tc_max_pairs() {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2, 1, 1);
  cfg.blockDim = dim3(TcCfg<LPAD>::THREADS, 1, 1);
  cfg.dynamicSmemBytes = TcCfg<LPAD>::SMEM;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // one query per process and device (it costs about a millisecond)
  static int cached[64];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && cached[dev] > 0) return cached[dev];
  int nc = 0;
  if (cudaOccupancyMaxActiveClusters(&nc, tc_pass_kernel<LPAD, false>, &cfg) != cudaSuccess) return 0;
  if (dev >= 0 && dev < 64) cached[dev] = nc;
  return nc;
}

int tc_setup(spca_sketch *h) {
  const int lp_total = tc_lpad(h->l);
  const int lp = tc_launch_lpad(h->l);
  h->tc_lp = lp;
  h->tc_groups = lp_total / lp;
  if (lp_total != h->lpad) {
    // the SIMT layout padded l to 32/64; the tensor-core path needs 64/128
    h->lpad = lp_total;
    h->bl = 64;
    dfree(h, h->omega_dev);
    h->omega_dev = nullptr;
    dfree(h, h->hpart);
    h->hpart = nullptr;
    CK(h, dalloc(h, &h->omega_dev, (size_t)h->n * h->lpad * 4));
    CK(h, dalloc(h, &h->hpart, (size_t)h->n * h->lpad * 4));
    CK(h, cudaMemsetAsync(h->hpart, 0, (size_t)h->n * h->lpad * 4, h->stream));
  }
  int bad = lp == 64 ? tc_set_smem_attrs<64>() : tc_set_smem_attrs<128>();  // per-launch template
  if (bad) return set_err(h, SPCA_ERR_CUDA, -1, "cannot raise dynamic shared memory for the tc kernel");
  CK(h, cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, h->device));
  h->max_pairs = lp == 64 ? tc_max_pairs<64>() : tc_max_pairs<128>();
  if (h->max_pairs < 1) return set_err(h, SPCA_ERR_CUDA, -1, "no CTA pair of the pass kernel fits an SM pair");
  // Omega^T rows padded to a 16-byte multiple (TMA strides), zero padding
  const int64_t ldw = round_up(h->n, 4);
  CK(h, dalloc(h, &h->tc_omega, (size_t)2 * h->lpad * ldw * 4));
  CK(h, cudaMemsetAsync(h->tc_omega, 0, (size_t)2 * h->lpad * ldw * 4, h->stream));
  float *whi = (float *)h->tc_omega;
  float *wlo = whi + (size_t)h->lpad * h->n;
  const uint32_t hr = (uint32_t)(lp / 2);
  int rc;
#if SPCA_BRAW
  // raw Omega^T (lpad rows): each CTA loads its l_pad/2 rows of the group per K block
  tc_omega_prepare_raw<<<grid_for((int64_t)h->lpad * h->n), 256, 0, h->stream>>>(
      h->omega64_dev, (int)h->n, (int)h->l, (int)h->lpad, whi, (int)ldw);
  CK_LAUNCH(h);
  rc = encode_2d(h, &h->tm_whi, whi, (uint64_t)h->n, (uint64_t)h->lpad, (uint64_t)ldw * 4, 32, hr);
  if (rc) return rc;
  h->tm_wlo = h->tm_whi;
  const uint32_t gbox = hr;
  constexpr int kGtParts = 1;  // raw G^T
#elif SPCA_BCOMB
  // one matrix of 2 lpad rows: each CTA's half of a column group is hi rows
  // then lo rows, loaded as ONE box of lp rows per K block
  tc_omega_prepare_comb<<<grid_for((int64_t)h->lpad * h->n), 256, 0, h->stream>>>(
      h->omega64_dev, (int)h->n, (int)h->l, (int)h->lpad, lp, whi, (int)ldw);
  CK_LAUNCH(h);
  rc = encode_2d(h, &h->tm_whi, whi, (uint64_t)h->n, (uint64_t)2 * h->lpad, (uint64_t)ldw * 4, 32, lp);
  if (rc) return rc;
  h->tm_wlo = h->tm_whi;
  const uint32_t gbox = (uint32_t)lp;
  constexpr int kGtParts = 2;
#else
  tc_omega_prepare<<<grid_for((int64_t)h->lpad * h->n), 256, 0, h->stream>>>(
      h->omega64_dev, (int)h->n, (int)h->l, (int)h->lpad, whi, wlo);
  CK_LAUNCH(h);
  // B tiles are loaded as l_pad/2-row halves (one per CTA of a pair) of one
  // column group; Omega^T holds every group (rows g*lp ..)
  rc = encode_2d(h, &h->tm_whi, whi, (uint64_t)h->n, (uint64_t)h->lpad, (uint64_t)h->n * 4, 32, hr);
  if (rc) return rc;
  rc = encode_2d(h, &h->tm_wlo, wlo, (uint64_t)h->n, (uint64_t)h->lpad, (uint64_t)h->n * 4, 32, hr);
  if (rc) return rc;
  const uint32_t gbox = hr;
  constexpr int kGtParts = 2;
#endif
  const FusedSched s = tc_base_sched(h);
  // G^T (raw, or hi / lo) of kSlots chunks of one launch: [groups][kSlots][parts x lp rows][R0], one
  // TMA map (groups: the column groups a merged launch sketches together)
  const int ng = std::max(1, h->tc_groups);  // room for a merged launch of every group
  h->tc_gt_kparts = kGtParts;
  h->tc_ws_bytes = (size_t)ng * kSlots * kGtParts * lp * s.R0 * 4;
  CK(h, dalloc(h, &h->tc_ws, h->tc_ws_bytes));
  rc = encode_2d(h, &h->tm_gT, h->tc_ws, (uint64_t)s.R0, (uint64_t)ng * kSlots * kGtParts * lp,
                 (uint64_t)s.R0 * 4, 32, gbox);
  if (rc) return rc;
  h->gpart_elems = (int64_t)kSlots * 2 * s.T * s.S * 128 * lp;  // per group
  CK(h, dalloc(h, &h->gpart, (size_t)ng * h->gpart_elems * 4));
  // ordering counters of one launch (at most flush_every chunks), per group
  h->tc_ctr_chunks = h->flush_every;
  CK(h, dalloc(h, &h->tc_ctr, (size_t)ng * (h->tc_ctr_chunks * (4 * s.T + 2) + 2 * s.X) * 4));
  if (getenv("SPCA_TC_TRACE")) {
    CK(h, dalloc(h, &h->trace, (size_t)kTraceWords * 8));
    CK(h, cudaMemsetAsync(h->trace, 0, (size_t)kTraceWords * 8, h->stream));
  }
  return SPCA_OK;
}

// Per-device ordering of pass-kernel launches across handles (see the launch).
struct PassSerial {
  std::mutex mu;
  cudaEvent_t last = nullptr;  // recorded behind the device's latest pass kernel
};
PassSerial &pass_serial(int device) {
  static PassSerial table[64];
  return table[device & 63];
}

// Remember TMA descriptors over a pushed device buffer so its full chunks
// are addressed by row offset without re-encoding.
int tc_register_source(spca_sketch *h, const void *a, int64_t rows, int64_t lda) {
  if (rows < h->chunk_rows || (lda % 4) != 0 || (reinterpret_cast<uintptr_t>(a) % 16) != 0 ||
      rows > INT32_MAX) {
    h->src_ptr = nullptr;
    return SPCA_OK;
  }
  if (h->src_ptr == a && h->src_rows == rows && h->src_lda == lda) return SPCA_OK;
  int rc = encode_a_maps(h, a, (uint64_t)rows, (uint64_t)lda * 4, &h->src_tg, &h->src_th, &h->src_tg3,
                         &h->src_th2);
  if (rc) return rc;
  h->src_ptr = a;
  h->src_rows = rows;
  h->src_lda = lda;
  return SPCA_OK;
}

// Unit order of a launch, built on the host: G units of chunk c sit at
// virtual times c*P + r (P = units of a full stage), H units at
// c*P + TS + lag*P + r; units are dealt in that order (G first on ties).
// lag = 2 reproduces the closed-form stage layout with D = 2; a fractional
// lag (SPCA_TC_LAGF) moves a chunk's H units closer to its G units, which
// keeps the chunk's rows in L2 for the re-read at the price of less slack for
// the G^T reduction. Every wait still points at a unit dealt earlier for
// 0.5 <= lag <= 3 (H(c) after G(c); G(c)'s slot reuse after H(c - kSlots)).
int tc_unit_order(spca_sketch *h, FusedSched &s) {
  // with per-tile G^T readiness (args.tile_ready) a chunk's H units can follow
  // its G units one stage later: l_pad 64 1.630 -> 1.601 ms at config 2 (A's
  // DRAM reads 8.4 -> 6.6 GB); l_pad 128 measured equal at lag 1 and 2
  double lag = h->tc_lp == 64 ? 1.0 : 2.0;
  if (const char *e = getenv("SPCA_TC_LAGF")) lag = std::max(0.5, std::min((double)kMaxLag, atof(e)));
  const int TS = s.T * s.S * s.Gr, TlS = s.Tl * s.S * s.Gr, XR = s.X * s.RS * s.Gr, P = TS + XR;
  if (s.C >= 32768 || std::max(TS, XR) >= 32768) {  // outside the table encoding: closed form
    s.order = nullptr;
    return SPCA_OK;
  }
  const bool same = h->order_dev && h->order_C == s.C && h->order_TS == TS && h->order_TlS == TlS &&
                    h->order_XR == XR && h->order_lag == lag;
  if (!same) {
    std::vector<std::pair<double, int>> keys;
    keys.reserve(s.total);
    for (int c = 0; c < s.C; ++c) {
      const int g = c == s.C - 1 ? TlS : TS;
      for (int r = 0; r < g; ++r) keys.push_back({(double)c * P + r, (c << 15) | r});
      for (int r = 0; r < XR; ++r)
        keys.push_back({(double)c * P + TS + lag * P + r + 0.25, (1 << 30) | (c << 15) | r});
    }
    std::stable_sort(keys.begin(), keys.end(),
                     [](const std::pair<double, int> &x, const std::pair<double, int> &y) { return x.first < y.first; });
    if ((int)keys.size() != s.total) return set_err(h, SPCA_ERR_STATE, -1, "unit order size mismatch");
    std::vector<int> ord(keys.size());
    for (size_t i = 0; i < keys.size(); ++i) ord[i] = keys[i].second;
    // Round alignment. Unit u runs on pair u mod ncl, so units [j ncl, (j + 1) ncl)
    // form a "round" that the pairs execute at about the same time. The W = S Gr
    // units of one G tile pair wait for one another in their epilogues (K-split
    // reduction): a tile whose units straddle a round boundary makes the earlier
    // round's CTAs wait a whole unit (~16 us) for the later round's. Where a tile
    // would straddle, the rest of the round is filled with the next H units of an
    // EARLIER chunk instead (their G^T dependencies were dealt at least a stage
    // before; the relative order of the H units, and so every summation order,
    // is unchanged: results stay bitwise equal). Opt-in (SPCA_TC_ALIGN=1): measured
    // SLOWER (config 2 1.634 -> 1.696 ms, config 3 10.85 -> 11.92, config 5 60.5 ->
    // 66.5): with tiles pinned to round starts the pairs' G / H mix becomes static
    // (4 to 68 G units per pair instead of 49 to 57) and H units cost ~20% more than
    // G units; the default order's 79-unit stages rotate over the 74 pairs
    // (profiles/r6_align_ab.txt).
    static const int align_on = getenv("SPCA_TC_ALIGN") ? atoi(getenv("SPCA_TC_ALIGN")) : 0;
    const int ncl = std::max(1, std::min(h->max_pairs, s.total));
    const int W = s.S * s.Gr;
    if (align_on && W > 1 && W <= ncl) {
      std::vector<int> out;
      out.reserve(ord.size());
      std::vector<char> taken(ord.size(), 0);
      size_t hscan = 0;  // next candidate filler (H units are pulled in sequence order)
      for (size_t i = 0; i < ord.size(); ++i) {
        if (taken[i]) continue;
        const int e = ord[i], kind = e >> 30, c = (e >> 15) & 0x7fff, r = e & 0x7fff;
        if (kind == 0 && r % W == 0) {
          int rem = ncl - (int)(out.size() % (size_t)ncl);
          if (rem < W) {  // the tile would straddle: fill the round with H units of earlier chunks
            hscan = std::max(hscan, i + 1);
            while (rem > 0 && hscan < ord.size()) {
              const int eh = ord[hscan];
              if (!taken[hscan] && (eh >> 30) == 1) {
                if (((eh >> 15) & 0x7fff) >= c) break;  // its own G units are not dealt yet
                taken[hscan] = 1;
                out.push_back(eh);
                --rem;
              }
              ++hscan;
              if (hscan > i + 4 * (size_t)P) break;  // bounded look-ahead
            }
          }
        }
        out.push_back(e);
      }
      if (out.size() == ord.size()) ord.swap(out);
    }
    if ((int64_t)ord.size() > h->order_cap) {
      dfree(h, h->order_dev);
      h->order_dev = nullptr;
      CK(h, dalloc(h, &h->order_dev, ord.size() * sizeof(int)));
      h->order_cap = (int64_t)ord.size();
    }
    // stream-ordered after every launch that read the previous table
    CK(h, cudaMemcpyAsync(h->order_dev, ord.data(), ord.size() * sizeof(int), cudaMemcpyHostToDevice, h->stream));
    CK(h, cudaStreamSynchronize(h->stream));  // ord is about to go out of scope
    h->order_C = s.C;
    h->order_TS = TS;
    h->order_TlS = TlS;
    h->order_XR = XR;
    h->order_lag = lag;
  }
  s.order = h->order_dev;
  return SPCA_OK;
}

// Buffers of the fused row normalisation (allocated on first use)
int tc_norm_buffers(spca_sketch *h, const FusedSched &s, int64_t rows_needed) {
  if (!h->rstat_part) {
    CK(h, dalloc(h, &h->rstat_part, (size_t)kSlots * 2 * s.T * s.S * 128 * 2 * sizeof(double)));
    CK(h, dalloc(h, &h->row_a0, (size_t)kSlots * s.R0 * sizeof(float)));
    CK(h, dalloc(h, &h->row_inv, (size_t)kSlots * s.R0 * sizeof(float)));
    CK(h, dalloc(h, &h->wsum, (size_t)h->lpad * sizeof(float)));
    omega_colsums<<<(unsigned)h->lpad, 256, 0, h->stream>>>(h->omega64_dev, (int)h->n, (int)h->l, (int)h->lpad,
                                                            h->wsum);
    CK_LAUNCH(h);
  }
  if (rows_needed > h->row_coef_cap) {
    const int64_t cap = std::max<int64_t>(rows_needed, std::max<int64_t>(2 * h->row_coef_cap, 4096));
    double *nb = nullptr;
    CK(h, dalloc(h, &nb, (size_t)cap * sizeof(double)));
    if (h->row_coef && h->rows_done > 0)
      CK(h, cudaMemcpyAsync(nb, h->row_coef, (size_t)h->rows_done * sizeof(double), cudaMemcpyDeviceToDevice,
                            h->stream));
    dfree(h, h->row_coef);
    h->row_coef = nb;
    h->row_coef_cap = cap;
  }
  return SPCA_OK;
}

// One launch of the pass kernel over `rows` rows at `a` (a whole number of
// canonical chunks, or one partial chunk at the end of the stream).
int tc_launch_rows(spca_sketch *h, const void *a, int64_t lda, int64_t rows) {
  if ((lda % 4) != 0 || (reinterpret_cast<uintptr_t>(a) % 16) != 0)
    return set_err(h, SPCA_ERR_CONFIG, -1, "tensor-core path needs 16-byte aligned rows");
  FusedSched s = tc_base_sched(h);
  const bool dual = tc_dual_groups(h);
  const bool merged = dual || tc_merged_groups(h);
  s.Gr = (merged && !dual) ? h->tc_groups : 1;  // DUAL: each unit covers both groups (one per pair)
  const int ngroups = merged ? h->tc_groups : 1;  // groups one launch sketches
  s.C = (int)ceil_div(rows, s.R0);
  s.rows_last = (int)(rows - (int64_t)(s.C - 1) * s.R0);
  s.ntl = (int)ceil_div(s.rows_last, 128);
  s.Tl = (int)ceil_div(s.ntl, 2);
  s.total = fused_total(s);
  s.order = nullptr;
  if (s.C > h->tc_ctr_chunks) return set_err(h, SPCA_ERR_STATE, -1, "tc launch exceeds its counters");
  if (h->normalize) {
    const int rc = tc_norm_buffers(h, s, h->rows_done + rows);
    if (rc) return rc;
  }
  if (!getenv("SPCA_TC_CLOSED_FORM")) {
    const int orc = tc_unit_order(h, s);
    if (orc) return orc;
  }
  CUtensorMap fa_g, fa_h, fa_g3, fa_h2;
  const CUtensorMap *ta_g, *ta_h, *ta_g3, *ta_h2;
  int row_base = 0;
  const char *base = (const char *)h->src_ptr;
  const int64_t row_bytes = lda * 4;
  // cached maps over the pushed buffer: whole chunks, or a partial last chunk
  // that ends exactly where the buffer ends (rows beyond it read as zeros)
  const int64_t rb = base && (const char *)a >= base && ((const char *)a - base) % row_bytes == 0
                         ? ((const char *)a - base) / row_bytes : -1;
  if (base && lda == h->src_lda && rb >= 0 &&
      (s.rows_last == s.R0 ? rb + rows <= h->src_rows : rb + rows == h->src_rows)) {
    row_base = (int)(((const char *)a - base) / row_bytes);
    ta_g = &h->src_tg;
    ta_h = &h->src_th;
    ta_g3 = &h->src_tg3;
    ta_h2 = &h->src_th2;
  } else {  // rows beyond the launch must read as zeros (TMA out of bounds)
    int rc = encode_a_maps(h, a, (uint64_t)rows, (uint64_t)row_bytes, &fa_g, &fa_h, &fa_g3, &fa_h2);
    if (rc) return rc;
    ta_g = &fa_g;
    ta_h = &fa_h;
    ta_g3 = &fa_g3;
    ta_h2 = &fa_h2;
  }
  const size_t ctr_words = (size_t)s.C * (4 * s.T + 2) + 2 * s.X;  // per group
  const int cs = dual ? 4 : 2;  // CTAs per cluster
  const int grid = cs * std::max(1, std::min(dual ? tc_max_quads() : h->max_pairs, s.total));
#if SPCA_BULK_EPI
  // H units add into the running H at L2 (bulk reduce-add): a launch that
  // starts a flush period starts from zero instead of overwriting
  if (h->chunks_since_flush == 0) CK(h, cudaMemsetAsync(h->hpart, 0, (size_t)h->n * h->lpad * 4, h->stream));
#endif
  for (int grp = 0; grp < (merged ? 1 : h->tc_groups); ++grp) {
  CK(h, cudaMemsetAsync(h->tc_ctr, 0, (size_t)ngroups * ctr_words * 4, h->stream));
  FusedArgs args{};
  args.s = s;
  args.n = (int)h->n;
  args.row_base = row_base;
  args.gpart = (float *)h->gpart;
  args.gT = (float *)h->tc_ws;
  args.g_out = (float *)h->g_dev + h->rows_done * h->lpad + grp * h->tc_lp;
  args.hpart = (float *)h->hpart + grp * h->tc_lp;
  args.cshift = h->shift_on ? h->cshift : nullptr;
  args.g3d = h->n % 32 == 0 ? 1 : 0;
  args.left = h->left_rows ? (const float *)h->left_dev + h->rows_done * h->lpad + grp * h->tc_lp : nullptr;
  if (h->normalize) {
    args.norm = 1;
    args.rstat_part = reinterpret_cast<float *>(h->rstat_part);
    args.row_a0 = h->row_a0;
    args.row_inv = h->row_inv;
    args.row_coef = h->row_coef + h->rows_done;
    args.wsum = h->wsum + grp * h->tc_lp;
  }
  args.wy0 = grp * h->tc_lp;
  args.gld = (int)h->lpad;
  args.colsum_on = grp == 0;
  args.colsum = h->hcs_dev + h->n * h->l;
  args.carry = h->compensated ? h->carry_dev : nullptr;
  args.seg_cnt = h->tc_ctr;
  args.ready = h->tc_ctr + (size_t)s.C * 2 * s.T;
  args.hdone = args.ready + s.C;
  args.hseq = args.hdone + s.C;
  args.trdy = args.hseq + 2 * s.X;  // [C][2T]
  args.ctr_group = (int)ctr_words;   // group g's counters at + g * ctr_words
  args.gpart_group = h->gpart_elems;
  args.gT_group = (int64_t)kSlots * h->tc_gt_kparts * h->tc_lp * s.R0;
  args.gT_rows_group = kSlots * h->tc_gt_kparts * h->tc_lp;
  static const int tile_ready = getenv("SPCA_TC_TILE_READY") ? atoi(getenv("SPCA_TC_TILE_READY")) : 1;
  args.tile_ready = tile_ready;
  args.accumulate = h->chunks_since_flush > 0 ? 1 : 0;
  args.first_row = h->rows_done;
  args.a = (const float *)a;
  args.lda = lda;
  args.bad_row = h->bad_dev;
  args.trace = h->trace;
  args.dbg = h->tc_debug;
  // instantiations: plain, fused row normalisation, column shift (exclusive modes)
  auto kern = h->tc_lp == 64
                  ? (h->normalize ? tc_pass_kernel<64, true>
                                  : (h->shift_on ? tc_pass_kernel<64, false, true> : tc_pass_kernel<64, false>))
                  : dual ? (h->shift_on ? tc_pass_kernel<128, false, true, true> : tc_pass_kernel<128, false, false, true>)
                  : (h->normalize ? tc_pass_kernel<128, true>
                                  : (h->shift_on ? tc_pass_kernel<128, false, true> : tc_pass_kernel<128, false>));
  const unsigned threads = h->tc_lp == 64 ? TcCfg<64>::THREADS : TcCfg<128>::THREADS;
  const unsigned smem = h->tc_lp == 64 ? TcCfg<64>::SMEM : TcCfg<128>::SMEM;
  // The pass kernel is persistent and its CTAs wait on one another: two of
  // them sharing the GPU (handles on different streams) could each hold part
  // of the SMs and wait forever for the rest. Every launch on a device is
  // therefore ordered after the previous one, whatever its stream.
  PassSerial &ps = pass_serial(h->device);
  std::lock_guard<std::mutex> lk(ps.mu);
  if (ps.last) {
    CK(h, cudaStreamWaitEvent(h->stream, ps.last, 0));
  } else {
    CK(h, cudaEventCreateWithFlags(&ps.last, cudaEventDisableTiming));
  }
  {
    // Cooperative launch: the driver co-schedules the whole grid (every CTA
    // resident at once, whatever else runs on the device), which the
    // persistent pass's inter-CTA waits rely on; a grid that cannot be
    // co-resident fails here (cudaErrorCooperativeLaunchTooLarge) instead of
    // hanging. Clusters of two CTAs (a pair), or four (DUAL: two pairs).
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3((unsigned)grid, 1, 1);
    lc.blockDim = dim3(threads, 1, 1);
    lc.dynamicSmemBytes = smem;
    lc.stream = h->stream;
    cudaLaunchAttribute at[1];  // the cluster shape (cs) is compiled into the kernel
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = h->tc_coop ? 1 : 0;
    lc.attrs = at;
    lc.numAttrs = 1;
#if SPCA_PAIRA
    cudaError_t le = cudaLaunchKernelEx(&lc, kern, *ta_g, *ta_h, h->tm_whi, h->tm_wlo, h->tm_gT, *ta_g3, *ta_h2, args);
#else
    (void)ta_g3;
    (void)ta_h2;
    cudaError_t le = cudaLaunchKernelEx(&lc, kern, *ta_g, *ta_h, h->tm_whi, h->tm_wlo, h->tm_gT, args);
#endif
    if (le != cudaSuccess) {
      cudaGetLastError();
      return set_err(h, SPCA_ERR_CUDA, -1, "pass kernel launch (grid %d, cluster %d, cooperative %d) failed: %s",
                     grid, cs, h->tc_coop ? 1 : 0, cudaGetErrorString(le));
    }
  }
  CK_LAUNCH(h);
  CK(h, cudaEventRecord(ps.last, h->stream));
  }
  h->chunks_since_flush += s.C;
  return SPCA_OK;
}

}  // namespace
