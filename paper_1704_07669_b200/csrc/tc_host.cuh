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

EncodeTiledFn tma_encoder() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  }
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
bool tc_supported_shape(int64_t n, int64_t l) { return n >= 32 && n % 4 == 0 && l >= 1 && l <= 128; }

int tc_lpad(int64_t l) { return l <= 64 ? 64 : 128; }

// Canonical chunk: large (up to 16384 rows, ~640 MB) so the per-kernel ramp
// and tail amortise; measured on B200 this beats L2-resident chunks, whose
// G/H kernels are too short to reach steady state. Whole 128-row tiles.
int64_t tc_chunk_rows(int64_t n, int64_t /*l*/) {
  int64_t mb = 640;
  if (const char *e = getenv("SPCA_TC_CHUNK_MB")) mb = std::max<int64_t>(1, atoll(e));  // tuning knob
  int64_t r = (int64_t)(mb << 20) / (4 * n);
  r = std::max<int64_t>(128, std::min<int64_t>(16384, r));
  return (r / 128) * 128;
}

int tc_hsplit(int64_t n, int64_t /*l*/) {
  // about two waves of H tiles over the 148 SMs (the G kernel of the next
  // chunk fills the gaps from the other stream)
  int64_t tiles = ceil_div(n, 128);
  int64_t hs = std::max<int64_t>(1, std::min<int64_t>(8, (2 * 148 + tiles / 2) / tiles));
  if (const char *e = getenv("SPCA_TC_HSPLIT")) hs = std::max<int64_t>(1, atoll(e));  // tuning knob
  return (int)hs;
}

int encode_2d(spca_sketch *h, CUtensorMap *map, const void *ptr, uint64_t inner, uint64_t outer,
              uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer) {
  EncodeTiledFn enc = tma_encoder();
  if (!enc) return set_err(h, SPCA_ERR_CUDA, -1, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void *>(ptr), dims, strides, box,
                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_err(h, SPCA_ERR_CUDA, -1, "tensor map encode failed (%d): dims %llu x %llu stride %llu",
                   (int)r, (unsigned long long)inner, (unsigned long long)outer,
                   (unsigned long long)row_bytes);
  return SPCA_OK;
}

template <int LPAD>
int tc_set_smem_attrs() {
  static bool done = false;
  if (done) return 0;
  cudaError_t e1 = cudaFuncSetAttribute(tc_g_kernel<LPAD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)TcCfg<LPAD>::SMEM);
  cudaError_t e2 = cudaFuncSetAttribute(tc_h_kernel<LPAD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)TcCfg<LPAD>::SMEM);
  if (e1 != cudaSuccess || e2 != cudaSuccess) return 1;
  done = true;
  return 0;
}

int tc_setup(spca_sketch *h) {
  const int lp = tc_lpad(h->l);
  if (lp != h->lpad) {
    // the SIMT layout padded l to 32/64; the tensor-core path needs 64/128/256
    h->lpad = lp;
    h->bl = 64;
    cudaFree(h->omega_dev);
    h->omega_dev = nullptr;
    cudaFree(h->hpart);
    h->hpart = nullptr;
    CK(h, cudaMalloc(&h->omega_dev, (size_t)h->n * h->lpad * 4));
    CK(h, cudaMalloc(&h->hpart, (size_t)h->hsplit * h->n * h->lpad * 4));
    CK(h, cudaMemsetAsync(h->hpart, 0, (size_t)h->hsplit * h->n * h->lpad * 4, h->stream));
  }
  int bad = lp == 64 ? tc_set_smem_attrs<64>() : tc_set_smem_attrs<128>();
  if (bad) return set_err(h, SPCA_ERR_CUDA, -1, "cannot raise dynamic shared memory for the tc kernels");
  CK(h, cudaMalloc(&h->tc_omega, (size_t)2 * h->lpad * h->n * 4));
  float *whi = (float *)h->tc_omega;
  float *wlo = whi + (size_t)h->lpad * h->n;
  tc_omega_prepare<<<grid_for((int64_t)h->lpad * h->n), 256, 0, h->stream>>>(
      h->omega64_dev, (int)h->n, (int)h->l, (int)h->lpad, whi, wlo);
  CK_LAUNCH(h);
  int rc = encode_2d(h, &h->tm_whi, whi, (uint64_t)h->n, (uint64_t)h->lpad, (uint64_t)h->n * 4, 32, h->lpad);
  if (rc) return rc;
  rc = encode_2d(h, &h->tm_wlo, wlo, (uint64_t)h->n, (uint64_t)h->lpad, (uint64_t)h->n * 4, 32, h->lpad);
  if (rc) return rc;
  if (getenv("SPCA_TC_SERIAL"))  // profiling knob: run G and H on one stream
    h->hstream = h->stream;
  else
    CK(h, cudaStreamCreateWithFlags(&h->hstream, cudaStreamNonBlocking));
  for (int i = 0; i < 2; ++i) {
    CK(h, cudaEventCreateWithFlags(&h->ev_g[i], cudaEventDisableTiming));
    CK(h, cudaEventCreateWithFlags(&h->ev_h[i], cudaEventDisableTiming));
  }
  CK(h, cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
  // two G^T slots (hi | lo each), so G of chunk c+1 overlaps H of chunk c
  h->tc_ws_bytes = (size_t)4 * h->chunk_rows * h->lpad * 4;
  CK(h, cudaMalloc(&h->tc_ws, h->tc_ws_bytes));
  for (int slot = 0; slot < 2; ++slot) {
    float *ghi = (float *)h->tc_ws + (size_t)slot * 2 * h->chunk_rows * h->lpad;
    float *glo = ghi + (size_t)h->chunk_rows * h->lpad;
    int rs = encode_2d(h, &h->slot_tgh[slot], ghi, (uint64_t)h->chunk_rows, (uint64_t)h->lpad,
                       (uint64_t)h->chunk_rows * 4, 32, h->lpad);
    if (rs) return rs;
    rs = encode_2d(h, &h->slot_tgl[slot], glo, (uint64_t)h->chunk_rows, (uint64_t)h->lpad,
                   (uint64_t)h->chunk_rows * 4, 32, h->lpad);
    if (rs) return rs;
  }
  int64_t tiles = ceil_div(h->chunk_rows, 128);
  int64_t ksplit_max = std::max<int64_t>(1, 148 / tiles) + 1;
  h->gpart_elems = ksplit_max * tiles * 128 * h->lpad;
  CK(h, cudaMalloc(&h->gpart, (size_t)h->gpart_elems * 4));
  if (getenv("SPCA_TC_TRACE")) {
    const size_t words = (size_t)kTraceTimeline + 4 * 1024;
    CK(h, cudaMalloc(&h->trace_g, words * 8));
    CK(h, cudaMalloc(&h->trace_h, words * 8));
    std::vector<unsigned long long> init(words, 0ull);
    for (size_t i = kTraceTimeline; i < words; i += 2) init[i] = ~0ull;  // span minima
    CK(h, cudaMemcpy(h->trace_g, init.data(), words * 8, cudaMemcpyHostToDevice));
    CK(h, cudaMemcpy(h->trace_h, init.data(), words * 8, cudaMemcpyHostToDevice));
  }
  CK(h, cudaStreamSynchronize(h->stream));
  return SPCA_OK;
}

template <int LPAD>
void tc_launch(spca_sketch *h, const CUtensorMap &ta_g, const CUtensorMap &ta_h, const CUtensorMap &tgh,
               const CUtensorMap &tgl, int row_base, int rows, int ksplit, int kseg, int rseg,
               float *gout, float *ghi, float *glo, int accumulate, int slot, int64_t *launches,
               cudaError_t *err) {
  const int tiles = (int)ceil_div(rows, 128);
  const int64_t gstride = (int64_t)tiles * 128 * LPAD;
  // G^T slot reuse: the H pass that read this slot two chunks ago must be done
  if (h->h_used[slot] && (*err = cudaStreamWaitEvent(h->stream, h->ev_h[slot], 0)) != cudaSuccess) return;
  tc_g_kernel<LPAD><<<dim3(tiles, ksplit), kTcThreads, TcCfg<LPAD>::SMEM, h->stream>>>(
      ta_g, h->tm_whi, h->tm_wlo, rows, (int)h->n, kseg, row_base, (float *)h->gpart, gstride,
      h->rows_done, h->bad_dev, h->tc_debug, h->trace_g, (int)h->chunk_seq);
  if ((*err = cudaGetLastError()) != cudaSuccess) return;
  ++*launches;
  tc_g_finalize<<<dim3((unsigned)ceil_div(rows, 8), LPAD / 32), dim3(32, 8), 0, h->stream>>>(
      (const float *)h->gpart, ksplit, gstride, rows, LPAD, (int)h->chunk_rows, gout, ghi, glo);
  if ((*err = cudaGetLastError()) != cudaSuccess) return;
  ++*launches;
  if ((*err = cudaEventRecord(h->ev_g[slot], h->stream)) != cudaSuccess) return;
  if ((*err = cudaStreamWaitEvent(h->hstream, h->ev_g[slot], 0)) != cudaSuccess) return;
  // H of this chunk runs on the second stream, concurrently with G of the next
  tc_h_kernel<LPAD><<<dim3((unsigned)ceil_div(h->n, 128), h->hsplit), kTcThreads, TcCfg<LPAD>::SMEM,
                      h->hstream>>>(ta_h, tgh, tgl, rows, (int)h->n, rseg, row_base, (float *)h->hpart,
                                    (int64_t)h->n * LPAD, h->cspart, accumulate, h->compensated ? 1 : 0,
                                    h->tc_debug >> 8, h->trace_h, (int)h->chunk_seq);
  if ((*err = cudaGetLastError()) != cudaSuccess) return;
  ++*launches;
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
  int rc = encode_2d(h, &h->src_tg, a, (uint64_t)h->n, (uint64_t)rows, (uint64_t)lda * 4, 32, 128);
  if (rc) return rc;
  rc = encode_2d(h, &h->src_th, a, (uint64_t)h->n, (uint64_t)rows, (uint64_t)lda * 4, 32, 32);
  if (rc) return rc;
  h->src_ptr = a;
  h->src_rows = rows;
  h->src_lda = lda;
  return SPCA_OK;
}

int tc_chunk(spca_sketch *h, const void *a, int64_t lda, int rows) {
  if ((lda % 4) != 0 || (reinterpret_cast<uintptr_t>(a) % 16) != 0)
    return set_err(h, SPCA_ERR_CONFIG, -1, "tensor-core path needs 16-byte aligned rows");
  const int slot = (int)(h->chunk_seq & 1);
  float *ghi = (float *)h->tc_ws + (size_t)slot * 2 * h->chunk_rows * h->lpad;
  float *glo = ghi + (size_t)h->chunk_rows * h->lpad;
  CUtensorMap fa_g, fa_h, fg_h, fg_l;
  const CUtensorMap *ta_g, *ta_h, *tgh, *tgl;
  int row_base = 0;
  const char *base = (const char *)h->src_ptr;
  const int64_t row_bytes = lda * 4;
  const bool full = rows == h->chunk_rows;
  if (full && base && lda == h->src_lda && (const char *)a >= base &&
      ((const char *)a - base) % row_bytes == 0 &&
      ((const char *)a - base) / row_bytes + rows <= h->src_rows) {
    row_base = (int)(((const char *)a - base) / row_bytes);
    ta_g = &h->src_tg;
    ta_h = &h->src_th;
  } else {
    int rc = encode_2d(h, &fa_g, a, (uint64_t)h->n, (uint64_t)rows, (uint64_t)row_bytes, 32, 128);
    if (rc) return rc;
    rc = encode_2d(h, &fa_h, a, (uint64_t)h->n, (uint64_t)rows, (uint64_t)row_bytes, 32, 32);
    if (rc) return rc;
    ta_g = &fa_g;
    ta_h = &fa_h;
  }
  if (full) {
    tgh = &h->slot_tgh[slot];
    tgl = &h->slot_tgl[slot];
  } else {  // partial chunk: rows beyond it must read as zeros (TMA out of bounds)
    int rc = encode_2d(h, &fg_h, ghi, (uint64_t)rows, (uint64_t)h->lpad, (uint64_t)h->chunk_rows * 4, 32, h->lpad);
    if (rc) return rc;
    rc = encode_2d(h, &fg_l, glo, (uint64_t)rows, (uint64_t)h->lpad, (uint64_t)h->chunk_rows * 4, 32, h->lpad);
    if (rc) return rc;
    tgh = &fg_h;
    tgl = &fg_l;
  }
  const int64_t tiles = ceil_div(rows, 128);
  int ksplit = (int)std::max<int64_t>(1, 148 / tiles);
  int kseg = (int)round_up(ceil_div(h->n, ksplit), 32);
  ksplit = (int)ceil_div(h->n, kseg);
  if ((int64_t)ksplit * tiles * 128 * h->lpad > h->gpart_elems)
    return set_err(h, SPCA_ERR_STATE, -1, "tc workspace too small");
  const int rseg = (int)round_up(ceil_div(rows, h->hsplit), 32);
  float *gout = (float *)h->g_dev + h->rows_done * h->lpad;
  const int acc = h->chunks_since_flush > 0 ? 1 : 0;
  cudaError_t err = cudaSuccess;
  if (h->lpad == 64)
    tc_launch<64>(h, *ta_g, *ta_h, *tgh, *tgl, row_base, rows, ksplit, kseg, rseg, gout, ghi, glo, acc, slot,
                  &h->launches, &err);
  else
    tc_launch<128>(h, *ta_g, *ta_h, *tgh, *tgl, row_base, rows, ksplit, kseg, rseg, gout, ghi, glo, acc, slot,
                   &h->launches, &err);
  if (err != cudaSuccess)
    return set_err(h, SPCA_ERR_CUDA, -1, "tc kernel launch failed: %s", cudaGetErrorString(err));
  h->chunk_seq++;
  return SPCA_OK;
}

}  // namespace
