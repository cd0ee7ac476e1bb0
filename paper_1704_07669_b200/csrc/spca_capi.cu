// spca_capi.cu — the C ABI of libspca.so (see include/spca.h).
//
// Owns the sketch accumulators on one GPU, re-chunks pushed rows into
// canonical chunks, stages host rows through pinned double buffers on a
// copy stream (host streaming) and launches the contraction
// kernels per chunk on the handle's compute stream.

#include <cuda_runtime.h>

#include <dlfcn.h>
#include <nccl.h>  // types and enums only: the library is resolved at run time (dlopen)

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <thread>
#include <vector>

#include "../../include/spca.h"
#include "common.cuh"
#include "epilogue.cuh"
#include "sketch_simt.cuh"
#include "handle.cuh"
#include "normalize.cuh"
#include "postpass.cuh"
#include "omega_rng.cuh"

using namespace spca;

namespace {

thread_local int g_tl_code = SPCA_OK;
thread_local char g_tl_msg[512] = {0};

int set_err(spca_sketch *h, int code, int64_t row, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (h) {
    h->last_code = code;
    h->last_bad_row = row;
    snprintf(h->last_msg, sizeof h->last_msg, "%s", buf);
  }
  g_tl_code = code;
  snprintf(g_tl_msg, sizeof g_tl_msg, "%s", buf);
  return code;
}

#define CK(h, call)                                                                        \
  do {                                                                                     \
    cudaError_t _e = (call);                                                               \
    if (_e != cudaSuccess) {                                                               \
      return set_err((h), _e == cudaErrorMemoryAllocation ? SPCA_ERR_OOM : SPCA_ERR_CUDA,  \
                     -1, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(_e), __FILE__, \
                     __LINE__);                                                            \
    }                                                                                      \
  } while (0)

#define CK_LAUNCH(h)                                                                       \
  do {                                                                                     \
    cudaError_t _e = cudaGetLastError();                                                   \
    if (_e != cudaSuccess)                                                                 \
      return set_err((h), SPCA_ERR_CUDA, -1, "kernel launch failed: %s (%s:%d)",          \
                     cudaGetErrorString(_e), __FILE__, __LINE__);                          \
    (h)->launches++;                                                                       \
  } while (0)

// Device buffers of a handle come from the device's stream-ordered pool
// (cudaMallocAsync / cudaFreeAsync on the handle's stream) whose release
// threshold is raised once per device: creating and destroying a handle
// then costs microseconds, where cudaMalloc / cudaFree (which synchronizes
// the device) cost milliseconds per pass. Buffers also touched by the copy
// stream (the host staging ring) keep plain cudaMalloc.
std::mutex g_pool_mu;
bool g_pool_ready[64];

void ensure_pool(int dev) {
  std::lock_guard<std::mutex> lk(g_pool_mu);
  if (dev < 0 || dev >= 64 || g_pool_ready[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  g_pool_ready[dev] = true;
}

cudaError_t dalloc(spca_sketch *h, void **p, size_t bytes) {
  return cudaMallocAsync(p, std::max<size_t>(bytes, 1), h->stream);
}
template <typename T>
cudaError_t dalloc(spca_sketch *h, T **p, size_t bytes) {
  return dalloc(h, reinterpret_cast<void **>(p), bytes);
}
void dfree(spca_sketch *h, void *p) {
  if (p) cudaFreeAsync(p, h->stream);
}

// Page-locked staging buffers cost ~0.3 s per GB to create (cudaHostAlloc
// pins every page), which a one-shot call such as single_pass_pca on a numpy
// array would pay on each call: handles take them from, and give them back
// to, a process-wide free list (portable allocations, any device; at most
// kPinnedCache bytes kept).
constexpr size_t kPinnedCache = size_t(4) << 30;
struct PinnedPool {
  std::mutex mu;
  std::vector<std::pair<size_t, void *>> free;
  size_t cached = 0;
};
PinnedPool &pinned_pool() {
  static PinnedPool *p = new PinnedPool;  // never destroyed: handles may outlive static teardown
  return *p;
}
cudaError_t pinned_get(void **p, size_t bytes) {
  PinnedPool &pp = pinned_pool();
  {
    std::lock_guard<std::mutex> lk(pp.mu);
    for (size_t i = 0; i < pp.free.size(); ++i) {
      if (pp.free[i].first == bytes) {
        *p = pp.free[i].second;
        pp.cached -= bytes;
        pp.free.erase(pp.free.begin() + (long)i);
        return cudaSuccess;
      }
    }
  }
  return cudaHostAlloc(p, bytes, cudaHostAllocPortable);
}
void pinned_put(void *p, size_t bytes) {
  if (!p) return;
  PinnedPool &pp = pinned_pool();
  std::lock_guard<std::mutex> lk(pp.mu);
  while (pp.cached + bytes > kPinnedCache && !pp.free.empty()) {  // oldest first
    cudaFreeHost(pp.free.front().second);
    pp.cached -= pp.free.front().first;
    pp.free.erase(pp.free.begin());
  }
  if (bytes > kPinnedCache) {
    cudaFreeHost(p);
    return;
  }
  pp.free.emplace_back(bytes, p);
  pp.cached += bytes;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

int grid_for(int64_t count, int threads = 256) {
  int64_t b = ceil_div(count, threads);
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 16));
}

int ensure_g(spca_sketch *h, int64_t rows_needed) {
  if (rows_needed <= h->g_cap) return SPCA_OK;
  int64_t cap = std::max<int64_t>(rows_needed, std::max<int64_t>(h->g_cap * 2, 4096));
  void *nb = nullptr;
  CK(h, dalloc(h, &nb, (size_t)cap * h->lpad * h->ds));
  if (h->g_dev && h->rows_done > 0) {
    CK(h, cudaMemcpyAsync(nb, h->g_dev, (size_t)h->rows_done * h->lpad * h->ds,
                          cudaMemcpyDeviceToDevice, h->stream));
  }
  dfree(h, h->g_dev);  // stream-ordered after the copy
  h->g_dev = nb;
  h->g_cap = cap;
  return SPCA_OK;
}

}  // namespace

// tensor-core path (uses set_err / CK / grid_for above)
#include "sketch_fused.cuh"
#include "tc_host.cuh"

#ifndef SPCA_SIMT_F64_TILE
#define SPCA_SIMT_F64_TILE 64  // 128 (two DMMA row tiles per warp, 8-deep K) measured 14.0 vs 12.3 ms
#endif

namespace {

// ---- SIMT chunk processing ------------------------------------------------
// Grid sizing of the SIMT path (CTAs per SM aimed at by the G split-K and the
// H row splits) and its canonical chunk (MB of A); env overrides for tuning.
int env_int(const char *name, int dflt) {
  const char *e = getenv(name);
  return e ? std::max(1, atoi(e)) : dflt;
}
const int kSimtGTarget = env_int("SPCA_SIMT_G_CTAS", 8);
const int kSimtHTarget = env_int("SPCA_SIMT_H_CTAS", 8);  // measured: 2 -> 8 = -15% at config 2 (fp64 31.7 -> 27.1 ms)
const int kSimtChunkMB = env_int("SPCA_SIMT_CHUNK_MB", 320);  // G split-K 8 CTAs/SM + 320 MB chunks: fp64 14.6 -> 12.3 ms

template <typename T, int BM, int BL, bool VEC>
void launch_g(spca_sketch *h, const T *a, int64_t lda, int rows, T *out, int64_t out_stride,
              int ksplit, int kseg) {
  dim3 grid((unsigned)ceil_div(rows, BM), (unsigned)(h->lpad / BL), (unsigned)ksplit);
  // fp64 with 128-row tiles: 8-deep K steps keep the double-buffered tiles under 48 KB
  simt_g_kernel<T, BM, BL, (sizeof(T) == 4 ? 32 : (BM > 64 && BL > 32 ? 8 : 16)), VEC><<<grid, kSimtThreads, 0, h->stream>>>(
      a, lda, rows, (int)h->n, (const T *)h->omega_dev, (int)h->lpad, out, (int)h->lpad,
      out_stride, kseg, h->rows_done, h->bad_dev);
}

template <typename T, int BN, int BL, bool VEC>
void launch_h(spca_sketch *h, const T *a, int64_t lda, int rows, const T *g, int rseg, int accumulate) {
  dim3 grid((unsigned)ceil_div(h->n, BN), (unsigned)(h->lpad / BL), (unsigned)h->hsplit);
  simt_h_kernel<T, BN, BL, (sizeof(T) == 4 ? 32 : (BN > 64 && BL > 32 ? 8 : 16)), VEC><<<grid, kSimtThreads, 0, h->stream>>>(
      a, lda, rows, (int)h->n, g, (int)h->lpad, (T *)h->hpart, (int)h->lpad,
      (int64_t)h->n * h->lpad, h->cspart, rseg, accumulate, h->compensated ? 1 : 0);
}

// tile rows (G) / columns (H) of the 64-wide l tiles: 64 for FFMA, 128 for
// fp64 (two 16-row DMMA tiles per warp: each B fragment feeds two MMAs)
template <typename T>
constexpr int kGM = sizeof(T) == 8 ? SPCA_SIMT_F64_TILE : 64;

template <typename T>
int simt_chunk(spca_sketch *h, const T *a, int64_t lda, int rows) {
  constexpr int VN = Vec<T>::n;
  const bool vec = (lda % VN == 0) && (h->n % VN == 0) &&
                   ((reinterpret_cast<uintptr_t>(a) % 16) == 0);
  const bool narrow = (h->bl == 32);
  const int bm = narrow ? 128 : kGM<T>;
  // split-K so that the G kernel fills the machine (~4 CTAs per SM)
  int64_t tiles = ceil_div(rows, bm) * (h->lpad / h->bl);
  int64_t kmax = std::max<int64_t>(1, ceil_div(h->n, 128));
  int ksplit = (int)std::min<int64_t>(kmax, std::max<int64_t>(1, ceil_div(148 * kSimtGTarget, tiles)));
  int kseg = (int)round_up(ceil_div(h->n, ksplit), 32);
  ksplit = (int)ceil_div(h->n, kseg);
  T *gout = (T *)h->g_dev + h->rows_done * h->lpad;
  T *p1_out = gout;
  int64_t p1_stride = 0;
  if (ksplit > 1) {
    int64_t need = (int64_t)ksplit * rows * h->lpad;
    if (need > h->gpart_elems) {
      dfree(h, h->gpart);
      h->gpart = nullptr;
      CK(h, dalloc(h, &h->gpart, (size_t)need * h->ds));
      h->gpart_elems = need;
    }
    p1_out = (T *)h->gpart;
    p1_stride = (int64_t)rows * h->lpad;
  }
  if (narrow) {
    if (vec) launch_g<T, 128, 32, true>(h, a, lda, rows, p1_out, p1_stride, ksplit, kseg);
    else launch_g<T, 128, 32, false>(h, a, lda, rows, p1_out, p1_stride, ksplit, kseg);
  } else {
    if (vec) launch_g<T, kGM<T>, 64, true>(h, a, lda, rows, p1_out, p1_stride, ksplit, kseg);
    else launch_g<T, kGM<T>, 64, false>(h, a, lda, rows, p1_out, p1_stride, ksplit, kseg);
  }
  CK_LAUNCH(h);
  if (ksplit > 1) {
    int64_t count = (int64_t)rows * h->lpad;
    simt_g_reduce<T><<<grid_for(count), 256, 0, h->stream>>>((const T *)h->gpart, ksplit,
                                                              p1_stride, count, gout);
    CK_LAUNCH(h);
  }
  int rseg = (int)round_up(ceil_div(rows, h->hsplit), 32);
  int acc = h->chunks_since_flush > 0 ? 1 : 0;
  // co-sketch: the H contraction takes the left operand's rows instead of G
  const T *hop = h->left_rows ? (const T *)h->left_dev + h->rows_done * h->lpad : gout;
  if (narrow) {
    if (vec) launch_h<T, 128, 32, true>(h, a, lda, rows, hop, rseg, acc);
    else launch_h<T, 128, 32, false>(h, a, lda, rows, hop, rseg, acc);
  } else {
    if (vec) launch_h<T, kGM<T>, 64, true>(h, a, lda, rows, hop, rseg, acc);
    else launch_h<T, kGM<T>, 64, false>(h, a, lda, rows, hop, rseg, acc);
  }
  CK_LAUNCH(h);
  return SPCA_OK;
}

int flush_h(spca_sketch *h) {
  if (h->chunks_since_flush == 0) return SPCA_OK;
  int64_t count = h->n * h->l;
  if (h->dtype == SPCA_F32)
    h_flush<float><<<grid_for(count), 256, 0, h->stream>>>(
        (const float *)h->hpart, h->hsplit, h->n * h->lpad, (int)h->n, (int)h->l, (int)h->lpad,
        h->hcs_dev);
  else
    h_flush<double><<<grid_for(count), 256, 0, h->stream>>>(
        (const double *)h->hpart, h->hsplit, h->n * h->lpad, (int)h->n, (int)h->l, (int)h->lpad,
        h->hcs_dev);
  CK_LAUNCH(h);
  h->chunks_since_flush = 0;
  return SPCA_OK;
}

void open_timing(spca_sketch *h) {
  if (h->timing && !h->t_open) {
    if (!h->t_start) cudaEventCreate(&h->t_start);
    if (!h->t_stop) cudaEventCreate(&h->t_stop);
    cudaEventRecord(h->t_start, h->stream);
    h->t_open = true;
    h->t_chunks = 0;
  }
}

int close_timing(spca_sketch *h, int64_t chunks) {
  if (h->timing) {
    CK(h, cudaEventRecord(h->t_stop, h->stream));
    h->t_chunks += chunks;
  }
  return SPCA_OK;
}

// normalize_rows kernels (csrc/normalize.cuh): the register-resident vector
// variant when the rows fit and are 16-byte aligned, else the three-sweep one
cudaError_t launch_normalize(const void *src, int64_t rows, int64_t n, int64_t ld_src, void *dst, int64_t ld_dst,
                             int dtype, cudaStream_t st) {
  const unsigned grid = (unsigned)std::min<int64_t>(rows, 148 * 8);
  const int64_t es = dtype == SPCA_F32 ? 4 : 8, ev = 16 / es;
  const bool vec = n % ev == 0 && ld_src % ev == 0 && ld_dst % ev == 0 &&
                   (reinterpret_cast<uintptr_t>(src) % 16) == 0 && (reinterpret_cast<uintptr_t>(dst) % 16) == 0;
  constexpr int kNV = 12;  // vectors per thread: rows up to 12288 fp32 / 6144 fp64 stay in registers
  if (vec && n <= (int64_t)kNormThreads * kNV * ev) {
    if (dtype == SPCA_F32)
      normalize_rows_vec_kernel<float, kNV><<<grid, kNormThreads, 0, st>>>((const float *)src, rows, n, ld_src,
                                                                           (float *)dst, ld_dst);
    else
      normalize_rows_vec_kernel<double, kNV><<<grid, kNormThreads, 0, st>>>((const double *)src, rows, n, ld_src,
                                                                            (double *)dst, ld_dst);
  } else if (dtype == SPCA_F32) {
    normalize_rows_kernel<float><<<grid, kNormThreads, 0, st>>>((const float *)src, rows, n, ld_src,
                                                                 (float *)dst, ld_dst);
  } else {
    normalize_rows_kernel<double><<<grid, kNormThreads, 0, st>>>((const double *)src, rows, n, ld_src,
                                                                  (double *)dst, ld_dst);
  }
  return cudaGetLastError();
}

// SIMT path: one canonical chunk (G, H, column sums), flush every ~1M rows
int process_chunk(spca_sketch *h, const void *a, int64_t lda, int64_t rows) {
  if (rows <= 0) return SPCA_OK;
  int rc = ensure_g(h, h->rows_done + rows);
  if (rc) return rc;
  if (h->normalize) {  // unfused on this path: normalize the chunk into a workspace first
    if (!h->norm_ws) CK(h, dalloc(h, &h->norm_ws, (size_t)h->chunk_rows * h->n * h->ds));
    CK(h, launch_normalize(a, rows, h->n, lda, h->norm_ws, h->n, h->dtype, h->stream));
    h->launches++;
    a = h->norm_ws;
    lda = h->n;
  } else if (h->shift_on) {  // column shift: the chunk minus 1 c^T into a workspace
    if (!h->norm_ws) CK(h, dalloc(h, &h->norm_ws, (size_t)h->chunk_rows * h->n * h->ds));
    if (h->dtype == SPCA_F32)
      shift_rows<float><<<grid_for(rows * h->n), 256, 0, h->stream>>>((const float *)a, rows, (int)h->n, lda,
                                                                      h->cshift, (float *)h->norm_ws, h->n);
    else
      shift_rows<double><<<grid_for(rows * h->n), 256, 0, h->stream>>>((const double *)a, rows, (int)h->n, lda,
                                                                       h->cshift, (double *)h->norm_ws, h->n);
    CK_LAUNCH(h);
    a = h->norm_ws;
    lda = h->n;
  }
  open_timing(h);
  if (h->dtype == SPCA_F32) {
    rc = simt_chunk<float>(h, (const float *)a, lda, (int)rows);
  } else {
    rc = simt_chunk<double>(h, (const double *)a, lda, (int)rows);
  }
  if (rc) return rc;
  colsum_accumulate<<<(unsigned)ceil_div(h->n, 256), 256, 0, h->stream>>>(
      h->cspart, h->hsplit, (int)h->n, h->hcs_dev + h->n * h->l,
      h->compensated ? h->carry_dev : nullptr);
  CK_LAUNCH(h);
  h->chunks_since_flush++;
  if (h->chunks_since_flush >= h->flush_every) {
    rc = flush_h(h);
    if (rc) return rc;
  }
  rc = close_timing(h, 1);
  if (rc) return rc;
  h->rows_done += rows;
  return SPCA_OK;
}

// Tensor-core path: `rows` rows (whole canonical chunks, or the final partial
// chunk) through the pass kernel, in launches that end at H flush points.
int process_rows_tc(spca_sketch *h, const char *a, int64_t lda, int64_t rows) {
  int rc = ensure_g(h, h->rows_done + rows);
  if (rc) return rc;
  open_timing(h);
  int64_t off = 0, chunks = 0;
  while (off < rows) {
    const int64_t room = std::max<int64_t>(1, h->flush_every - h->chunks_since_flush);
    const int64_t take = std::min<int64_t>(rows - off, room * h->chunk_rows);
    rc = tc_launch_rows(h, a + (size_t)off * lda * 4, lda, take);
    if (rc) return rc;
    h->rows_done += take;
    chunks += ceil_div(take, h->chunk_rows);
    off += take;
    if (h->chunks_since_flush >= h->flush_every) {
      rc = flush_h(h);
      if (rc) return rc;
    }
  }
  return close_timing(h, chunks);
}

int push_host_rows(spca_sketch *h, const char *a, int64_t rows, int64_t lda, bool pageable, bool final = false,
                   bool device_src = false);

// Rows already on the device: feed canonical chunks, keep the remainder in `tail`.
int push_device_rows(spca_sketch *h, const char *a, int64_t rows, int64_t lda, bool final = false) {
  const int64_t R0 = h->chunk_rows;
  const size_t row_bytes = (size_t)h->n * h->ds;
  const size_t pitch = (size_t)h->ldp * h->ds;  // rows of the library's own buffers
  int64_t off = 0;
  // TMA addresses rows whose stride is a multiple of 16 bytes from a 16-byte
  // aligned base; other sources are re-strided through the staging ring
  const bool tma_ok = lda % 4 == 0 && (reinterpret_cast<uintptr_t>(a) % 16) == 0;
  if (h->precision == SPCA_PREC_TC && !tma_ok)  // re-strided on the copy stream, overlapped with the pass
    return push_host_rows(h, a, rows, lda, false, final, true);
  if (h->precision == SPCA_PREC_TC) {
    int rr = tc_register_source(h, a, rows, lda);
    if (rr) return rr;
  }
  if (h->tail_rows > 0) {
    int64_t take = std::min(R0 - h->tail_rows, rows);
    CK(h, cudaMemcpy2DAsync((char *)h->tail + h->tail_rows * pitch, pitch, a,
                            (size_t)lda * h->ds, row_bytes, (size_t)take,
                            cudaMemcpyDeviceToDevice, h->stream));
    h->tail_rows += take;
    off = take;
    if (h->tail_rows == R0) {
      int rc = h->precision == SPCA_PREC_TC ? process_rows_tc(h, (const char *)h->tail, h->ldp, R0)
                                            : process_chunk(h, h->tail, h->ldp, R0);
      if (rc) return rc;
      h->tail_rows = 0;
    }
  }
  if (h->precision == SPCA_PREC_TC) {  // all whole chunks (and a final partial one) in one go
    const int64_t take = final ? rows - off : ((rows - off) / R0) * R0;
    if (take > 0) {
      int rc = process_rows_tc(h, a + (size_t)off * lda * h->ds, lda, take);
      if (rc) return rc;
      off += take;
    }
  }
  while (rows - off >= R0) {
    int rc = process_chunk(h, a + (size_t)off * lda * h->ds, lda, R0);
    if (rc) return rc;
    off += R0;
  }
  if (off < rows && final) {  // SIMT path: the last partial chunk straight from the source
    int rc = process_chunk(h, a + (size_t)off * lda * h->ds, lda, rows - off);
    if (rc) return rc;
    off = rows;
  }
  if (off < rows) {
    int64_t rem = rows - off;
    CK(h, cudaMemcpy2DAsync((char *)h->tail, pitch, a + (size_t)off * lda * h->ds,
                            (size_t)lda * h->ds, row_bytes, (size_t)rem,
                            cudaMemcpyDeviceToDevice, h->stream));
    h->tail_rows = rem;
  }
  return SPCA_OK;
}

// Pageable rows into the page-locked staging buffer on several host threads:
// one thread's memcpy (~14 GB/s) would cap a numpy input far below the
// host link (~55 GB/s); pieces of >= 32 MB per thread.
const unsigned kCopyThreads = (unsigned)env_int("SPCA_COPY_THREADS", 16);

void host_rows_copy(char *dst, size_t dpitch, const char *src, size_t spitch, size_t row_bytes, int64_t rows,
                    int min_shift = 25) {
  auto copy = [=](int64_t r0, int64_t r1) {
    if (dpitch == spitch && dpitch == row_bytes) {
      memcpy(dst + r0 * dpitch, src + r0 * spitch, (size_t)(r1 - r0) * row_bytes);
    } else {
      for (int64_t r = r0; r < r1; ++r) memcpy(dst + r * dpitch, src + r * spitch, row_bytes);
    }
  };
  const int64_t bytes = rows * (int64_t)row_bytes;
  if (rows == 1 && row_bytes >= (8u << 20)) {  // one long run: split it into byte ranges
    constexpr int64_t kSeg = 4 << 20;
    host_rows_copy(dst, (size_t)kSeg, src, (size_t)kSeg, (size_t)kSeg, bytes / kSeg, min_shift);
    const int64_t done = (bytes / kSeg) * kSeg;
    if (done < bytes) memcpy(dst + done, src + done, (size_t)(bytes - done));
    return;
  }
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const int nt = (int)std::min<int64_t>(std::min<unsigned>(hw, kCopyThreads), std::max<int64_t>(1, bytes >> min_shift));
  if (nt <= 1) {
    copy(0, rows);
    return;
  }
  std::vector<std::thread> pool;
  const int64_t per = (rows + nt - 1) / nt;
  int64_t mine_end = std::min(rows, per);  // this thread's share (grows if a spawn fails)
  for (int t = 1; t < nt; ++t) {
    const int64_t r0 = t * per, r1 = std::min(rows, r0 + per);
    if (r0 >= r1) break;
    try {
      pool.emplace_back(copy, r0, r1);
    } catch (...) {  // no more threads: this thread copies the rest itself
      mine_end = -r0;
      break;
    }
  }
  if (mine_end < 0) copy(-mine_end, rows);  // the part no thread took
  copy(0, std::min(rows, per));
  for (auto &th : pool) th.join();
}

// Large pageable uploads (Omega, the co-sketch operand): through two
// page-locked 32 MB bounce buffers, each filled by host_rows_copy on up to
// 8 threads (4 MB per thread) while the previous one is in flight (a pageable
// cudaMemcpy runs at ~10-14 GB/s). The buffers are allocated once per process
// (portable: any device may use them, one upload at a time under the mutex);
// the completion events belong to the call and to the current device.
// Synchronous on return, also on every error path (no copy out of a bounce
// buffer is left in flight for the next caller to overwrite).
cudaError_t upload_pageable(void *dst, const void *src, size_t bytes, cudaStream_t st) {
  constexpr size_t kBounce = 32u << 20;
  static std::mutex mu;
  static void *bounce[2] = {nullptr, nullptr};
  if (bytes < 2 * kBounce) return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st);
  std::lock_guard<std::mutex> lk(mu);
  for (int i = 0; i < 2; ++i) {
    if (!bounce[i]) {
      cudaError_t e = cudaHostAlloc(&bounce[i], kBounce, cudaHostAllocPortable);
      if (e != cudaSuccess) return e;
    }
  }
  cudaEvent_t done[2] = {nullptr, nullptr};
  bool recorded[2] = {false, false};
  cudaError_t e = cudaSuccess;
  for (int i = 0; i < 2 && e == cudaSuccess; ++i) e = cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming);
  size_t off = 0;
  for (int k = 0; e == cudaSuccess && off < bytes; ++k) {
    const int i = k & 1;
    const size_t n = std::min(kBounce, bytes - off);
    if (recorded[i]) {
      e = cudaEventSynchronize(done[i]);  // the buffer's previous copy has landed
      if (e != cudaSuccess) break;
    }
    host_rows_copy((char *)bounce[i], n, (const char *)src + off, n, n, 1, 22);
    e = cudaMemcpyAsync((char *)dst + off, bounce[i], n, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaEventRecord(done[i], st);
    if (e == cudaSuccess) recorded[i] = true;
    off += n;
  }
  cudaError_t es = cudaStreamSynchronize(st);  // nothing left in flight, success or not
  for (int i = 0; i < 2; ++i)
    if (done[i]) cudaEventDestroy(done[i]);
  return e != cudaSuccess ? e : es;
}

int ensure_staging(spca_sketch *h, bool need_pinned) {
  const size_t bytes = (size_t)h->stage_rows * h->ldp * h->ds;
  for (int i = 0; i < 2; ++i) {
    if (!h->dstage[i]) CK(h, cudaMalloc(&h->dstage[i], bytes));
    if (!h->copy_done[i]) CK(h, cudaEventCreateWithFlags(&h->copy_done[i], cudaEventDisableTiming));
    if (!h->comp_done[i]) CK(h, cudaEventCreateWithFlags(&h->comp_done[i], cudaEventDisableTiming));
    if (need_pinned && !h->pinned[i]) CK(h, pinned_get(&h->pinned[i], bytes));
  }
  if (!h->copy_stream) CK(h, cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking));
  return SPCA_OK;
}

// Rows staged through the double-buffered device staging ring on the copy
// stream: host rows (pinned or pageable), or device rows whose stride the
// pass kernel's TMA cannot address (device_src: re-strided D2D copies)
int push_host_rows(spca_sketch *h, const char *a, int64_t rows, int64_t lda, bool pageable, bool final,
                   bool device_src) {
  int rc = ensure_staging(h, pageable);
  if (rc) return rc;
  if (device_src) {  // the copy stream must see the work that produced the rows
    if (!h->src_ready) CK(h, cudaEventCreateWithFlags(&h->src_ready, cudaEventDisableTiming));
    CK(h, cudaEventRecord(h->src_ready, h->stream));
    CK(h, cudaStreamWaitEvent(h->copy_stream, h->src_ready, 0));
  }
  const size_t row_bytes = (size_t)h->n * h->ds;
  const size_t pitch = (size_t)h->ldp * h->ds;  // staging rows (16-byte multiple on the TC path)
  int64_t off = 0;
  while (off < rows) {
    int64_t take = std::min(h->stage_rows, rows - off);
    int i = h->stage_idx;
    h->stage_idx ^= 1;
    // the device buffer i is free once the compute that read it is done
    if (h->stage_used[i]) CK(h, cudaStreamWaitEvent(h->copy_stream, h->comp_done[i], 0));
    const char *src = a + (size_t)off * lda * h->ds;
    if (pageable) {
      if (h->stage_used[i]) CK(h, cudaEventSynchronize(h->copy_done[i]));
      char *dst = (char *)h->pinned[i];
      host_rows_copy(dst, pitch, src, (size_t)lda * h->ds, row_bytes, take);
      src = dst;
      CK(h, cudaMemcpyAsync(h->dstage[i], src, (size_t)take * pitch, cudaMemcpyHostToDevice,
                            h->copy_stream));
    } else {
      if (device_src) {  // a copy kernel (2-D DMA of odd-pitched rows is slow)
        if (h->dtype == SPCA_F32)
          restride_rows<float><<<148 * 8, 256, 0, h->copy_stream>>>((const float *)src, lda, take, (int)h->n,
                                                                    (float *)h->dstage[i], h->ldp);
        else
          restride_rows<double><<<148 * 8, 256, 0, h->copy_stream>>>((const double *)src, lda, take, (int)h->n,
                                                                     (double *)h->dstage[i], h->ldp);
        CK_LAUNCH(h);
      } else {
        CK(h, cudaMemcpy2DAsync(h->dstage[i], pitch, src, (size_t)lda * h->ds, row_bytes, (size_t)take,
                                cudaMemcpyHostToDevice, h->copy_stream));
      }
    }
    CK(h, cudaEventRecord(h->copy_done[i], h->copy_stream));
    CK(h, cudaStreamWaitEvent(h->stream, h->copy_done[i], 0));
    rc = push_device_rows(h, (const char *)h->dstage[i], take, h->ldp, final && off + take == rows);
    if (rc) return rc;
    CK(h, cudaEventRecord(h->comp_done[i], h->stream));
    h->stage_used[i] = true;
    off += take;
  }
  return SPCA_OK;
}

int collect_timers(spca_sketch *h) {
  if (h->t_open) {
    float ms = 0.f;
    CK(h, cudaEventSynchronize(h->t_stop));
    CK(h, cudaEventElapsedTime(&ms, h->t_start, h->t_stop));
    h->kernel_ms += ms;
    h->timed_chunks += h->t_chunks;
    h->t_open = false;
    h->t_chunks = 0;
  }
  return SPCA_OK;
}

int check_bad_row(spca_sketch *h) {
  unsigned long long bad = 0;
  CK(h, cudaMemcpyAsync(&bad, h->bad_dev, sizeof bad, cudaMemcpyDeviceToHost, h->stream));
  CK(h, cudaStreamSynchronize(h->stream));
  if (bad != (unsigned long long)kNoBadRow) {
    return set_err(h, SPCA_ERR_DATA, (int64_t)bad, "non-finite value in row %lld", (long long)bad);
  }
  return SPCA_OK;
}

}  // namespace

extern "C" {

int spca_abi_version(void) { return SPCA_ABI_VERSION; }

const char *spca_build_info(void) {
  return "libspca sm_100a: SIMT(FFMA/DFMA) + tcgen05 split-precision sketch; " __DATE__ " " __TIME__;
}

int spca_sketch_create(spca_handle_t *out, int64_t n, int64_t l, int dtype, int precision,
                       const double *omega, int omega_where, int device, void *stream,
                       int64_t rows_hint, int compensated) {
  if (!out) return set_err(nullptr, SPCA_ERR_CONFIG, -1, "null handle pointer");
  *out = nullptr;
  if (n < 1 || l < 1) return set_err(nullptr, SPCA_ERR_FORMAT, -1, "omega must be 2-d and non-empty (n=%lld, l=%lld)", (long long)n, (long long)l);
  // any sketch width the reference accepts (l <= min(m, n), algorithms.py:89-101);
  // the bound only keeps l_pad * rows and the launch grids inside int range
  if (l > (1 << 16)) return set_err(nullptr, SPCA_ERR_CONFIG, -1, "sketch width l=%lld > 65536 unsupported", (long long)l);
  if (n > INT32_MAX / 2) return set_err(nullptr, SPCA_ERR_CONFIG, -1, "n too large");
  if (dtype != SPCA_F32 && dtype != SPCA_F64) return set_err(nullptr, SPCA_ERR_CONFIG, -1, "bad dtype %d", dtype);
  if (!omega) return set_err(nullptr, SPCA_ERR_FORMAT, -1, "omega is null");
  if (precision == SPCA_PREC_AUTO)
    precision = (dtype == SPCA_F32 && tc_supported_shape(n, l) && tc_available(device)) ? SPCA_PREC_TC
                                                                                       : SPCA_PREC_SIMT;
  if (precision == SPCA_PREC_TC && dtype != SPCA_F32)
    return set_err(nullptr, SPCA_ERR_CONFIG, -1, "tensor-core path is f32 only (fp64 uses DFMA)");
  if (precision == SPCA_PREC_TC && !tc_supported_shape(n, l))
    return set_err(nullptr, SPCA_ERR_CONFIG, -1, "tensor-core path does not support n=%lld l=%lld", (long long)n, (long long)l);

  spca_sketch *h = new (std::nothrow) spca_sketch();
  if (!h) return set_err(nullptr, SPCA_ERR_OOM, -1, "out of host memory");
  h->device = device;
  DeviceGuard dg(device);
  h->dtype = dtype;
  h->precision = precision;
  h->ds = dtype == SPCA_F32 ? 4 : 8;
  h->n = n;
  h->l = l;
  h->bl = l <= 32 ? 32 : 64;
  h->lpad = round_up(l, h->bl);
  h->compensated = compensated != 0;
  auto fail = [&](int rc) {
    spca_sketch_destroy(h);
    g_tl_code = rc;
    return rc;
  };
  if (stream) {
    h->stream = (cudaStream_t)stream;
  } else {
    if (cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking) != cudaSuccess)
      return fail(set_err(nullptr, SPCA_ERR_CUDA, -1, "stream create failed"));
    h->own_stream = true;
  }
  // canonical chunk (SIMT path): ~320 MB of A, 128..4096 rows, multiple of 128
  {
    int64_t r = (int64_t)((int64_t)kSimtChunkMB << 20) / (n * (int64_t)h->ds);
    r = std::max<int64_t>(128, std::min<int64_t>(4096, r));
    h->chunk_rows = (r / 128) * 128;
    if (h->precision == SPCA_PREC_TC) h->chunk_rows = tc_chunk_rows(n, l);
  }
  h->stage_rows = h->chunk_rows;
  if (h->precision == SPCA_PREC_TC)  // host staging in ~512 MB pieces: many chunks per launch
    h->stage_rows = h->chunk_rows * std::max<int64_t>(1, (512ll << 20) / (h->chunk_rows * n * 4));
  // row splits of the H kernel: enough CTAs with the n tiles
  {
    int bn = h->bl == 32 ? 128 : 64;
    int64_t tiles = ceil_div(n, bn) * (h->lpad / h->bl);
    int64_t want = ceil_div(148 * kSimtHTarget, tiles);
    h->hsplit = (int)std::max<int64_t>(1, std::min<int64_t>(8, want));
    if (h->precision == SPCA_PREC_TC) h->hsplit = 1;  // the pass kernel keeps one running H
  }
  // flush the fp32 H partials into fp64 every ~1M rows
  h->flush_every = (int)std::max<int64_t>(1, (1 << 20) / h->chunk_rows);
  if (const char *d = getenv("SPCA_TC_DEBUG")) h->tc_debug = atoi(d);
  if (const char *d = getenv("SPCA_TC_COOP")) h->tc_coop = atoi(d);

  const size_t ds = h->ds;
  int rc;
#define TRY(call)                                                                      \
  do {                                                                                 \
    cudaError_t _e = (call);                                                           \
    if (_e != cudaSuccess)                                                             \
      return fail(set_err(nullptr, _e == cudaErrorMemoryAllocation ? SPCA_ERR_OOM : SPCA_ERR_CUDA, -1, \
                          "%s: %s", #call, cudaGetErrorString(_e)));                   \
  } while (0)
  ensure_pool(device);
  TRY(dalloc(h, &h->omega_dev, (size_t)n * h->lpad * ds));
  TRY(dalloc(h, &h->omega64_dev, (size_t)n * l * 8));
  TRY(dalloc(h, &h->hcs_dev, (size_t)n * (l + 1) * 8));
  TRY(cudaMemsetAsync(h->hcs_dev, 0, (size_t)n * (l + 1) * 8, h->stream));
  if (h->compensated) {
    TRY(dalloc(h, &h->carry_dev, (size_t)n * 8));
    TRY(cudaMemsetAsync(h->carry_dev, 0, (size_t)n * 8, h->stream));
  }
  TRY(dalloc(h, &h->hpart, (size_t)h->hsplit * n * h->lpad * ds));
  TRY(cudaMemsetAsync(h->hpart, 0, (size_t)h->hsplit * n * h->lpad * ds, h->stream));
  TRY(dalloc(h, &h->cspart, (size_t)h->hsplit * n * 8));
  TRY(cudaMemsetAsync(h->cspart, 0, (size_t)h->hsplit * n * 8, h->stream));
  TRY(dalloc(h, &h->bad_dev, 2 * sizeof(unsigned long long)));
  {
    unsigned long long init[2] = {(unsigned long long)kNoBadRow, (unsigned long long)kNoBadRow};
    TRY(cudaMemcpyAsync(h->bad_dev, init, sizeof init, cudaMemcpyHostToDevice, h->stream));
    TRY(cudaStreamSynchronize(h->stream));
  }
  h->ldp = h->precision == SPCA_PREC_TC ? round_up(n, 4) : n;
  TRY(dalloc(h, &h->tail, (size_t)h->chunk_rows * h->ldp * ds));
  // Omega: upload fp64, derive the compute-precision copy
  {
    double *om_src = nullptr;
    if (omega_where == SPCA_MEM_DEVICE) {
      om_src = const_cast<double *>(omega);
    } else {
      TRY(dalloc(h, &om_src, (size_t)n * l * 8));
      cudaError_t ue = omega_where == SPCA_MEM_PAGEABLE
                           ? upload_pageable(om_src, omega, (size_t)n * l * 8, h->stream)
                           : cudaMemcpyAsync(om_src, omega, (size_t)n * l * 8, cudaMemcpyHostToDevice, h->stream);
      if (ue != cudaSuccess) {
        dfree(h, om_src);  // not yet owned by the handle: fail() would not release it
        TRY(ue);
      }
    }
    if (dtype == SPCA_F32)
      omega_prepare<float><<<grid_for(n * h->lpad), 256, 0, h->stream>>>(
          om_src, (int)n, (int)l, (int)h->lpad, (float *)h->omega_dev, h->omega64_dev);
    else
      omega_prepare<double><<<grid_for(n * h->lpad), 256, 0, h->stream>>>(
          om_src, (int)n, (int)l, (int)h->lpad, (double *)h->omega_dev, h->omega64_dev);
    cudaError_t le = cudaGetLastError();
    if (le != cudaSuccess) return fail(set_err(nullptr, SPCA_ERR_CUDA, -1, "omega_prepare: %s", cudaGetErrorString(le)));
    h->launches++;
    if (omega_where != SPCA_MEM_DEVICE) dfree(h, om_src);  // stream-ordered after omega_prepare
  }
  if (h->precision == SPCA_PREC_TC) {
    rc = tc_setup(h);
    if (rc) return fail(rc);
  }
  if (rows_hint > 0) {
    rc = ensure_g(h, rows_hint);
    if (rc) return fail(rc);
  }
#undef TRY
  *out = h;
  return SPCA_OK;
}

}  // extern "C"

namespace {
int push_impl(spca_handle_t h, const void *a, int64_t rows, int64_t ld, int64_t first_row, int where,
              bool final) {
  if (!h) return set_err(nullptr, SPCA_ERR_STATE, -1, "null handle");
  if (h->finished) return set_err(h, SPCA_ERR_STATE, -1, "push after finish");
  if (h->final_pushed) return set_err(h, SPCA_ERR_STATE, -1, "push after the final push");
  if (rows < 0) return set_err(h, SPCA_ERR_FORMAT, first_row, "negative row count");
  if (first_row != h->rows_seen)
    return set_err(h, SPCA_ERR_FORMAT, first_row,
                   "block starts at row %lld but %lld rows were consumed (blocks must be consecutive)",
                   (long long)first_row, (long long)h->rows_seen);
  if (rows == 0 && !final) return SPCA_OK;
  if (rows > 0 && !a) return set_err(h, SPCA_ERR_FORMAT, first_row, "null block pointer");
  if (rows > 0 && ld < h->n)
    return set_err(h, SPCA_ERR_FORMAT, first_row, "block at row %lld has row stride %lld < n=%lld",
                   (long long)first_row, (long long)ld, (long long)h->n);
  if (h->left_rows && h->rows_seen + rows > h->left_rows)
    return set_err(h, SPCA_ERR_CAPABILITY, first_row,
                   "stream yielded more rows than the co-sketch operand has (%lld)", (long long)h->left_rows);
  DeviceGuard dg(h->device);
  int rc = SPCA_OK;
  if (h->shift_on && !h->shift_set && rows > 0) {  // c = the mean of the pass's first rows
    // a sample of up to 256 rows: the sketch then holds deviations of size
    // ~ spread * sqrt(n / sample) around the mean instead of the mean itself
    const int pad = (int)round_up(h->n, 256);
    const int sr = (int)std::min<int64_t>(rows, 256);
    const void *src = a;
    int64_t sld = ld;
    void *tmp = nullptr;
    if (where != SPCA_MEM_DEVICE) {
      CK(h, dalloc(h, &tmp, (size_t)sr * h->n * h->ds));
      CK(h, cudaMemcpy2DAsync(tmp, (size_t)h->n * h->ds, a, (size_t)ld * h->ds, (size_t)h->n * h->ds, (size_t)sr,
                              cudaMemcpyHostToDevice, h->stream));
      src = tmp;
      sld = h->n;
    }
    if (h->dtype == SPCA_F32)
      shift_capture<float><<<(unsigned)ceil_div(pad, 256), 256, 0, h->stream>>>((const float *)src, sr, sld,
                                                                                (int)h->n, pad, h->cshift);
    else
      shift_capture<double><<<(unsigned)ceil_div(pad, 256), 256, 0, h->stream>>>((const double *)src, sr, sld,
                                                                                 (int)h->n, pad, h->cshift);
    CK_LAUNCH(h);
    dfree(h, tmp);
    h->shift_set = true;
  }
  if (rows == 0) {
    // final push of nothing: still flush the staged tail now
  } else if (where == SPCA_MEM_DEVICE) {
    rc = push_device_rows(h, (const char *)a, rows, ld, final);
  } else if (where == SPCA_MEM_PINNED) {
    rc = push_host_rows(h, (const char *)a, rows, ld, false, final);
  } else if (where == SPCA_MEM_PAGEABLE) {
    rc = push_host_rows(h, (const char *)a, rows, ld, true, final);
  } else {
    return set_err(h, SPCA_ERR_CONFIG, -1, "bad memory kind %d", where);
  }
  if (rc) return rc;
  if (final && h->tail_rows > 0) {  // rows == 0, or a tail left by earlier pushes
    rc = h->precision == SPCA_PREC_TC ? process_rows_tc(h, (const char *)h->tail, h->ldp, h->tail_rows)
                                      : process_chunk(h, h->tail, h->ldp, h->tail_rows);
    if (rc) return rc;
    h->tail_rows = 0;
  }
  h->rows_seen += rows;
  if (final) h->final_pushed = true;
  return SPCA_OK;
}
}  // namespace

extern "C" {

int spca_sketch_push(spca_handle_t h, const void *a, int64_t rows, int64_t ld, int64_t first_row,
                     int where) {
  return push_impl(h, a, rows, ld, first_row, where, false);
}

int spca_sketch_push_final(spca_handle_t h, const void *a, int64_t rows, int64_t ld, int64_t first_row,
                           int where) {
  return push_impl(h, a, rows, ld, first_row, where, true);
}

int spca_sketch_set_normalize(spca_handle_t h, int on) {
  if (!h) return set_err(nullptr, SPCA_ERR_STATE, -1, "null handle");
  if (h->rows_seen > 0 || h->tail_rows > 0 || h->rows_done > 0)
    return set_err(h, SPCA_ERR_STATE, -1, "set_normalize must precede the first push of a pass");
  if (on && h->shift_on)
    return set_err(h, SPCA_ERR_CONFIG, -1, "the column shift and row normalisation are exclusive");
  h->normalize = on != 0;
  return SPCA_OK;
}

int spca_sketch_set_shift(spca_handle_t h, int on) {
  if (!h) return set_err(nullptr, SPCA_ERR_STATE, -1, "null handle");
  if (h->rows_seen > 0 || h->tail_rows > 0 || h->rows_done > 0)
    return set_err(h, SPCA_ERR_STATE, -1, "set_shift must precede the first push of a pass");
  if (on && h->normalize)
    return set_err(h, SPCA_ERR_CONFIG, -1, "the column shift and row normalisation are exclusive");
  if (on && !h->cshift) {
    DeviceGuard dg(h->device);
    CK(h, dalloc(h, &h->cshift, (size_t)round_up(h->n, 256) * sizeof(float)));
    CK(h, cudaMemsetAsync(h->cshift, 0, (size_t)round_up(h->n, 256) * sizeof(float), h->stream));
  }
  h->shift_on = on != 0;
  h->shift_set = false;
  return SPCA_OK;
}

int spca_sketch_set_left(spca_handle_t h, const double *left, int64_t rows, int where) {
  if (!h) return set_err(nullptr, SPCA_ERR_STATE, -1, "null handle");
  if (h->rows_seen > 0 || h->tail_rows > 0 || h->rows_done > 0)
    return set_err(h, SPCA_ERR_STATE, -1, "set_left must precede the first push of a pass");
  if (rows < 0 || (rows > 0 && !left)) return set_err(h, SPCA_ERR_FORMAT, -1, "bad left operand (%lld rows)", (long long)rows);
  if (rows > INT32_MAX / 2) return set_err(h, SPCA_ERR_CONFIG, -1, "left operand too tall");
  DeviceGuard dg(h->device);
  if (rows > h->left_rows || rows == 0) {
    dfree(h, h->left_dev);
    dfree(h, h->left64_dev);
    h->left_dev = nullptr;
    h->left64_dev = nullptr;
  }
  h->left_rows = 0;
  if (rows == 0) return SPCA_OK;
  if (!h->left_dev) {
    CK(h, dalloc(h, &h->left_dev, (size_t)rows * h->lpad * h->ds));
    CK(h, dalloc(h, &h->left64_dev, (size_t)rows * h->l * 8));
  }
  const double *src = left;
  double *tmp = nullptr;
  if (where != SPCA_MEM_DEVICE) {
    CK(h, dalloc(h, &tmp, (size_t)rows * h->l * 8));
    cudaError_t ue = where == SPCA_MEM_PAGEABLE
                         ? upload_pageable(tmp, left, (size_t)rows * h->l * 8, h->stream)
                         : cudaMemcpyAsync(tmp, left, (size_t)rows * h->l * 8, cudaMemcpyHostToDevice, h->stream);
    if (ue != cudaSuccess) {
      cudaStreamSynchronize(h->stream);
      dfree(h, tmp);
      CK(h, ue);
    }
    src = tmp;
  }
  // same conversion as Omega: compute-precision copy (rows x lpad) + the fp64 values used
  if (h->dtype == SPCA_F32)
    omega_prepare<float><<<grid_for(rows * h->lpad), 256, 0, h->stream>>>(
        src, (int)rows, (int)h->l, (int)h->lpad, (float *)h->left_dev, h->left64_dev);
  else
    omega_prepare<double><<<grid_for(rows * h->lpad), 256, 0, h->stream>>>(
        src, (int)rows, (int)h->l, (int)h->lpad, (double *)h->left_dev, h->left64_dev);
  CK_LAUNCH(h);
  dfree(h, tmp);
  // a pageable source must not be released before the copy has read it
  if (where != SPCA_MEM_DEVICE) CK(h, cudaStreamSynchronize(h->stream));
  h->left_rows = rows;
  return SPCA_OK;
}

int spca_sketch_reset(spca_handle_t h) {
  if (!h) return set_err(nullptr, SPCA_ERR_STATE, -1, "null handle");
  DeviceGuard dg(h->device);
  // after finish the stream has drained (finish ends with its one
  // synchronization): the reset is then fully asynchronous; an abandoned pass
  // is drained first so its sources may be released by the caller
  const bool drained = h->finished || (h->rows_seen == 0 && h->tail_rows == 0);
  if (!drained) CK(h, cudaStreamSynchronize(h->stream));
  CK(h, cudaMemsetAsync(h->hcs_dev, 0, (size_t)h->n * (h->l + 1) * 8, h->stream));
  if (h->carry_dev) CK(h, cudaMemsetAsync(h->carry_dev, 0, (size_t)h->n * 8, h->stream));
  // bad_dev[1] holds the "no bad row" sentinel (set at create): a device copy, no host staging
  CK(h, cudaMemcpyAsync(h->bad_dev, h->bad_dev + 1, sizeof(unsigned long long), cudaMemcpyDeviceToDevice,
                        h->stream));
  h->tail_rows = 0;
  h->rows_seen = 0;
  h->rows_done = 0;
  h->chunks_since_flush = 0;
  h->shift_set = false;
  h->finished = false;
  h->final_pushed = false;
  h->last_code = SPCA_OK;
  h->last_bad_row = -1;
  h->last_msg[0] = 0;
  return SPCA_OK;
}

int spca_sketch_sync(spca_handle_t h) {
  if (!h) return set_err(nullptr, SPCA_ERR_STATE, -1, "null handle");
  DeviceGuard dg(h->device);
  CK(h, cudaStreamSynchronize(h->stream));
  int rc = collect_timers(h);
  if (rc) return rc;
  return check_bad_row(h);
}

int spca_sketch_rows(spca_handle_t h, int64_t *rows_seen) {
  if (!h || !rows_seen) return set_err(h, SPCA_ERR_STATE, -1, "null argument");
  *rows_seen = h->rows_seen;
  return SPCA_OK;
}

int64_t spca_sketch_chunk_rows(spca_handle_t h) { return h ? h->chunk_rows : -1; }

int spca_sketch_precision(spca_handle_t h) { return h ? h->precision : -1; }

int spca_sketch_finish(spca_handle_t h, double *g_out, double *h_out, double *colsum_out,
                       int64_t *rows_seen, int out_where) {
  if (!h) return set_err(nullptr, SPCA_ERR_STATE, -1, "null handle");
  DeviceGuard dg(h->device);
  int rc;
  if (!h->finished) {
    if (h->tail_rows > 0) {
      rc = h->precision == SPCA_PREC_TC ? process_rows_tc(h, (const char *)h->tail, h->ldp, h->tail_rows)
                                        : process_chunk(h, h->tail, h->ldp, h->tail_rows);
      if (rc) return rc;
      h->tail_rows = 0;
    }
    rc = flush_h(h);
    if (rc) return rc;
    if (h->rows_seen > h->g64_cap) {
      dfree(h, h->g64_dev);
      h->g64_dev = nullptr;
      CK(h, dalloc(h, &h->g64_dev, (size_t)std::max<int64_t>(1, h->rows_seen) * h->l * 8));
      h->g64_cap = h->rows_seen;
    }
    if (h->rows_seen > 0) {
      int64_t count = h->rows_seen * h->l;
      if (h->dtype == SPCA_F32)
        g_widen<float><<<grid_for(count), 256, 0, h->stream>>>((const float *)h->g_dev, (int)h->lpad,
                                                               h->rows_seen, (int)h->l, h->g64_dev);
      else
        g_widen<double><<<grid_for(count), 256, 0, h->stream>>>((const double *)h->g_dev, (int)h->lpad,
                                                                h->rows_seen, (int)h->l, h->g64_dev);
      CK_LAUNCH(h);
    }
    if (h->shift_on && h->shift_set && h->rows_seen > 0) {
      // undo the column shift in fp64 (epilogue.cuh shift_fix_h): G, H, col_sums of A itself
      double *wg = nullptr;
      CK(h, dalloc(h, &wg, (size_t)2 * h->l * 8));
      const bool co = h->left_rows > 0;
      shift_terms<<<(unsigned)h->l, 256, 0, h->stream>>>(h->cshift, h->omega64_dev, (int)h->n, (int)h->l,
                                                          co ? h->left64_dev : h->g64_dev, h->rows_seen, wg,
                                                          wg + h->l);
      CK_LAUNCH(h);
      shift_fix_h<<<grid_for(h->n * h->l), 256, 0, h->stream>>>(h->hcs_dev, (int)h->n, (int)h->l, h->cshift, wg,
                                                                 wg + h->l, h->rows_seen, co ? 1 : 0);
      CK_LAUNCH(h);
      shift_fix_colsum<<<(unsigned)ceil_div(h->n, 256), 256, 0, h->stream>>>(h->hcs_dev + h->n * h->l, (int)h->n,
                                                                             h->cshift, h->rows_seen);
      CK_LAUNCH(h);
      g_add_row<<<grid_for(h->rows_seen * h->l), 256, 0, h->stream>>>(h->g64_dev, h->rows_seen, (int)h->l, wg);
      CK_LAUNCH(h);
      dfree(h, wg);
    }
    if (h->normalize && h->precision == SPCA_PREC_TC && h->rows_seen > 0) {
      // fused normalisation: H -= 1 (G_hat^T coef)^T, colsum -= sum(coef) (sketch_fused.cuh)
      double *c = nullptr;
      CK(h, dalloc(h, &c, (size_t)(h->l + 1) * 8));
      norm_coef_sums<<<(unsigned)(h->l + 1), 256, 0, h->stream>>>(h->left_rows ? h->left64_dev : h->g64_dev,
                                                                   h->rows_seen, (int)h->l, h->row_coef, c);
      CK_LAUNCH(h);
      norm_correct<<<grid_for(h->n * (h->l + 1)), 256, 0, h->stream>>>(h->hcs_dev, (int)h->n, (int)h->l, c);
      CK_LAUNCH(h);
      dfree(h, c);
    }
  }
  const bool first_finish = !h->finished;
  cudaMemcpyKind kind = out_where == SPCA_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  if (g_out && h->rows_seen > 0)
    CK(h, cudaMemcpyAsync(g_out, h->g64_dev, (size_t)h->rows_seen * h->l * 8, kind, h->stream));
  if (h_out) CK(h, cudaMemcpyAsync(h_out, h->hcs_dev, (size_t)h->n * h->l * 8, kind, h->stream));
  if (colsum_out)
    CK(h, cudaMemcpyAsync(colsum_out, h->hcs_dev + h->n * h->l, (size_t)h->n * 8, kind, h->stream));
  if (rows_seen) *rows_seen = h->rows_seen;
  // the first non-finite row comes back behind the outputs: a copy into
  // pageable memory returns once the stream has drained (the one synchronization)
  if (first_finish) {
    CK(h, cudaMemcpyAsync(&h->bad_seen, h->bad_dev, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                          h->stream));
  }
  CK(h, cudaStreamSynchronize(h->stream));
  if (first_finish) {
    rc = collect_timers(h);
    if (rc) return rc;
    if (h->bad_seen != (unsigned long long)kNoBadRow)
      return set_err(h, SPCA_ERR_DATA, (int64_t)h->bad_seen, "non-finite value in row %lld",
                     (long long)h->bad_seen);
    h->finished = true;
  }
  return SPCA_OK;
}

int spca_device_views(spca_handle_t h, double **g_dev, double **hcs_dev) {
  if (!h) return set_err(nullptr, SPCA_ERR_STATE, -1, "null handle");
  if (!h->finished) return set_err(h, SPCA_ERR_STATE, -1, "device views need a finished sketch");
  if (g_dev) *g_dev = h->g64_dev;
  if (hcs_dev) *hcs_dev = h->hcs_dev;
  return SPCA_OK;
}

// NCCL entry points, resolved from the process's libnccl.so.2 at first use
// (the one the caller's communicator came from when it is already loaded).
struct NcclFns {
  ncclResult_t (*all_reduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  const char *(*error_string)(ncclResult_t) = nullptr;
};

static const NcclFns *nccl_fns() {
  static NcclFns f;
  static bool tried = false;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (!tried) {
    tried = true;
    void *lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW);
    if (lib) {
      f.all_reduce = (decltype(f.all_reduce))dlsym(lib, "ncclAllReduce");
      f.group_start = (decltype(f.group_start))dlsym(lib, "ncclGroupStart");
      f.group_end = (decltype(f.group_end))dlsym(lib, "ncclGroupEnd");
      f.error_string = (decltype(f.error_string))dlsym(lib, "ncclGetErrorString");
    }
  }
  return (f.all_reduce && f.group_start && f.group_end) ? &f : nullptr;
}

int spca_allreduce(spca_handle_t h, void *nccl_comm, int64_t *rows_total) {
  if (!h || !nccl_comm) return set_err(h, SPCA_ERR_STATE, -1, "null argument");
  if (!h->finished) return set_err(h, SPCA_ERR_STATE, -1, "allreduce needs a finished sketch");
  const NcclFns *nf = nccl_fns();
  if (!nf) return set_err(h, SPCA_ERR_CAPABILITY, -1, "libnccl.so.2 not found");
  DeviceGuard dg(h->device);
  double *rows = nullptr;
  CK(h, dalloc(h, &rows, sizeof(double)));
  const double local = (double)h->rows_seen;
  CK(h, cudaMemcpyAsync(rows, &local, sizeof local, cudaMemcpyHostToDevice, h->stream));
  ncclComm_t comm = (ncclComm_t)nccl_comm;
  ncclResult_t r = nf->group_start();
  if (r == ncclSuccess)
    r = nf->all_reduce(h->hcs_dev, h->hcs_dev, (size_t)h->n * (h->l + 1), ncclFloat64, ncclSum, comm, h->stream);
  if (r == ncclSuccess) r = nf->all_reduce(rows, rows, 1, ncclFloat64, ncclSum, comm, h->stream);
  const ncclResult_t r2 = nf->group_end();
  if (r == ncclSuccess) r = r2;
  if (r != ncclSuccess) {
    dfree(h, rows);
    return set_err(h, SPCA_ERR_CUDA, -1, "NCCL all-reduce failed: %s",
                   nf->error_string ? nf->error_string(r) : "unknown");
  }
  double total = 0.0;
  CK(h, cudaMemcpyAsync(&total, rows, sizeof total, cudaMemcpyDeviceToHost, h->stream));
  dfree(h, rows);
  CK(h, cudaStreamSynchronize(h->stream));
  if (rows_total) *rows_total = (int64_t)(total + 0.5);
  return SPCA_OK;
}

int spca_omega_used(spca_handle_t h, double *out, int out_where) {
  if (!h || !out) return set_err(h, SPCA_ERR_STATE, -1, "null argument");
  DeviceGuard dg(h->device);
  CK(h, cudaMemcpyAsync(out, h->omega64_dev, (size_t)h->n * h->l * 8,
                        out_where == SPCA_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                        h->stream));
  CK(h, cudaStreamSynchronize(h->stream));
  return SPCA_OK;
}

int spca_g_colsum(spca_handle_t h, double *out, int out_where) {
  if (!h || !out) return set_err(h, SPCA_ERR_STATE, -1, "null argument");
  if (!h->finished) return set_err(h, SPCA_ERR_STATE, -1, "g_colsum needs a finished sketch");
  DeviceGuard dg(h->device);
  double *d = nullptr;
  CK(h, dalloc(h, &d, (size_t)h->l * 8));
  column_sums64<<<(unsigned)h->l, 256, 0, h->stream>>>(h->g64_dev, h->rows_seen, (int)h->l, d);
  CK_LAUNCH(h);
  CK(h, cudaMemcpyAsync(out, d, (size_t)h->l * 8,
                        out_where == SPCA_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                        h->stream));
  dfree(h, d);
  CK(h, cudaStreamSynchronize(h->stream));
  return SPCA_OK;
}

int spca_normalize_rows(const void *src, int64_t rows, int64_t n, int64_t ld_src, void *dst, int64_t ld_dst,
                        int dtype, void *stream) {
  if (rows < 0 || n < 1 || ld_src < n || ld_dst < n)
    return set_err(nullptr, SPCA_ERR_CONFIG, -1, "normalize_rows: bad shape %lld x %lld (ld %lld, %lld)",
                   (long long)rows, (long long)n, (long long)ld_src, (long long)ld_dst);
  if (rows == 0) return SPCA_OK;
  if (!src || !dst) return set_err(nullptr, SPCA_ERR_STATE, -1, "normalize_rows: null pointer");
  if (dtype != SPCA_F32 && dtype != SPCA_F64)
    return set_err(nullptr, SPCA_ERR_CONFIG, -1, "normalize_rows: bad dtype %d", dtype);
  const cudaError_t e = launch_normalize(src, rows, n, ld_src, dst, ld_dst, dtype, (cudaStream_t)stream);
  if (e != cudaSuccess) return set_err(nullptr, SPCA_ERR_CUDA, -1, "normalize_rows launch: %s", cudaGetErrorString(e));
  return SPCA_OK;
}

// ---------------------------------------------------------------- post-pass
namespace {
// the sweep kernel instantiated for an even block width 2..16 and one of
// the five sweep kinds of spca_qb_block
extern "C++" {  // templates inside the extern "C" block
template <int B>
const void *qb_kernel_b(int kind) {
  using namespace spca;
  switch (kind) {
    case kQbX | kQbP | kQbW | kQbOut: return (const void *)qb_sweep_kernel<B, kQbX | kQbP | kQbW | kQbOut>;
    case kQbW: return (const void *)qb_sweep_kernel<B, kQbW>;
    case kQbP: return (const void *)qb_sweep_kernel<B, kQbP>;
    case kQbX | kQbW | kQbOut: return (const void *)qb_sweep_kernel<B, kQbX | kQbW | kQbOut>;
    case kQbW | kQbOut: return (const void *)qb_sweep_kernel<B, kQbW | kQbOut>;
    default: return (const void *)qb_sweep_kernel<B, kQbOut>;
  }
}
const void *qb_kernel(int b, int kind) {
  switch (b) {
    case 2: return qb_kernel_b<2>(kind);
    case 4: return qb_kernel_b<4>(kind);
    case 6: return qb_kernel_b<6>(kind);
    case 8: return qb_kernel_b<8>(kind);
    case 10: return qb_kernel_b<10>(kind);
    case 12: return qb_kernel_b<12>(kind);
    case 14: return qb_kernel_b<14>(kind);
    default: return qb_kernel_b<16>(kind);
  }
}
}  // extern "C++"
// rows per tile and ring depth: the largest tile (up to 256 rows) whose
// three-stage ring fits two CTAs per SM (110 KB each), else one CTA per SM
// (up to 220 KB), else 16 rows and two stages. SPCA_QB_TR / SPCA_QB_ST
// override (tuning).
void qb_tiling(int c0, int b, int nslab, int *tr, int *stages) {
  static const int env_tr = getenv("SPCA_QB_TR") ? atoi(getenv("SPCA_QB_TR")) : 0;
  static const int env_st = getenv("SPCA_QB_ST") ? atoi(getenv("SPCA_QB_ST")) : 0;
  if (env_tr >= 16 && env_tr % 16 == 0 && env_tr <= 256 && (env_st == 2 || env_st == 3) &&
      spca::qb_sweep_smem(c0, b, env_tr, nslab, env_st) <= (220u << 10)) {
    *tr = env_tr;
    *stages = env_st;
    return;
  }
  for (size_t cap : {(size_t)110 << 10, (size_t)220 << 10})
    for (int t : {256, 128, 64, 32, 16})
      for (int st : {3, 2})
        if (spca::qb_sweep_smem(c0, b, t, nslab, st) <= cap) {
          *tr = t;
          *stages = st;
          return;
        }
  *tr = 16;
  *stages = 2;
}
constexpr int kQbMaxOcc = 4;  // resident sweep CTAs per SM counted for the partials (bound)
// CTAs of one sweep: one wave of resident CTAs of that kernel and tiling
// (the kernel loops over row tiles); raises the kernels' shared-memory limit
int qb_parts(int64_t m, int c0, int b, int nslab, int kind, int tr, int stages) {
  int dev = 0, sms = 148, occ = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const void *kern = qb_kernel(b, kind);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 << 10);
  cudaGetLastError();  // a refused attribute must not surface as the next launch's error
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, spca::kQbThreads,
                                                    spca::qb_sweep_smem(c0, b, tr, nslab, stages)) != cudaSuccess)
    occ = 1;
  occ = std::max(1, std::min(kQbMaxOcc, occ));
  const int64_t tiles = (m + tr - 1) / tr;
  return (int)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)sms * occ));
}
// 2-D fp64 tensor map over rows of a row-major matrix (TMA), box {bi, bo}
bool qb_map(CUtensorMap *map, const void *ptr, uint64_t inner, uint64_t outer, uint64_t row_bytes, uint32_t bi,
            uint32_t bo, bool swz) {
  EncodeTiledFn enc = tma_encoder();
  if (!enc) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_bytes};
  cuuint32_t box[2] = {bi, bo};
  cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void *>(ptr), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace

int64_t spca_qb_workspace_elems(int64_t m, int c0_max, int b) {
  if (m < 1 || c0_max < 0 || b < 1) return 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // partials of the widest sweep (at most kQbMaxOcc CTAs per SM), the reduced sums, x
  const int64_t most = (int64_t)sms * kQbMaxOcc * b * (c0_max + b);
  return most + (int64_t)b * (c0_max + b) + (int64_t)c0_max * b + 64;
}

int spca_qb_block(int64_t m, int c0, int b, double *q, int64_t ldq, const double *g, int64_t ldg,
                  const double *x, double *ybuf, double *ws, int64_t ws_elems, double *p_out,
                  double *factors, int *flag, const double *tol, void *stream) {
  if (m < 1 || m > INT32_MAX || c0 < 0 || b < 2 || b > spca::kQbMaxB || (b & 1) || (c0 & 1) ||
      c0 + b > spca::kQbMaxCat || ldq < c0 + b || (ldq & 1) || ldg < b || (ldg & 1))
    return set_err(nullptr, SPCA_ERR_CONFIG, -1, "qb_block: unsupported shape m %lld c0 %d b %d ldq %lld",
                   (long long)m, c0, b, (long long)ldq);
  if (!q || !g || !ybuf || !ws || !p_out || !factors || !flag || !tol || (c0 > 0 && !x))
    return set_err(nullptr, SPCA_ERR_STATE, -1, "qb_block: null pointer");
  if (((uintptr_t)q | (uintptr_t)g | (uintptr_t)ybuf) & 15)
    return set_err(nullptr, SPCA_ERR_CONFIG, -1, "qb_block: operands must be 16-byte aligned");
  if (ws_elems < spca_qb_workspace_elems(m, c0, b))
    return set_err(nullptr, SPCA_ERR_CONFIG, -1, "qb_block: workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  const int ncat = c0 + b;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double *part = ws;
  double *red = part + (size_t)sms * kQbMaxOcc * b * ncat;  // b x ncat
  double *xt = red + (size_t)b * ncat;                      // c0 x b
  int parts = 1;  // of the last sweep (its reduction)
  const int bb = b * b;  // factors: see qb_small_kernel
  double *M1 = factors + 6 * bb, *M12 = factors + 7 * bb, *M3 = factors + 8 * bb, *M34 = factors + 9 * bb;
  // factors[10]: skip flags of the two second CholeskyQR passes (one-pass CholeskyQR for a
  // well-conditioned block, decided on the device by op 1 / op 3)
  double *skip1 = factors + 10 * bb, *skip2 = skip1 + 1;
  static const bool cq2_always = getenv("SPCA_QB_CQ2") != nullptr;  // A/B knob: always two passes
  const unsigned rblocks = (unsigned)ceil_div((int64_t)b * ncat, 32);
  // from_g: the sweep's y rows are G_i (tensor map, row stride ldg), else the
  // contiguous scratch ybuf (one bulk copy per tile)
  auto sweep = [&](bool from_g, const double *mt, const double *xx, double *out, int64_t ldo, int wp, int ww,
                   const double *skip = nullptr) -> cudaError_t {
    spca::QbSweepArgs a{};
    a.skip = skip;
    const bool need_q = c0 > 0 && (xx != nullptr || wp);
    const int nslab = need_q ? (c0 + 15) / 16 : 0;
    const int kind = (xx ? spca::kQbX : 0) | (wp ? spca::kQbP : 0) | (ww ? spca::kQbW : 0) | (out ? spca::kQbOut : 0);
    int tr = 16, stages = 2;
    qb_tiling(c0, b, nslab, &tr, &stages);
    parts = qb_parts(m, c0, b, nslab, kind, tr, stages);
    a.m = m;
    a.c0 = c0;
    a.b = b;
    a.tr = tr;
    a.stages = stages;
    a.nslab = nslab;
    a.mt = mt;
    a.y1d = from_g ? nullptr : ybuf;  // ybuf is m x b contiguous
    CUtensorMap tq, ty;  // boxes of tr rows (the Q map also stands in for an unused y map)
    if (!qb_map(&tq, q, (uint64_t)ldq, (uint64_t)m, (uint64_t)ldq * 8, 16, (uint32_t)tr, true))
      return cudaErrorInvalidValue;
    if (from_g) {
      if (!qb_map(&ty, g, (uint64_t)b, (uint64_t)m, (uint64_t)ldg * 8, (uint32_t)b, (uint32_t)tr, false))
        return cudaErrorInvalidValue;
    } else {
      ty = tq;
    }
    a.x = xx;
    a.out = out;
    a.ldo = ldo;
    a.part = part;
    const size_t smem = spca::qb_sweep_smem(c0, b, tr, a.nslab, stages);
    void *args[] = {(void *)&tq, (void *)&ty, (void *)&a};
    return cudaLaunchKernel(qb_kernel(b, kind), dim3(parts), dim3(spca::kQbThreads), args, smem, st);
  };
  auto reduce = [&](double *dst, double *xtrans) -> cudaError_t {
    spca::qb_reduce_kernel<<<rblocks, 256, 0, st>>>(part, parts, b, ncat, dst, xtrans, c0);
    return cudaGetLastError();
  };
  auto small = [&](int op, const double *r, double *skip_out) -> cudaError_t {
    spca::qb_small_kernel<<<1, 32, 0, st>>>(op, b, ncat, c0, r, factors, flag, tol, cq2_always ? 0 : 1, skip_out);
    return cudaGetLastError();
  };
  // reduction of the t^T t block + the b x b step; skip: the step was done by op 1 / op 3
  auto wfinish = [&](int op, const double *skip, double *skip_out) -> cudaError_t {
    spca::qb_wfinish_kernel<<<1, 256, 0, st>>>(op, b, ncat, c0, part, parts, factors, flag, tol, skip,
                                               cq2_always ? 0 : 1, skip_out);
    return cudaGetLastError();
  };
  static const bool sync_each = getenv("SPCA_QB_SYNC") != nullptr;  // debugging: fault localisation
#define QB_TRY(call)                                                                             \
  do {                                                                                           \
    cudaError_t _e = (call);                                                                     \
    if (_e == cudaSuccess && sync_each) _e = cudaStreamSynchronize(st);                          \
    if (_e != cudaSuccess)                                                                       \
      return set_err(nullptr, SPCA_ERR_CUDA, -1, "qb_block %s: %s", #call, cudaGetErrorString(_e)); \
  } while (0)
  // S1: y = G_i - Q X; [y^T Q | y^T y] (kept for the B update)
  QB_TRY(sweep(true, nullptr, c0 ? x : nullptr, ybuf, b, c0 ? 1 : 0, 1));
  QB_TRY(reduce(p_out, nullptr));
  QB_TRY(small(1, p_out, skip1));
  // S2: Q1 = y R1^-1, Q1^T Q1 (skipped on the device for a well-conditioned y)
  QB_TRY(sweep(false, M1, nullptr, nullptr, 0, 0, 1, skip1));
  QB_TRY(wfinish(2, skip1, nullptr));
  if (c0 > 0) {  // S3: Q^T Q2 (Q2 = y R1^-1 R2^-1), kept transposed as the next X
    QB_TRY(sweep(false, M12, nullptr, nullptr, 0, 1, 0));
    QB_TRY(reduce(red, xt));
  }
  // S4: z = Q2 - Q (Q^T Q2), z^T z
  QB_TRY(sweep(false, M12, c0 ? xt : nullptr, ybuf, b, 0, 1));
  QB_TRY(wfinish(3, nullptr, skip2));
  // S5: Z1 = z R3^-1, Z1^T Z1 (skipped on the device for a well-conditioned z)
  QB_TRY(sweep(false, M3, nullptr, nullptr, 0, 0, 1, skip2));
  QB_TRY(wfinish(4, skip2, nullptr));
  // S6: Q_i = z R3^-1 R4^-1 into Q's columns [c0, c0 + b)
  QB_TRY(sweep(false, M34, nullptr, q + c0, ldq, 0, 0));
#undef QB_TRY
  return SPCA_OK;
}

// --- the B side of a QB block (postpass.cuh): X = B[:c0] Omega_i and B_i
extern "C++" {
namespace {
int64_t qb_proj_chunk(int64_t n, int sms) {
  int64_t kc = (n + 2 * (int64_t)sms - 1) / (2 * sms);  // about two CTAs per SM
  kc = std::max<int64_t>(32, (kc + 31) / 32 * 32);
  return std::min<int64_t>(kc, 1536);  // shared-memory stage: kc x b doubles <= 192 KB
}
template <int B>
cudaError_t qb_proj_launch(int64_t n, int c0, const double *bm, int64_t ldb, const double *om, int64_t ldo,
                           double *x, double *ws, int sms, cudaStream_t st) {
  const int64_t kc = qb_proj_chunk(n, sms);
  const int chunks = (int)((n + kc - 1) / kc);
  const size_t smem = (size_t)kc * B * sizeof(double);
  static std::once_flag once;
  static cudaError_t ae = cudaSuccess;
  std::call_once(once, [] {
    ae = cudaFuncSetAttribute(spca::qb_omega_proj_kernel<B>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              1536 * B * (int)sizeof(double));
  });
  if (ae != cudaSuccess) return ae;
  spca::qb_omega_proj_kernel<B><<<chunks, 256, smem, st>>>(n, c0, bm, ldb, om, ldo, kc, ws);
  spca::qb_reduce_kernel<<<(unsigned)ceil_div((int64_t)c0 * B, 32), 256, 0, st>>>(ws, chunks, c0, B, x, nullptr, 0);
  return cudaGetLastError();
}
template <int B>
cudaError_t qb_brows_launch(int64_t n, int c0, const double *bm, int64_t ldb, const double *h, int64_t ldh,
                            const double *p_out, const double *x, const double *ri, double *bout, cudaStream_t st) {
  const size_t smem = ((size_t)c0 * B + B * B) * sizeof(double);
  spca::qb_b_rows_kernel<B><<<(unsigned)ceil_div(n, 256), 256, smem, st>>>(n, c0, bm, ldb, h, ldh, p_out, x, ri,
                                                                           bout);
  return cudaGetLastError();
}
}  // namespace
}  // extern "C++"

int64_t spca_qb_omega_proj_ws(int64_t n, int c0_max, int b) {
  if (n < 1 || c0_max < 0 || b < 1) return 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t kc = qb_proj_chunk(n, sms);
  return ((n + kc - 1) / kc) * (int64_t)std::max(c0_max, 1) * b;
}

int spca_qb_omega_proj(int64_t n, int c0, int b, const double *bm, int64_t ldb, const double *omega, int64_t ldo,
                       double *x, double *ws, int64_t ws_elems, void *stream) {
  if (n < 1 || c0 < 1 || b < 2 || b > spca::kQbMaxB || (b & 1) || !bm || !omega || !x || !ws)
    return set_err(nullptr, SPCA_ERR_CONFIG, -1, "qb_omega_proj: unsupported arguments (n %lld c0 %d b %d)",
                   (long long)n, c0, b);
  if (ws_elems < spca_qb_omega_proj_ws(n, c0, b))
    return set_err(nullptr, SPCA_ERR_CONFIG, -1, "qb_omega_proj: workspace too small");
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e;
  switch (b) {
    case 2: e = qb_proj_launch<2>(n, c0, bm, ldb, omega, ldo, x, ws, sms, st); break;
    case 4: e = qb_proj_launch<4>(n, c0, bm, ldb, omega, ldo, x, ws, sms, st); break;
    case 6: e = qb_proj_launch<6>(n, c0, bm, ldb, omega, ldo, x, ws, sms, st); break;
    case 8: e = qb_proj_launch<8>(n, c0, bm, ldb, omega, ldo, x, ws, sms, st); break;
    case 10: e = qb_proj_launch<10>(n, c0, bm, ldb, omega, ldo, x, ws, sms, st); break;
    case 12: e = qb_proj_launch<12>(n, c0, bm, ldb, omega, ldo, x, ws, sms, st); break;
    case 14: e = qb_proj_launch<14>(n, c0, bm, ldb, omega, ldo, x, ws, sms, st); break;
    default: e = qb_proj_launch<16>(n, c0, bm, ldb, omega, ldo, x, ws, sms, st); break;
  }
  if (e != cudaSuccess) return set_err(nullptr, SPCA_ERR_CUDA, -1, "qb_omega_proj: %s", cudaGetErrorString(e));
  return SPCA_OK;
}

int spca_qb_b_rows(int64_t n, int c0, int b, const double *bm, int64_t ldb, const double *h, int64_t ldh,
                   const double *p_out, const double *x, const double *r_i, double *b_out, void *stream) {
  if (n < 1 || c0 < 0 || c0 + b > spca::kQbMaxCat || b < 2 || b > spca::kQbMaxB || (b & 1) || !h || !p_out ||
      !r_i || !b_out || (c0 > 0 && (!bm || !x)))
    return set_err(nullptr, SPCA_ERR_CONFIG, -1, "qb_b_rows: unsupported arguments (n %lld c0 %d b %d)",
                   (long long)n, c0, b);
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e;
  switch (b) {
    case 2: e = qb_brows_launch<2>(n, c0, bm, ldb, h, ldh, p_out, x, r_i, b_out, st); break;
    case 4: e = qb_brows_launch<4>(n, c0, bm, ldb, h, ldh, p_out, x, r_i, b_out, st); break;
    case 6: e = qb_brows_launch<6>(n, c0, bm, ldb, h, ldh, p_out, x, r_i, b_out, st); break;
    case 8: e = qb_brows_launch<8>(n, c0, bm, ldb, h, ldh, p_out, x, r_i, b_out, st); break;
    case 10: e = qb_brows_launch<10>(n, c0, bm, ldb, h, ldh, p_out, x, r_i, b_out, st); break;
    case 12: e = qb_brows_launch<12>(n, c0, bm, ldb, h, ldh, p_out, x, r_i, b_out, st); break;
    case 14: e = qb_brows_launch<14>(n, c0, bm, ldb, h, ldh, p_out, x, r_i, b_out, st); break;
    default: e = qb_brows_launch<16>(n, c0, bm, ldb, h, ldh, p_out, x, r_i, b_out, st); break;
  }
  if (e != cudaSuccess) return set_err(nullptr, SPCA_ERR_CUDA, -1, "qb_b_rows: %s", cudaGetErrorString(e));
  return SPCA_OK;
}

int spca_center_correct(spca_handle_t h, int64_t m_total, const double *gsum, double *mean_out,
                        int mean_where) {
  if (!h) return set_err(nullptr, SPCA_ERR_STATE, -1, "null handle");
  if (!h->finished) return set_err(h, SPCA_ERR_STATE, -1, "center_correct needs a finished sketch");
  if (m_total <= 0) return set_err(h, SPCA_ERR_EMPTY, -1, "cannot center a sketch of zero rows");
  DeviceGuard dg(h->device);
  const int64_t n = h->n, l = h->l;
  double *mu = nullptr, *w = nullptr, *gs = nullptr;
  CK(h, dalloc(h, &mu, (size_t)n * 8));
  CK(h, dalloc(h, &w, (size_t)l * 8));
  CK(h, dalloc(h, &gs, (size_t)l * 8));
  double *colsum = h->hcs_dev + n * l;
  mean_from_colsum<<<(unsigned)ceil_div(n, 256), 256, 0, h->stream>>>(colsum, (int)n, 1.0 / (double)m_total, mu);
  CK_LAUNCH(h);
  mu_omega<<<(unsigned)l, 256, 0, h->stream>>>(mu, h->omega64_dev, (int)n, (int)l, w);
  CK_LAUNCH(h);
  if (gsum) {
    CK(h, cudaMemcpyAsync(gs, gsum, (size_t)l * 8, cudaMemcpyDefault, h->stream));
  } else {
    // 1^T of the H operand: G, or the co-sketch operand's rows that were pushed
    column_sums64<<<(unsigned)l, 256, 0, h->stream>>>(h->left_rows ? h->left64_dev : h->g64_dev,
                                                      h->rows_seen, (int)l, gs);
    CK_LAUNCH(h);
  }
  if (h->rows_seen > 0) {
    g_center<<<grid_for(h->rows_seen * l), 256, 0, h->stream>>>(h->g64_dev, h->rows_seen, (int)l, w);
    CK_LAUNCH(h);
  }
  h_center<<<grid_for(n * l), 256, 0, h->stream>>>(h->hcs_dev, (int)n, (int)l, mu, gs, colsum);
  CK_LAUNCH(h);
  if (mean_out)
    CK(h, cudaMemcpyAsync(mean_out, mu, (size_t)n * 8,
                          mean_where == SPCA_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                          h->stream));
  dfree(h, mu);
  dfree(h, w);
  dfree(h, gs);
  CK(h, cudaStreamSynchronize(h->stream));
  return SPCA_OK;
}

int spca_gaussian_device(double *out, int64_t count, uint64_t seed, uint64_t stream_id, const double *w,
                         const uint64_t *k, const double *f, double r_tail, double inv_r, void *stream) {
  using namespace spca::rng;
  if (count < 0 || (count > 0 && (!out || !w || !k || !f)))
    return set_err(nullptr, SPCA_ERR_CONFIG, -1, "gaussian_device: bad arguments");
  if (count == 0) return SPCA_OK;
  cudaStream_t st = (cudaStream_t)stream;
  Tables tab;
  memcpy(tab.w, w, sizeof(tab.w));
  memcpy(tab.k, k, sizeof(tab.k));
  memcpy(tab.f, f, sizeof(tab.f));
  tab.r_tail = r_tail;
  tab.inv_r = inv_r;
  // raw draws to cover: 1.0222 per value on average (std ~0.15 per value)
  const int64_t n_raw = (int64_t)(1.03 * (double)count) + 4096;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  ensure_pool(dev);  // the staging buffer stays in the stream-ordered pool between calls
  const int64_t want_seg = (int64_t)sms * 32;  // ~4 resident warps of 8 per SM
  int64_t L = std::max<int64_t>(1024, (n_raw + want_seg - 1) / want_seg);
  L = (L + 31) / 32 * 32;
  const int nseg = (int)((n_raw + L - 1) / L);
  const int64_t margin = 512;
  const int64_t ev_cap = count / 512 + 1024;  // tails: ~2.6e-4 per value
  struct Ctl {
    unsigned long long ev_n;
    int flags, undecided;
  };
  // staged values of the single walk (PASS 3): nseg x L doubles
  double *stage = nullptr;
  if (cudaMallocAsync((void **)&stage, (size_t)nseg * L * sizeof(double), st) != cudaSuccess)
    return set_err(nullptr, SPCA_ERR_CUDA, -1, "gaussian_device: staging allocation failed");
  char *buf = nullptr;
  const size_t seg_bytes = (size_t)nseg * 8;
  const size_t bytes = 4 * seg_bytes + sizeof(Ctl) + (size_t)ev_cap * sizeof(TailEvent) + 64;
  if (cudaMallocAsync((void **)&buf, bytes, st) != cudaSuccess) {
    cudaFreeAsync(stage, st);
    return set_err(nullptr, SPCA_ERR_CUDA, -1, "gaussian_device: allocation of %zu bytes failed", bytes);
  }
  int64_t *cnt = (int64_t *)buf, *entry = cnt + nseg, *exit_ = entry + nseg, *off = exit_ + nseg;
  Ctl *ctl = (Ctl *)(off + nseg);
  TailEvent *ev = (TailEvent *)(((uintptr_t)(ctl + 1) + 31) & ~(uintptr_t)31);
  int rc = SPCA_OK;
  Ctl hc{};
  std::vector<TailEvent> hev;
  const unsigned blocks = (unsigned)((nseg + 7) / 8);
  const uint64_t key0 = seed, key1 = stream_id;
  cudaMemsetAsync(ctl, 0, sizeof(Ctl), st);
  gauss_walk<3><<<blocks, 256, 0, st>>>(tab, key0, key1, L, margin, nseg, cnt, entry, exit_, nullptr, stage,
                                        count, ev, ev_cap, &ctl->ev_n, &ctl->undecided);
  gauss_scan<<<1, 1024, 0, st>>>(cnt, entry, exit_, nseg, count, off, &ctl->flags);
  gauss_gather<<<nseg, 256, 0, st>>>(stage, L, cnt, off, out, count);
  std::vector<int64_t> hoff;
  if (cudaGetLastError() != cudaSuccess || cudaMemcpyAsync(&hc, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st) ||
      cudaStreamSynchronize(st) != cudaSuccess) {
    cudaFreeAsync(stage, st);
    cudaFreeAsync(buf, st);
    return set_err(nullptr, SPCA_ERR_CUDA, -1, "gaussian_device: kernel failed: %s",
                   cudaGetErrorString(cudaGetLastError()));
  }
  if (hc.flags || hc.undecided || (int64_t)hc.ev_n > ev_cap) {
    rc = set_err(nullptr, SPCA_ERR_STATE, -1,
                 "gaussian_device: cannot vouch for the draw (chain %d, undecided %d, tails %llu): draw on the host",
                 hc.flags, hc.undecided, hc.ev_n);
  } else if (hc.ev_n > 0) {
    // tail values: numpy computes R + (-1/R) log1p(-u1) with libm's log1p
    hev.resize(hc.ev_n);
    std::vector<int64_t> pj(hc.ev_n);
    std::vector<double> pv(hc.ev_n);
    hoff.resize(nseg);
    if (cudaMemcpy(hev.data(), ev, hc.ev_n * sizeof(TailEvent), cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(hoff.data(), off, (size_t)nseg * 8, cudaMemcpyDeviceToHost) != cudaSuccess) {
      rc = set_err(nullptr, SPCA_ERR_CUDA, -1, "gaussian_device: event copy failed");
    } else {
      size_t np = 0;  // staged index w L + i -> value index off[w] + i (tails past count dropped)
      for (size_t i = 0; i < hev.size(); ++i) {
        const int64_t w = hev[i].j / L, jj = hoff[w] + (hev[i].j - w * L);
        if (jj >= count) continue;
        const double xx = (-inv_r) * std::log1p(-next_double(hev[i].u1));
        pj[np] = jj;
        pv[np] = hev[i].neg ? -(r_tail + xx) : r_tail + xx;
        ++np;
      }
      hev.resize(np);
      pj.resize(np);
      pv.resize(np);
      int64_t *dj = nullptr;
      if (np == 0) {
        // every tail lay past the requested count
      } else if (cudaMallocAsync((void **)&dj, hev.size() * 16, st) != cudaSuccess ||
          cudaMemcpyAsync(dj, pj.data(), hev.size() * 8, cudaMemcpyHostToDevice, st) != cudaSuccess ||
          cudaMemcpyAsync(dj + hev.size(), pv.data(), hev.size() * 8, cudaMemcpyHostToDevice, st) != cudaSuccess) {
        rc = set_err(nullptr, SPCA_ERR_CUDA, -1, "gaussian_device: patch upload failed");
      } else {
        gauss_patch<<<(unsigned)((hev.size() + 255) / 256), 256, 0, st>>>(out, dj, (const double *)(dj + hev.size()),
                                                                          (int64_t)hev.size());
        if (cudaGetLastError() != cudaSuccess) rc = set_err(nullptr, SPCA_ERR_CUDA, -1, "gaussian_device: patch failed");
      }
      if (dj) cudaFreeAsync(dj, st);
      // the host vectors must outlive the async copies
      if (cudaStreamSynchronize(st) != cudaSuccess && rc == SPCA_OK)
        rc = set_err(nullptr, SPCA_ERR_CUDA, -1, "gaussian_device: patch sync failed");
    }
  }
  cudaFreeAsync(stage, st);
  cudaFreeAsync(buf, st);
  return rc;
}

int spca_last_error(spca_handle_t h, int *code, int64_t *bad_row, char *msg, size_t msg_len) {
  if (h) {
    if (code) *code = h->last_code;
    if (bad_row) *bad_row = h->last_bad_row;
    if (msg && msg_len) snprintf(msg, msg_len, "%s", h->last_msg);
    return h->last_code;
  }
  if (code) *code = g_tl_code;
  if (bad_row) *bad_row = -1;
  if (msg && msg_len) snprintf(msg, msg_len, "%s", g_tl_msg);
  return g_tl_code;
}

int64_t spca_kernel_launches(spca_handle_t h) { return h ? h->launches : -1; }

int spca_enable_kernel_timing(spca_handle_t h, int enable) {
  if (!h) return set_err(nullptr, SPCA_ERR_STATE, -1, "null handle");
  h->timing = enable != 0;
  h->kernel_ms = 0.0;
  h->timed_chunks = 0;
  return SPCA_OK;
}

int spca_kernel_time_ms(spca_handle_t h, double *ms, int64_t *launches) {
  if (!h) return set_err(nullptr, SPCA_ERR_STATE, -1, "null handle");
  DeviceGuard dg(h->device);
  CK(h, cudaStreamSynchronize(h->stream));
  int rc = collect_timers(h);
  if (rc) return rc;
  if (ms) *ms = h->kernel_ms;
  if (launches) *launches = h->timed_chunks;
  return SPCA_OK;
}

// Profiling aid (not part of include/spca.h): copy the per-CTA timeline of
// the last pass-kernel launch (sketch_fused.cuh kTraceStride layout).
int spca_debug_trace(spca_handle_t h, int which, unsigned long long *out, int64_t count) {
  if (!h) return SPCA_ERR_STATE;
  (void)which;
  if (!h->trace) return set_err(h, SPCA_ERR_STATE, -1, "tracing off (set SPCA_TC_TRACE)");
  DeviceGuard dg(h->device);
  CK(h, cudaStreamSynchronize(h->stream));
  CK(h, cudaMemcpy(out, h->trace, (size_t)std::min<int64_t>(count, kTraceWords) * 8, cudaMemcpyDeviceToHost));
  return SPCA_OK;
}

// Profiling aid (not part of include/spca.h): copy the pass kernel's K-split
// partial slots ([kSlots][2T][S][128][lpad] fp32).
int spca_debug_gpart(spca_handle_t h, float *out, int64_t count) {
  if (!h || !h->gpart) return SPCA_ERR_STATE;
  DeviceGuard dg(h->device);
  CK(h, cudaStreamSynchronize(h->stream));
  CK(h, cudaMemcpy(out, h->gpart, (size_t)std::min<int64_t>(count, h->gpart_elems) * 4, cudaMemcpyDeviceToHost));
  return SPCA_OK;
}

void spca_sketch_destroy(spca_handle_t h) {
  if (!h) return;
  DeviceGuard dg(h->device);
  // host staging (pinned buffers, copy stream) is released after the work
  // that reads it; device buffers go back to the pool in stream order
  const bool host_side = h->copy_stream || h->pinned[0] || h->pinned[1] || h->dstage[0] || h->dstage[1];
  if (h->stream && host_side) cudaStreamSynchronize(h->stream);
  for (cudaEvent_t e : {h->t_start, h->t_stop, h->src_ready})
    if (e) cudaEventDestroy(e);
  if (h->copy_stream) {
    cudaStreamSynchronize(h->copy_stream);
    cudaStreamDestroy(h->copy_stream);
  }
  for (auto &t : h->timers) {
    cudaEventDestroy(t.start);
    cudaEventDestroy(t.stop);
  }
  if (h->stream) {
    void *pooled[] = {h->omega_dev, h->omega64_dev, h->tc_omega, h->g_dev, h->g64_dev, h->hcs_dev,
                      h->carry_dev, h->hpart, h->cspart, h->gpart, h->tc_ws, h->bad_dev, h->tail,
                      h->trace, h->tc_ctr, h->order_dev, h->norm_ws, h->rstat_part, h->row_a0,
                      h->row_inv, h->row_coef, h->wsum, h->left_dev, h->left64_dev, h->cshift};
    for (void *p : pooled) dfree(h, p);
  }
  for (void *p : {h->dstage[0], h->dstage[1]})
    if (p) cudaFree(p);
  for (int i = 0; i < 2; ++i) {
    pinned_put(h->pinned[i], (size_t)h->stage_rows * h->ldp * h->ds);
    if (h->copy_done[i]) cudaEventDestroy(h->copy_done[i]);
    if (h->comp_done[i]) cudaEventDestroy(h->comp_done[i]);
  }
  if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
  delete h;
}

}  // extern "C"
