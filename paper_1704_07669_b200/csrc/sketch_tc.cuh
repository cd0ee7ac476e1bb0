// sketch_tc.cuh — tcgen05 (5th-gen tensor core) split-precision sketch path.
// Included by spca_capi.cu after the error helpers. Stub until the kernels land.
#pragma once

namespace {

bool tc_available(int /*device*/) { return false; }
bool tc_supported_shape(int64_t /*n*/, int64_t /*l*/) { return false; }
int64_t tc_chunk_rows(int64_t /*n*/, int64_t /*l*/) { return 1024; }
int tc_hsplit(int64_t /*n*/, int64_t /*l*/) { return 1; }
int tc_setup(spca_sketch *h) {
  return set_err(h, SPCA_ERR_CONFIG, -1, "tensor-core path not built");
}
int tc_chunk(spca_sketch *h, const void *, int64_t, int) {
  return set_err(h, SPCA_ERR_CONFIG, -1, "tensor-core path not built");
}

}  // namespace
