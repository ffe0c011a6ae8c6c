// sample_general.cu — general filter/draw path (rows without a small top-k):
// placeholder that flags rows it would own; replaced by the weighted radix
// sampler.
#include "sampler.cuh"

namespace dp {

template <int MODE>
__global__ void general_placeholder_kernel(SampleArgs a) {
  const int ridx = blockIdx.x * blockDim.x + threadIdx.x;
  const int nrows = a.row_count ? *a.row_count : a.n_rows;
  if (ridx >= nrows) return;
  const int row = a.rows ? a.rows[ridx] : ridx;
  const dp_params_t p = a.params[row];
  const int64_t n = dom_n(a, MODE);
  const int32_t plen = pen_len(a, row, p);
  const int32_t k = p.top_k;
  const uint32_t kp = (uint32_t)min64(n, (int64_t)k + (MODE == kHot ? 0 : plen));
  const bool topk_row = k > 0 && (int64_t)k < n && kp <= (uint32_t)a.kcap && (uint32_t)(k + 2 * plen) <= (uint32_t)a.lcap;
  if (topk_row) return;
  a.token[row] = -1;
  a.logprob[row] = 0.0;
  a.flags[row] = DP_FLAG_DEGENERATE;
}

cudaError_t launch_general(const SampleArgs& a, int dtype, int mode, int grid_rows, cudaStream_t st) {
  (void)dtype;
  const unsigned g = (unsigned)((grid_rows + 127) / 128);
  if (mode == kFull) general_placeholder_kernel<kFull><<<g, 128, 0, st>>>(a);
  else if (mode == kHot) general_placeholder_kernel<kHot><<<g, 128, 0, st>>>(a);
  else general_placeholder_kernel<kTail><<<g, 128, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace dp
