// Gather + DFT of one block of shifts of one cycle, in shared memory (K1+K2).
//
// Reads x[(j*(n/b) - tau) mod n] for j < b and each of `cnt` shifts (taus
// already reduced into [0, n), bucketize.py:96) into bufA, then runs the
// Stockham DFT.  Returns the smem buffer holding the cnt x b unscaled spectra;
// the caller applies numpy's 1/b (a multiply by the reciprocal).
#pragma once

#include "smem_dft.cuh"

namespace afft {

template <int kMaxR = 8>
__device__ inline cd* gather_dft_block(const char* xs, int dtype, int64_t n, int64_t b,
                                       const DftPlan& plan, const int64_t* tau, int cnt, cd* tw,
                                       cd* bufA, cd* bufB) {
  const int tid = threadIdx.x, nt = blockDim.x;
  build_twiddles(tw, (int)b, tid, nt);
  const int64_t step = n / b;
  const int total = cnt * (int)b;
  for (int e = tid; e < total; e += nt) {
    const int t = e / (int)b;
    const int64_t j = e - (int64_t)t * b;
    int64_t idx = j * step - tau[t];
    if (idx < 0) idx += n;
    bufA[e] = load_sample(xs, dtype, idx);
  }
  __syncthreads();
  return smem_dft<kMaxR>(bufA, bufB, cnt, plan, tw, tid, nt);
}

}  // namespace afft
