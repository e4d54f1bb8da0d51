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
  if (cnt == 3 && dtype == AFFT_C64 && tau[0] == 0 && tau[1] == 1 && tau[2] == 2 &&
      (reinterpret_cast<uintptr_t>(xs) & 15) == 0 && step >= 2) {
    // FFAST's consecutive delays (0, 1, 2): bucket j's three samples are the adjacent
    // x[js - 2], x[js - 1], x[js] (j >= 1), read as one 16-byte pair load plus one
    // 8-byte load instead of three scattered 8-byte loads
    const float2* x2 = reinterpret_cast<const float2*>(xs);
    for (int j = tid; j < (int)b; j += nt) {
      const int64_t i0 = (int64_t)j * step;
      cd s0, s1, s2;  // x[i0], x[i0 - 1], x[i0 - 2]
      if (j == 0) {
        s0 = load_sample(xs, dtype, 0);
        s1 = load_sample(xs, dtype, n - 1);
        s2 = load_sample(xs, dtype, n - 2);
      } else if (((i0 - 2) & 1) == 0) {
        const float4 p = __ldg(reinterpret_cast<const float4*>(x2 + (i0 - 2)));
        const float2 q = __ldg(x2 + i0);
        s2 = cd{(double)p.x, (double)p.y};
        s1 = cd{(double)p.z, (double)p.w};
        s0 = cd{(double)q.x, (double)q.y};
      } else {
        const float2 q = __ldg(x2 + (i0 - 2));
        const float4 p = __ldg(reinterpret_cast<const float4*>(x2 + (i0 - 1)));
        s2 = cd{(double)q.x, (double)q.y};
        s1 = cd{(double)p.x, (double)p.y};
        s0 = cd{(double)p.z, (double)p.w};
      }
      bufA[j] = s0;
      bufA[b + j] = s1;
      bufA[2 * b + j] = s2;
    }
  } else {
    for (int e = tid; e < total; e += nt) {
      const int t = e / (int)b;
      const int64_t j = e - (int64_t)t * b;
      int64_t idx = j * step - tau[t];
      if (idx < 0) idx += n;
      bufA[e] = load_sample(xs, dtype, idx);
    }
  }
  __syncthreads();
  return smem_dft<kMaxR>(bufA, bufB, cnt, plan, tw, tid, nt);
}

}  // namespace afft
