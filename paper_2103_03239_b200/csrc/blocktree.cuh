// blocktree.cuh -- the reference pairwise tree (core.hpp:72-81) evaluated by a
// whole CTA; bit-identical to pairwise_rt (pairwise.cuh).
#pragma once
#include <cstdint>

namespace mb200 {

// The same tree evaluated by a whole CTA (bit-identical: identical leaves,
// identical joins).  Node (k, i) at depth k covers the range reached by the
// bits of i from the most significant (0 = left half floor(len/2), 1 = right
// half); a node of <= 8 elements is a leaf (sequential from +0), a larger one
// is left + right.  Depth K is the first at which every node has <= 8
// elements; levels are evaluated K -> 0 with one barrier each, children in
// `lvl[(k+1)&1]`.  Nodes below a leaf are evaluated too and never read.
// `lvl` is shared scratch of 2 * kBlockTreeMaxNodes doubles.  n <= 8192.
constexpr int kBlockTreeMaxNodes = 1024;

__device__ __forceinline__ void tree_node_range(std::uint32_t n, int k, std::uint32_t i,
                                                std::uint32_t& lo, std::uint32_t& len) {
  lo = 0;
  len = n;
  for (int b = k - 1; b >= 0; --b) {
    const std::uint32_t h = len / 2;
    if ((i >> b) & 1u) {
      lo += h;
      len -= h;
    } else {
      len = h;
    }
  }
}

template <class Load>
__device__ double pairwise_block(Load& ld, std::uint32_t n, double* lvl) {
  int K = 0;
  while (((n + (1u << K) - 1) >> K) > 8) ++K;  // ceil(n / 2^K) <= 8
  for (int k = K; k >= 0; --k) {
    double* cur = lvl + (k & 1) * kBlockTreeMaxNodes;
    const double* kid = lvl + ((k + 1) & 1) * kBlockTreeMaxNodes;
    for (std::uint32_t i = threadIdx.x; i < (1u << k); i += blockDim.x) {
      std::uint32_t lo, len;
      tree_node_range(n, k, i, lo, len);
      double s;
      if (len <= 8) {
        s = 0.0;
        for (std::uint32_t q = 0; q < len; ++q) s = __dadd_rn(s, ld(lo + q));
      } else {
        s = __dadd_rn(kid[2 * i], kid[2 * i + 1]);
      }
      cur[i] = s;
    }
    __syncthreads();
  }
  const double r = lvl[0];
  __syncthreads();  // lvl may be reused by the caller
  return r;
}

}  // namespace mb200
