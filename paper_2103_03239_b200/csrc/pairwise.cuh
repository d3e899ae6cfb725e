// pairwise.cuh -- the reference pairwise tree (core.hpp:72-81) for a RUNTIME
// element count, evaluated iteratively with an explicit stack (no device
// recursion): n <= 8 sums sequentially from +0, larger n splits at floor(n/2)
// and adds left + right.  Used for groups larger than the compile-time cases
// and for the all-peer column means of the diagnostics (n = N).
#pragma once
#include <cstdint>

namespace mb200 {

template <typename V, class Load, class Add>
__device__ V pairwise_rt(Load& ld, std::uint32_t n, Add add, V zero) {
  constexpr int kDepth = 64;
  std::uint32_t f_lo[kDepth], f_n[kDepth];
  std::uint8_t f_phase[kDepth];
  V vals[kDepth];
  int sp = 0, vsp = 0;
  f_lo[0] = 0;
  f_n[0] = n;
  f_phase[0] = 0;
  sp = 1;
  while (sp > 0) {
    const int t = sp - 1;
    const std::uint32_t lo = f_lo[t], cnt = f_n[t];
    if (cnt <= 8) {
      V s = zero;
      for (std::uint32_t i = 0; i < cnt; ++i) s = add(s, ld(lo + i));
      vals[vsp++] = s;
      --sp;
      continue;
    }
    const std::uint32_t h = cnt / 2;
    if (f_phase[t] == 0) {
      f_phase[t] = 1;
      f_lo[sp] = lo;
      f_n[sp] = h;
      f_phase[sp] = 0;
      ++sp;
    } else if (f_phase[t] == 1) {
      f_phase[t] = 2;
      f_lo[sp] = lo + h;
      f_n[sp] = cnt - h;
      f_phase[sp] = 0;
      ++sp;
    } else {
      const V b = vals[--vsp];
      const V a = vals[--vsp];
      vals[vsp++] = add(a, b);
      --sp;
    }
  }
  return vals[0];
}

}  // namespace mb200
