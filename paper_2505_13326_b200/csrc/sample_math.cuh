// Per-element arithmetic of the Gumbel-max sampler (readings R24, R25), shared by the
// stand-alone sampler (k_sample.cu) and the sampler fused into the LM-head GEMM epilogue.
//   key_v = logit_v / tau + G_v,  G_v = -ln(-ln u_v),  u_v = ((w >> 8) + 0.5) 2^-24,
//   w = Philox4x32-10((v >> 2, s, request_id, branch), seed)[v & 3];  ties -> lowest v.
// fp32; -ln u is evaluated as log1p(-(2^24 - x - 0.5) 2^-24) in the upper half so that u
// is represented exactly.
#pragma once
#include "common.cuh"

__device__ __forceinline__ float gumbel_from_word(uint32_t w) {
  uint32_t x = w >> 8;
  float lnu;
  if (x < (1u << 23)) lnu = logf(((float)x + 0.5f) * (1.0f / 16777216.0f));
  else lnu = log1pf(-(((float)((1u << 24) - x)) - 0.5f) * (1.0f / 16777216.0f));
  return -logf(-lnu);
}

__device__ __forceinline__ void better(float& bk, int& bv, float k, int v) {
  if (k > bk || (k == bk && v < bv)) { bk = k; bv = v; }
}

// Exact pruning (no change to any result): with E = -ln u >= 1 - u, the key l' + G = l' - ln E
// is < l' - ln(1 - u), so an entry whose (1 - u) exceeds exp(l' - bound) (0.1% margin, which
// covers the fp32 rounding of every step) cannot reach `bound` -- a key some entry already
// has -- and its two logarithms are skipped.  bound = -inf disables pruning.
__device__ __forceinline__ bool gumbel_cannot_reach(uint32_t w, float lp, float bound) {
  const float one_minus_u = ((float)((1u << 24) - (w >> 8)) - 0.5f) * (1.0f / 16777216.0f);
  return one_minus_u > __expf(lp - bound) * 1.001f;
}

// fold 4 consecutive vocab entries v0..v0+3 (v0 % 4 == 0) into (bk, bv); entries whose key
// provably stays below `bound` are skipped (see gumbel_cannot_reach).  The skip threshold is
// computed once per group from the group's largest l': exp(l'_j - bound) <= exp(max l' -
// bound), so the per-entry test is weaker than gumbel_cannot_reach's and skips only entries
// that test would skip as well (every result is unchanged).
__device__ __forceinline__ void sample_group4(float& bk, int& bv, const float* lv, int v0, int V, int s, uint32_t rid,
                                              uint32_t b, uint32_t k0, uint32_t k1, float tau, bool mask_eos,
                                              int eos, float bound = -INFINITY) {
  u32x4 w{0, 0, 0, 0};
  if (tau > 0.f) w = philox4x32_10(u32x4{(uint32_t)(v0 >> 2), (uint32_t)s, rid, b}, k0, k1);
  const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
  float lp[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) lp[j] = tau == 1.0f ? lv[j] : lv[j] / tau;
  const float thr = __expf(fmaxf(fmaxf(lp[0], lp[1]), fmaxf(lp[2], lp[3])) - bound) * 1.001f;
  const bool full = v0 + 3 < V && !mask_eos;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int v = v0 + j;
    if (!full && (v >= V || (mask_eos && v == eos))) continue;
    float key;
    if (tau > 0.f) {
      const float one_minus_u = ((float)((1u << 24) - (ws[j] >> 8)) - 0.5f) * (1.0f / 16777216.0f);
      if (one_minus_u > thr) continue;
      key = lp[j] + gumbel_from_word(ws[j]);
    } else {
      key = lv[j];
    }
    better(bk, bv, key, v);
  }
}
