// Reference-structured (SIMT) attention kernels.
//  * k_attn_decode_simple: one CTA per (row, query head) over [prefix ; suffix] read through
//    the page tables (the fp32 parity mode, and the "flat" cross-check of the cascade kernel).
//  * k_attn_prefill: causal attention of prompt positions over the prefix blocks (Alg. 1 L15).
// The bf16 hot path uses the cascade kernel in k_attn_cascade.cu.
#include "kernels.h"

namespace {

template <typename T, int HD>
struct KVSrc {
  const T* pool;
  Dims D;
  int layer, kvh;
  __device__ __forceinline__ const T* tile(long long blk, int kv) const {
    return pool + kv_tile_off(D, layer, blk, kv, kvh);
  }
};

// Online-softmax attention of one query (in smem) over n_tok tokens supplied by tok_loc().
// 4 warps split the tokens; lanes split hd.  Writes o (length HD) to out.
template <typename T, int HD, typename Loc>
__device__ void attend_one(const float* qs, const KVSrc<T, HD>& src, int n_tok, Loc tok_loc, T* out,
                           float* dbg) {
  constexpr int PER = HD / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float scale = rsqrtf((float)HD);
  float m = -INFINITY, l = 0.f, acc[PER];
#pragma unroll
  for (int i = 0; i < PER; ++i) acc[i] = 0.f;
  for (int j = warp; j < n_tok; j += 4) {
    long long blk;
    int t;
    tok_loc(j, blk, t);
    const T* K = src.tile(blk, 0);
    const T* V = src.tile(blk, 1);
    float dot = 0.f;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      int e = lane + 32 * i;
      dot += qs[e] * to_f(K[kv_swz<T>(t, e, HD)]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    float sc = dot * scale;
    float mn = fmaxf(m, sc);
    float corr = expf(m - mn), p = expf(sc - mn);
    l = l * corr + p;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      int e = lane + 32 * i;
      acc[i] = acc[i] * corr + p * to_f(V[kv_swz<T>(t, e, HD)]);
    }
    m = mn;
  }
  __shared__ float sm[4], sl[4], so[4][HD];
  if (lane == 0) { sm[warp] = m; sl[warp] = l; }
#pragma unroll
  for (int i = 0; i < PER; ++i) so[warp][lane + 32 * i] = acc[i];
  __syncthreads();
  if (warp == 0) {
    float M = fmaxf(fmaxf(sm[0], sm[1]), fmaxf(sm[2], sm[3]));
    float w[4], L = 0.f;
#pragma unroll
    for (int k = 0; k < 4; ++k) { w[k] = sm[k] == -INFINITY ? 0.f : expf(sm[k] - M); L += sl[k] * w[k]; }
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      int e = lane + 32 * i;
      float o = 0.f;
#pragma unroll
      for (int k = 0; k < 4; ++k) o += so[k][e] * w[k];
      o /= L;
      out[e] = from_f<T>(o);
      if (dbg) dbg[e] = o;
    }
  }
}

template <typename T, int HD>
__global__ void __launch_bounds__(128) k_attn_decode_simple(const T* __restrict__ q, const T* __restrict__ pool,
                                                            T* __restrict__ out, float* __restrict__ dbg, Dims D,
                                                            int layer, Rows rows, Reqs reqs) {
  const int r = blockIdx.x, head = blockIdx.y;
  if (rows.status[r] != RUNNING_ST) return;
  __shared__ float qs[HD];
  for (int e = threadIdx.x; e < HD; e += blockDim.x) qs[e] = to_f(q[((long long)r * D.qh + head) * HD + e]);
  __syncthreads();
  const int slot = rows.slot[r];
  const int npre = reqs.P[slot] - 1;
  const int nsuf = rows.ell[r] + 1;            // this step's entry already appended
  const int* ptab = reqs.prefix + (long long)slot * D.MPB;
  const int* rtab = rows.table + (long long)r * D.MBR;
  const int bs = D.bs;
  KVSrc<T, HD> src{pool, D, layer, head / D.g};
  auto loc = [=] __device__(int j, long long& blk, int& t) {
    if (j < npre) { blk = ptab[j / bs]; t = j % bs; }
    else { j -= npre; blk = rtab[j / bs]; t = j % bs; }
  };
  long long o = ((long long)r * D.qh + head) * HD;
  attend_one<T, HD>(qs, src, npre + nsuf, loc, out + o, dbg ? dbg + o : nullptr);
}

template <typename T, int HD>
__global__ void __launch_bounds__(128) k_attn_prefill(const T* __restrict__ q, const T* __restrict__ pool,
                                                      T* __restrict__ out, Dims D, int layer, Reqs reqs,
                                                      const int* __restrict__ pf_slot, const int* __restrict__ pf_pos) {
  const int i = blockIdx.x, head = blockIdx.y;
  const int slot = pf_slot[i], p = pf_pos[i];
  __shared__ float qs[HD];
  for (int e = threadIdx.x; e < HD; e += blockDim.x) qs[e] = to_f(q[((long long)i * D.qh + head) * HD + e]);
  __syncthreads();
  const int* ptab = reqs.prefix + (long long)slot * D.MPB;
  const int bs = D.bs;
  KVSrc<T, HD> src{pool, D, layer, head / D.g};
  auto loc = [=] __device__(int j, long long& blk, int& t) { blk = ptab[j / bs]; t = j % bs; };
  attend_one<T, HD>(qs, src, p + 1, loc, out + ((long long)i * D.qh + head) * HD, nullptr);
}

// f2 PRM pass: query i is suffix entry e = sf_ent[i] of batch row sf_row[i] (-1: padding),
// attending to [prefix ; suffix entries 0..e] (its own entry was appended by this layer).
template <typename T, int HD>
__global__ void __launch_bounds__(128) k_attn_suffix(const T* __restrict__ q, const T* __restrict__ pool,
                                                     T* __restrict__ out, Dims D, int layer, Rows rows, Reqs reqs,
                                                     const int* __restrict__ sf_row, const int* __restrict__ sf_ent) {
  const int i = blockIdx.x, head = blockIdx.y;
  const int r = sf_row[i];
  if (r < 0) return;
  const int e = sf_ent[i];
  __shared__ float qs[HD];
  for (int x = threadIdx.x; x < HD; x += blockDim.x) qs[x] = to_f(q[((long long)i * D.qh + head) * HD + x]);
  __syncthreads();
  const int slot = rows.slot[r];
  const int npre = reqs.P[slot] - 1;
  const int* ptab = reqs.prefix + (long long)slot * D.MPB;
  const int* rtab = rows.table + (long long)r * D.MBR;
  const int bs = D.bs;
  KVSrc<T, HD> src{pool, D, layer, head / D.g};
  auto loc = [=] __device__(int j, long long& blk, int& t) {
    if (j < npre) { blk = ptab[j / bs]; t = j % bs; }
    else { j -= npre; blk = rtab[j / bs]; t = j % bs; }
  };
  attend_one<T, HD>(qs, src, npre + e + 1, loc, out + ((long long)i * D.qh + head) * HD, nullptr);
}
}  // namespace

template <typename T>
void launch_attn_suffix(const T* q, const T* pool, T* out, Dims D, int layer, Rows rows, Reqs reqs,
                        const int* sf_row, const int* sf_ent, int n, cudaStream_t s) {
  if (n <= 0) return;
  dim3 grid(n, D.qh);
  if (D.hd == 128) k_attn_suffix<T, 128><<<grid, 128, 0, s>>>(q, pool, out, D, layer, rows, reqs, sf_row, sf_ent);
  else k_attn_suffix<T, 64><<<grid, 128, 0, s>>>(q, pool, out, D, layer, rows, reqs, sf_row, sf_ent);
}
template void launch_attn_suffix<float>(const float*, const float*, float*, Dims, int, Rows, Reqs, const int*,
                                        const int*, int, cudaStream_t);
template void launch_attn_suffix<bf16>(const bf16*, const bf16*, bf16*, Dims, int, Rows, Reqs, const int*,
                                       const int*, int, cudaStream_t);

template <typename T>
void launch_attn_decode_simple(const T* q, const T* pool, T* out, float* dbg, Dims D, int layer, Rows rows,
                               Reqs reqs, int n, cudaStream_t s) {
  if (n <= 0) return;
  dim3 grid(n, D.qh);
  if (D.hd == 128) k_attn_decode_simple<T, 128><<<grid, 128, 0, s>>>(q, pool, out, dbg, D, layer, rows, reqs);
  else k_attn_decode_simple<T, 64><<<grid, 128, 0, s>>>(q, pool, out, dbg, D, layer, rows, reqs);
}
template <typename T>
void launch_attn_prefill(const T* q, const T* pool, T* out, Dims D, int layer, Reqs reqs, const int* pf_slot,
                         const int* pf_pos, int n, cudaStream_t s) {
  if (n <= 0) return;
  dim3 grid(n, D.qh);
  if (D.hd == 128) k_attn_prefill<T, 128><<<grid, 128, 0, s>>>(q, pool, out, D, layer, reqs, pf_slot, pf_pos);
  else k_attn_prefill<T, 64><<<grid, 128, 0, s>>>(q, pool, out, D, layer, reqs, pf_slot, pf_pos);
}
template void launch_attn_decode_simple<float>(const float*, const float*, float*, float*, Dims, int, Rows, Reqs,
                                               int, cudaStream_t);
template void launch_attn_decode_simple<bf16>(const bf16*, const bf16*, bf16*, float*, Dims, int, Rows, Reqs, int,
                                              cudaStream_t);
template void launch_attn_prefill<float>(const float*, const float*, float*, Dims, int, Reqs, const int*,
                                         const int*, int, cudaStream_t);
template void launch_attn_prefill<bf16>(const bf16*, const bf16*, bf16*, Dims, int, Reqs, const int*, const int*, int,
                                        cudaStream_t);
