// Decoder elementwise kernels: weight init, embedding gather, RMSNorm, RoPE + paged KV
// append, SwiGLU, PRM head tail.  (SURVEY §8(a) rows a2, a3, a5, a6, a8.)
#include <cstdio>

#include "kernels.h"

// ------------------------------------------------------------ device weight init
// N(0, std^2) via Philox + Box-Muller; norms 1 + N(0, 0.1^2).  Inputs only: the
// values do not matter for timing runs (parity runs pass host_weights).
// Element gi of tensor tid is a function of (seed, tid, gi) only, so a TP rank's shard
// (local element i = global goff + (i / cl) * cf + c0 + i % cl) equals the TP = 1 tensor's.
template <typename T>
__global__ void k_init_tensor(T* p, long long n, int tid, int is_norm, float std, unsigned long long seed,
                              long long cl, long long cf, long long c0, long long goff) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long stride = (long long)gridDim.x * blockDim.x;
  for (; i < n; i += stride) {
    const long long gi = goff + (i / cl) * cf + c0 + i % cl;
    long long pr = gi >> 1;
    u32x4 w = philox4x32_10(u32x4{(uint32_t)pr, (uint32_t)(pr >> 32), (uint32_t)tid, 0xC0FFEEu},
                            (uint32_t)seed, (uint32_t)(seed >> 32));
    float u1 = ((w.x >> 8) + 0.5f) * (1.0f / 16777216.0f);
    float u2 = ((w.y >> 8) + 0.5f) * (1.0f / 16777216.0f);
    float r = sqrtf(-2.0f * logf(u1));
    float z = (gi & 1) ? r * sinpif(2.0f * u2) : r * cospif(2.0f * u2);
    p[i] = from_f<T>(is_norm ? 1.0f + 0.1f * z : std * z);
  }
}
template <typename T>
void launch_init_slice(T* p, long long n, int tid, int is_norm, float std, unsigned long long seed, long long cl,
                       long long cf, long long c0, long long goff, cudaStream_t s) {
  if (n <= 0) return;
  long long blocks = (n + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;
  k_init_tensor<T><<<(int)blocks, 256, 0, s>>>(p, n, tid, is_norm, std, seed, cl, cf, c0, goff);
}
template <typename T>
void launch_init_tensor(T* p, long long n, int tid, int is_norm, float std, unsigned long long seed,
                        cudaStream_t s) {
  launch_init_slice<T>(p, n, tid, is_norm, std, seed, n > 0 ? n : 1, n > 0 ? n : 1, 0, 0, s);
}

// ------------------------------------------------------------ embedding: h = E[tok]
template <typename T>
__global__ void k_embed(const int* __restrict__ tok, const T* __restrict__ emb, float* __restrict__ h, int d) {
  pdl_wait();
  pdl_trigger();
  int r = blockIdx.x;
  const T* e = emb + (long long)tok[r] * d;
  for (int i = threadIdx.x; i < d; i += blockDim.x) h[(long long)r * d + i] = to_f(e[i]);
}
template <typename T>
void launch_embed(const int* tok, const T* emb, float* h, int n, int d, cudaStream_t s) {
  if (n > 0) launch_pdl(k_embed<T>, dim3(n), dim3(256), 0, s, tok, emb, h, d);
}

// ------------------------------------------------------------ RMSNorm (+ residual partials)
// h[r] += sum_{s < np} parts[s][r]   (split-K partials of the previous projection, summed in
// split order: deterministic), then out = h * rsqrt(mean(h^2) + eps) * g.  Rows with status
// != RUNNING are skipped when status is given (the final norm keeps the z of finished rows
// for the PRM, O6).
template <typename T> __device__ __forceinline__ void store4(T* p, float4 v);
template <> __device__ __forceinline__ void store4<float>(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
template <> __device__ __forceinline__ void store4<bf16>(bf16* p, float4 v) {
  __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
  uint2 u;
  u.x = *reinterpret_cast<uint32_t*>(&a);
  u.y = *reinterpret_cast<uint32_t*>(&b);
  *reinterpret_cast<uint2*>(p) = u;
}
template <typename T> __device__ __forceinline__ float4 load4(const T* p);
template <> __device__ __forceinline__ float4 load4<float>(const float* p) { return *reinterpret_cast<const float4*>(p); }
template <> __device__ __forceinline__ float4 load4<bf16>(const bf16* p) {
  uint2 u = *reinterpret_cast<const uint2*>(p);
  __nv_bfloat162 a = *reinterpret_cast<__nv_bfloat162*>(&u.x), b = *reinterpret_cast<__nv_bfloat162*>(&u.y);
  return make_float4(__low2float(a), __high2float(a), __low2float(b), __high2float(b));
}

// one CTA per row, float4 vectorised (d % 4 == 0, checked at init); the CTA width depends
// on d only (rmsnorm_threads), so a row's rounding never depends on the batch size
template <typename T>
__global__ void __launch_bounds__(512) k_rmsnorm(float* __restrict__ h, const float* __restrict__ parts, int np,
                                                  long long pstride, const T* __restrict__ g, T* __restrict__ out,
                                                  float* __restrict__ out32, const int* __restrict__ status, int n,
                                                  int d, float eps) {
  pdl_wait();
  pdl_trigger();
  const int r = blockIdx.x;
  if (status && status[r] != RUNNING_ST) return;

  float4* x = reinterpret_cast<float4*>(h + (long long)r * d);
  const int d4 = d >> 2;
  float ss = 0.f;
  for (int i = threadIdx.x; i < d4; i += blockDim.x) {
    float4 v = x[i];
    for (int sp = 0; sp < np; ++sp) {   // split order: deterministic
      // L2 loads (.cg): under tensor parallelism the partials were written by another rank's
      // kernel, outside this stream's dependency chain, so no L1 / read-only-cache line may serve them
      const float4 p = __ldcg(reinterpret_cast<const float4*>(parts + sp * pstride + (long long)r * d) + i);
      v.x += p.x; v.y += p.y; v.z += p.z; v.w += p.w;
    }
    if (np) x[i] = v;
    ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  __shared__ float red[16];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  float tot = 0.f;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red[w];   // fixed order
  const float inv = rsqrtf(tot / d + eps);
  for (int i = threadIdx.x; i < d4; i += blockDim.x) {
    const float4 v = x[i];
    const float4 gg = load4<T>(g + 4 * i);
    const float4 y = make_float4(v.x * inv * gg.x, v.y * inv * gg.y, v.z * inv * gg.z, v.w * inv * gg.w);
    store4<T>(out + (long long)r * d + 4 * i, y);
    if (out32) reinterpret_cast<float4*>(out32 + (long long)r * d)[i] = y;
  }
}
// 128 threads up to d = 2048 (C2: d = 1536), then ~16 elements per thread up to 512 threads:
// small-M decode (14B / 70B) has few rows, and a 128-thread CTA per 8192-wide row left the
// kernel latency-bound (19.6 us per launch at 64 rows on the 70B shape)
static int rmsnorm_threads(int d) {
  if (d % 128 == 0 && d / 4 <= 512) return d / 4;   // one float4 per thread (C2: 384 threads)
  int t = 128;
  while (t < 512 && d / t > 16) t *= 2;
  return t;
}
// Tensor parallelism: one warp waits until every rank's partial tiles of the projection have
// landed (arrival counter >= the expected count the local producer set), and only then lets
// the RMSNorm launch (pdl_trigger after the wait).  The wait occupies one warp, never the SMs
// the peers' GEMMs need -- which matters when ranks share a GPU (tests) -- and a peer that
// never delivers traps after 20 s instead of hanging the device.
__global__ void k_tp_wait(const unsigned long long* __restrict__ cnt, const unsigned long long* __restrict__ expect) {
  pdl_wait();   // the local producer has finished: *expect is final
  if (threadIdx.x == 0) {
    const unsigned long long target = *reinterpret_cast<const volatile unsigned long long*>(expect);
#ifdef SART_TP_DEBUG
    printf("tp wait cnt %p target %llu now %llu\n", (const void*)cnt, target, *(const volatile unsigned long long*)cnt);
#endif
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
      unsigned long long v, t;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(cnt) : "memory");
      if (v >= target) break;
      __nanosleep(64);
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 20000000000ull) {   // a peer never delivered (20 s): fail, do not hang
#ifdef SART_TP_DEBUG
        printf("k_tp_wait timeout: counter %llu < expected %llu (cnt %p)\n", v, target, (const void*)cnt);
        break;
#else
        __trap();
#endif
      }
    }
    __threadfence();
  }
  __syncwarp();
  pdl_trigger();
}
template <typename T>
void launch_rmsnorm(float* h, const float* parts, int np, const T* g, T* out, float* out32, const int* status, int n,
                    int d, float eps, cudaStream_t s, const unsigned long long* tp_cnt,
                    const unsigned long long* tp_expect) {
  if (n <= 0) return;
  if (tp_cnt) launch_pdl(k_tp_wait, dim3(1), dim3(32), 0, s, tp_cnt, tp_expect);
  launch_pdl(k_rmsnorm<T>, dim3(n), dim3(rmsnorm_threads(d)), 0, s, h, parts, np, (long long)n * d, g, out, out32,
             status, n, d, eps);
}

// ------------------------------------------------------------ RoPE + KV append
// qkv (fp32, bias included) -> q (rotated) into qout[r][qh][hd]; k (rotated), v into the
// paged pool.  Decode: suffix entry l of row r at table[r][l/bs], slot l%bs, position
// P-1+l.  Prefill: prefix position p0+r at prefix[slot][p/bs], slot p%bs.
template <typename T>
__global__ void k_rope_append(const float* __restrict__ parts, int np, long long pstride,
                              const float* __restrict__ bias, T* __restrict__ qout, T* __restrict__ pool,
                              const float* __restrict__ rope_cs, Dims D, int layer, Rows rows, Reqs reqs,
                              RopeArgs a) {
  int r = blockIdx.x;
  int pos, blk, slot_in_blk;
  bool write_kv = true;
  if (a.sf_row) {                                  // f2 PRM pass: suffix entry of a batch row
    const int row = a.sf_row[r];
    if (row < 0) return;
    const int l = a.pf_pos[r];
    pos = reqs.P[rows.slot[row]] - 1 + l;
    blk = rows.table[(long long)row * D.MBR + l / D.bs];
    slot_in_blk = l % D.bs;
  } else if (a.pf_slot) {
    pos = a.pf_pos[r];
    blk = reqs.prefix[(long long)a.pf_slot[r] * D.MPB + pos / D.bs];
    slot_in_blk = pos % D.bs;
  } else {
    if (rows.status[r] != RUNNING_ST) return;
    int l = rows.ell[r];
    pos = reqs.P[rows.slot[r]] - 1 + l;
    blk = rows.table[(long long)r * D.MBR + l / D.bs];
    slot_in_blk = l % D.bs;
  }
  const int half = D.hd / 2;
  const float* x = parts + (long long)r * D.qkv;
  const float* cs = rope_cs + (long long)pos * D.hd;   // [cos(half) | sin(half)]
  int pairs = (D.qh + 2 * D.kvh) * half;
  for (int t = threadIdx.x; t < pairs; t += blockDim.x) {
    int head = t / half, i = t % half;
    const int e1 = head * D.hd + i, e2 = e1 + half;
    float x1 = bias[e1], x2 = bias[e2];
    for (int sp = 0; sp < np; ++sp) { x1 += x[sp * pstride + e1]; x2 += x[sp * pstride + e2]; }   // split order
    if (head < D.qh + D.kvh) {                      // q or k: rotate-half
      float c = cs[i], sn = cs[half + i];
      float y1 = x1 * c - x2 * sn, y2 = x2 * c + x1 * sn;
      x1 = y1; x2 = y2;
    }
    if (head < D.qh) {
      T* q = qout + ((long long)r * D.qh + head) * D.hd;
      q[i] = from_f<T>(x1);
      q[i + half] = from_f<T>(x2);
    } else if (write_kv) {
      int kv = head < D.qh + D.kvh ? 0 : 1;
      int h = kv == 0 ? head - D.qh : head - D.qh - D.kvh;
      T* tile = pool + kv_tile_off(D, layer, blk, kv, h);
      tile[kv_swz<T>(slot_in_blk, i, D.hd)] = from_f<T>(x1);
      tile[kv_swz<T>(slot_in_blk, i + half, D.hd)] = from_f<T>(x2);
    }
  }
}
template <typename T>
void launch_rope_append(const float* parts, int np, const float* bias, T* qout, T* pool, const float* rope_cs, Dims D,
                        int layer, Rows rows, Reqs reqs, RopeArgs a, int n, cudaStream_t s) {
  if (n > 0)
    k_rope_append<T><<<n, 256, 0, s>>>(parts, np, (long long)n * D.qkv, bias, qout, pool, rope_cs, D, layer, rows,
                                       reqs, a);
}

// ------------------------------------------------------------ SwiGLU: act = SiLU(g) * u
template <typename T>
__global__ void k_swiglu(const float* __restrict__ gu, T* __restrict__ act, int F) {
  int r = blockIdx.x;
  const float* x = gu + (long long)r * 2 * F;
  for (int i = threadIdx.x; i < F; i += blockDim.x) {
    float g = x[i], u = x[F + i];
    act[(long long)r * F + i] = from_f<T>(g / (1.0f + expf(-g)) * u);
  }
}
template <typename T>
void launch_swiglu(const float* gu, T* act, int n, int F, cudaStream_t s) {
  if (n > 0) k_swiglu<T><<<n, 256, 0, s>>>(gu, act, F);
}

// ------------------------------------------------------------ PRM head tail
// hid = z W1^T + b1 (fp32, from the GEMM); score = softmax(ReLU(hid) W2^T + b2)[1].
__global__ void k_prm_head2(const float* __restrict__ hid, const float* __restrict__ w2,
                            const float* __restrict__ b2, float* __restrict__ score, int d) {
  int r = blockIdx.x;
  float a0 = 0.f, a1 = 0.f;
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    float x = fmaxf(hid[(long long)r * d + i], 0.f);
    a0 += x * w2[i];
    a1 += x * w2[d + i];
  }
  __shared__ float r0[32], r1[32];
  for (int o = 16; o > 0; o >>= 1) {
    a0 += __shfl_xor_sync(0xffffffffu, a0, o);
    a1 += __shfl_xor_sync(0xffffffffu, a1, o);
  }
  if ((threadIdx.x & 31) == 0) { r0[threadIdx.x >> 5] = a0; r1[threadIdx.x >> 5] = a1; }
  __syncthreads();
  if (threadIdx.x == 0) {
    float l0 = b2[0], l1 = b2[1];
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { l0 += r0[w]; l1 += r1[w]; }
    float m = fmaxf(l0, l1);
    float e0 = expf(l0 - m), e1 = expf(l1 - m);
    score[r] = e1 / (e0 + e1);
  }
}
void launch_prm_head2(const float* hid, const float* w2, const float* b2, float* score, int n, int d,
                      cudaStream_t s) {
  if (n > 0) k_prm_head2<<<n, 256, 0, s>>>(hid, w2, b2, score, d);
}

template <typename T>
__global__ void k_convert(const float* __restrict__ in, T* __restrict__ out, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = from_f<T>(in[i]);
}
template <typename T>
void launch_convert(const float* in, T* out, long long n, cudaStream_t s) {
  if (n > 0) k_convert<T><<<(int)((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096), 256, 0, s>>>(in, out, n);
}
template <typename T>
__global__ void k_to_f32(const T* __restrict__ in, float* __restrict__ out, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = to_f(in[i]);
}
template <typename T>
void launch_to_f32(const T* in, float* out, long long n, cudaStream_t s) {
  if (n > 0) k_to_f32<T><<<(int)((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096), 256, 0, s>>>(in, out, n);
}

// ------------------------------------------------------------ f2 PRM pass
// Token list of one packed chunk: segment {first token, count, row, first entry}; token
// t0 + j is suffix entry e = e0 + j of that row, whose input is the last prompt token for
// e = 0 (R22) and the generated token y_e = hist[e-1] otherwise.
__global__ void k_prm_tokens(Dims D, Rows rows, Reqs reqs, const int4* __restrict__ seg, int* __restrict__ tok,
                             int* __restrict__ row, int* __restrict__ ent) {
  const int4 sg = seg[blockIdx.x];
  const int r = sg.z, slot = rows.slot[r];
  const long long sb = (long long)slot * SART_MAXN + rows.b[r];
  for (int j = threadIdx.x; j < sg.y; j += blockDim.x) {
    const int e = sg.w + j, t = sg.x + j;
    tok[t] = e == 0 ? reqs.first_tok[slot] : reqs.hist[sb * D.cap + (e - 1)];
    row[t] = r;
    ent[t] = e;
  }
}
void launch_prm_tokens(Dims D, Rows rows, Reqs reqs, const int4* seg, int nseg, int* tok, int* row, int* ent,
                       cudaStream_t s) {
  if (nseg > 0) k_prm_tokens<<<nseg, 256, 0, s>>>(D, rows, reqs, seg, tok, row, ent);
}
// zrow[row] = z[token of the row's last entry] (the PRM's score position)
template <typename T>
__global__ void k_prm_gather(const T* __restrict__ z, T* __restrict__ zrow, const int4* __restrict__ gat, int d) {
  const int4 g = gat[blockIdx.x];
  for (int i = threadIdx.x; i < d; i += blockDim.x) zrow[(long long)g.x * d + i] = z[(long long)g.y * d + i];
}
template <typename T>
void launch_prm_gather(const T* z, T* zrow, const int4* gat, int ng, int d, cudaStream_t s) {
  if (ng > 0) k_prm_gather<T><<<ng, 256, 0, s>>>(z, zrow, gat, d);
}

#define INST(T)                                                                                        \
  template void launch_init_tensor<T>(T*, long long, int, int, float, unsigned long long, cudaStream_t); \
  template void launch_embed<T>(const int*, const T*, float*, int, int, cudaStream_t);                  \
  template void launch_rmsnorm<T>(float*, const float*, int, const T*, T*, float*, const int*, int, int, \
                                  float, cudaStream_t, const unsigned long long*,                       \
                                  const unsigned long long*);                                           \
  template void launch_init_slice<T>(T*, long long, int, int, float, unsigned long long, long long,     \
                                     long long, long long, long long, cudaStream_t);                    \
  template void launch_rope_append<T>(const float*, int, const float*, T*, T*, const float*, Dims, int, \
                                      Rows, Reqs, RopeArgs, int, cudaStream_t);                         \
  template void launch_swiglu<T>(const float*, T*, int, int, cudaStream_t);                             \
  template void launch_convert<T>(const float*, T*, long long, cudaStream_t);                           \
  template void launch_to_f32<T>(const T*, float*, long long, cudaStream_t);                           \
  template void launch_prm_gather<T>(const T*, T*, const int4*, int, int, cudaStream_t);
INST(float)
INST(bf16)

// gate|up rows [2F][d] -> 256-row tiles [gate 128 | up 128] for the fused SwiGLU epilogue
__global__ void k_interleave(const bf16* __restrict__ src, bf16* __restrict__ dst, int F, int d) {
  const int r = blockIdx.x;              // destination row
  const int tile = r / 256, w = r % 256;
  const int sr = w < 128 ? tile * 128 + w : F + tile * 128 + (w - 128);
  for (int i = threadIdx.x; i < d; i += blockDim.x) dst[(long long)r * d + i] = src[(long long)sr * d + i];
}
void launch_interleave_gate_up(bf16* w, bf16* tmp, int F, int d, cudaStream_t s) {
  cudaMemcpyAsync(tmp, w, sizeof(bf16) * 2 * (size_t)F * d, cudaMemcpyDeviceToDevice, s);
  k_interleave<<<2 * F, 256, 0, s>>>(tmp, w, F, d);
}
