// Shared device-side definitions of the SART engine (sm_100a).
#pragma once
#include <cstdlib>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

typedef __nv_bfloat16 bf16;

#define SART_MAXN 32          // branches per request (one warp lane each)
#define RUNNING_ST 1          // == SART_BR_RUNNING
#define ST_EOS 2
#define ST_CAP 3
#define ST_PRUNED 4
#define ST_ES 5
#define ST_STOP 7             // es_every_step (R43): stopped mid-window by early stop, EarlyStopped at the boundary
#define ST_WAIT 8             // R44: admitted, waiting for its interleaved prefill (starts at rows.start)

template <typename T> __device__ __forceinline__ float to_f(T x);
template <> __device__ __forceinline__ float to_f<float>(float x) { return x; }
template <> __device__ __forceinline__ float to_f<bf16>(bf16 x) { return __bfloat162float(x); }
template <typename T> __device__ __forceinline__ T from_f(float x);
template <> __device__ __forceinline__ float from_f<float>(float x) { return x; }
template <> __device__ __forceinline__ bf16 from_f<bf16>(float x) { return __float2bfloat16_rn(x); }

// Model and engine dimensions (plain values, passed by value to kernels).
struct Dims {
  int L, d, qh, kvh, hd, F, V, qkv, g;
  int bs, R, S, MBR, MPB, cap, T, eos, nbnd_max, max_pos;
  long long NB;
  float theta, eps, tau;
  unsigned long long seed;
  int select_mode;
};

// Paged KV pool: [L][NB][2][kvh][bs][hd] elements of T.  Inside one (layer, block,
// k|v, head) tile the 16-byte chunk c of token row t is stored at chunk c ^ (t & 7)
// so that 8 consecutive token rows read at the same logical column hit 8 distinct
// bank groups (ldmatrix / 1-D bulk copies need no further swizzle).
__host__ __device__ __forceinline__ long long kv_tile_off(const Dims& D, int layer, long long blk,
                                                          int kv, int h) {
  return ((((long long)layer * D.NB + blk) * 2 + kv) * D.kvh + h) * (long long)D.bs * D.hd;
}
template <typename T>
__host__ __device__ __forceinline__ int kv_swz(int t, int e, int hd) {
  constexpr int EPC = 16 / sizeof(T);
  return t * hd + (((e / EPC) ^ (t & 7)) * EPC) + (e % EPC);
}

// Per-row state of current_batch (Alg. 1 "current_batch", D3/D5).
struct Rows {
  int* slot;      // request slot
  int* b;         // branch index (paper's j, 0-based)
  int* ell;       // steps decoded == tokens generated
  int* status;    // RUNNING_ST while decoding, ST_EOS / ST_CAP when done this window
  int* done_step;
  int* done_wstep;
  int* nbnd;      // boundaries seen while running (script index)
  int* tok;       // next input token
  int* term;      // terminal state decided at the boundary
  int* nblk;      // blocks owned
  int* start;     // R44: first window step it decodes in its first window (status ST_WAIT until then)
  float* score;
  int* table;     // [R][MBR]
};

// Per-request slot state (meta[i] of Alg. 1 L16 plus bookkeeping).
struct Reqs {
  long long* id;
  int *N, *M, *P, *beta, *prune, *phase, *maxp, *nc, *np, *nes, *npre, *first_tok;
  int *has_script, *has_answer, *has_forced, *nbnd;
  int* ncw;         // completed branches including this window's so far (es_every_step, R43)
  float *alpha, *thr;
  int* prefix;      // [S][MPB]
  int* br_state;    // [S][32]
  int* br_len;      // [S][32]
  int* br_label;    // [S][32]
  float* br_score;  // [S][32]
  int* sc_len;      // [S][32] forced_len (0 = none)
  int* sc_answer;   // [S][32]
  float* sc_final;  // [S][32]
  float* sc_scores; // [S][32][nbnd_max]
  int* forced;      // [S][32][cap] or null
  int* hist;        // [S][32][cap]
  int* final_flag;  // [S]
};

// Device-side counters shared by host and kernels.
struct Ctr {
  int live;        // rows still running in this window
  int wstep;       // window step index (1..T)
  int steps;       // decode steps since init
  int n_rows;
  long long free_top;
  long long committed;
  int n_final;
  int windows;
  long long branch_tokens;
  double attn_bytes;   // algorithmic attention bytes (profiling)
  int final_slots[1]; // [S] (allocated with the struct)
};

struct DevResult {
  long long request_id;
  int answer_vote, vote_count, chosen_max_reward, answer_max_reward;
  int num_completed, num_pruned, num_early_stopped;
  int finalize_reason, phase_at_end;
  float threshold_at_end;
  int selected_branch;
  int branch_len[SART_MAXN];
  int branch_state[SART_MAXN];
  float branch_score[SART_MAXN];
};

#define CUDA_KCHECK() (cudaGetLastError())

// Philox4x32-10 (Salmon et al., SC'11): used by the sampler (R25) and by the
// device weight initialiser.
struct u32x4 { uint32_t x, y, z, w; };
__device__ __forceinline__ u32x4 philox4x32_10(u32x4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = u32x4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
  }
  return c;
}

// Programmatic dependent launch (PDL): a kernel launched with programmatic stream
// serialization may start while its predecessor drains; it must call pdl_wait() before it
// reads anything the predecessor produced (or writes anything the predecessor reads).
// pdl_trigger() lets the next kernel in the stream start its own prologue.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

#ifdef __CUDACC__
#include <mutex>
#include <set>
#include <utility>
// SM count of the CURRENT device (engines on different devices in one process each see their
// own), cached per ordinal
inline int device_sms() {
  static int cache[64] = {};
  int d = 0;
  cudaGetDevice(&d);
  if (d < 0 || d >= 64) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
    return v;
  }
  if (!cache[d]) cudaDeviceGetAttribute(&cache[d], cudaDevAttrMultiProcessorCount, d);
  return cache[d];
}
// cudaFuncAttributeMaxDynamicSharedMemorySize is a per-device setting of a kernel: set it once
// per (kernel, device, size)
template <typename Kern>
inline void ensure_dyn_smem(Kern kernel, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<std::pair<const void*, int>, int>> done;
  int d = 0;
  cudaGetDevice(&d);
  const auto key = std::make_pair(std::make_pair((const void*)kernel, d), bytes);
  std::lock_guard<std::mutex> lk(mu);
  if (done.count(key)) return;
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  done.insert(key);
}
// launch with the PDL attribute (also captured into CUDA graphs as programmatic edges)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  // SART_NO_PDL=1: plain stream order (diagnostics)
  static const int pdl = getenv("SART_NO_PDL") && atoi(getenv("SART_NO_PDL")) ? 0 : 1;
  attr[0].val.programmaticStreamSerializationAllowed = pdl;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
#endif
