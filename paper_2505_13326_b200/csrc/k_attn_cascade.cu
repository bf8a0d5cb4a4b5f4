// Cascade paged decode attention (the dominant HBM-bound kernel).
//
//   o_i = sum_t softmax_t(q_i . k_t / sqrt(hd)) v_t   over [prefix (P-1 tokens, shared) ;
//                                                           suffix (l+1 tokens, per branch)]
//
// PAPER P:306 shares the prompt's KV across a request's branches.  We read it ONCE per
// request and kv head: a "prefix unit" multiplies the shared prefix KV by the queries of
// all live branches of the request at once (up to 64 query rows = rows x g heads), while a
// "suffix unit" covers one branch's private KV.  Every unit covers a chunk of <= CH tokens;
// each writes a normalised partial output and its log-sum-exp, and a merge kernel combines
// the partials of each (row, head) in a fixed order (deterministic, PP4).
//
// Kernel structure (one persistent CTA per SM, 8 consumer warps + 1 producer warp):
//   producer   one lane issues 1-D bulk copies (cp.async.bulk ... mbarrier::complete_tx) of
//              whole paged blocks (bs x hd K tile and V tile, contiguous in the pool) into a
//              4-stage ring of 64-token stages;
//   consumers  two groups of 4 warps take alternate stages; mma.sync m16n8k16 bf16 for
//              S = Q K^T and O += P V with fp32 online softmax; the pool's XOR pre-swizzle
//              (common.cuh kv_swz) makes the ldmatrix reads bank-conflict free.
// Tensor cores are used because QK^T / PV are dense contractions, but the kernel is
// HBM-bound (about g flop per byte); the design goal is bytes in flight, not MMA rate.
#include "kernels.h"

namespace {
constexpr int NCW = 8;                 // consumer warps
constexpr int NTH = (NCW + 1) * 32;    // + producer warp
constexpr int STG = 4;                 // pipeline stages
constexpr int ST_TOK = 64;             // tokens per stage

__device__ __forceinline__ uint32_t s_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s_u32(b)), "r"(c));
}
__device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s_u32(b)) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t par) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W_%=;\n\t}" ::"r"(s_u32(b)),
      "r"(par)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   s_u32(dst)),
               "l"(src), "r"(bytes), "r"(s_u32(bar))
               : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void mma16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// Decoded work item.  Units come from the per-window plan; the token range depends on the
// current step (rows grow by one token per step).
struct ItemInfo {
  int valid;        // 0: skip
  int nq;           // query rows (<= 64)
  int t0, t1;       // token range in the source sequence
  const int* tab;   // block table of the source (prefix table or row table)
  int slot_idx;     // partial-output slot index
  int unit;
};

__device__ __forceinline__ ItemInfo decode_item(const AttnPlan& pl, const Dims& D, const Rows& rows, const Reqs& reqs,
                                                int unit) {
  ItemInfo it{};
  it.unit = unit;
  const int4 u = pl.units[unit];
  const int type = u.x, c = u.z;
  if (type == 0) {                               // suffix unit: (row, chunk)
    const int r = u.y;
    if (rows.status[r] != RUNNING_ST) return it;
    const int len = rows.ell[r] + 1;
    it.t0 = c * pl.CH;
    it.t1 = min(it.t0 + pl.CH, len);
    if (it.t0 >= it.t1) return it;
    it.nq = D.g;
    it.tab = rows.table + (long long)r * D.MBR;
    it.slot_idx = pl.npc_max + c;
  } else {                                       // prefix unit: (group, chunk)
    const int gi = u.y;
    const int slot = pl.grp_slot[gi];
    const int n = pl.grp_n[gi];
    bool any = false;
    for (int k = 0; k < n; ++k) any |= rows.status[pl.grp_rows[gi * pl.qr_max + k]] == RUNNING_ST;
    if (!any) return it;
    const int len = reqs.P[slot] - 1;
    it.t0 = c * pl.CH;
    it.t1 = min(it.t0 + pl.CH, len);
    if (it.t0 >= it.t1) return it;
    it.nq = n * D.g;
    it.tab = reqs.prefix + (long long)slot * D.MPB;
    it.slot_idx = c;
  }
  it.valid = 1;
  return it;
}

// query row j of an item -> (batch row, q head)
__device__ __forceinline__ void q_of(const AttnPlan& pl, const Dims& D, int unit, int kvh, int j, int& row, int& head) {
  const int4 u = pl.units[unit];
  if (u.x == 0) {
    row = u.y;
    head = kvh * D.g + j;
  } else {
    row = pl.grp_rows[u.y * pl.qr_max + j / D.g];
    head = kvh * D.g + j % D.g;
  }
}

template <int HD>
struct SmemA {
  alignas(128) bf16 k[STG][ST_TOK * HD];
  alignas(128) bf16 v[STG][ST_TOK * HD];
  float mo[NCW][16][HD];       // per-warp partial O (merge)
  float mm[NCW][16], ml[NCW][16];
  uint64_t full[STG], empty[STG];
};

template <int HD>
__global__ void __launch_bounds__(NTH, 1)
    k_attn_cascade(const bf16* __restrict__ q, const bf16* __restrict__ pool, float* __restrict__ part_o,
                   float* __restrict__ part_lse, Dims D, int layer, Rows rows, Reqs reqs, AttnPlan pl) {
  extern __shared__ __align__(128) uint8_t sraw[];
  SmemA<HD>& sm = *reinterpret_cast<SmemA<HD>*>(sraw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_items = *pl.n_units * D.kvh;
  const float sl2 = 1.4426950408889634f * rsqrtf((float)HD);   // log2(e) / sqrt(hd)

  for (int e = threadIdx.x; e < STG * ST_TOK * HD / 8; e += NTH) {
    reinterpret_cast<uint4*>(sm.k)[e] = make_uint4(0, 0, 0, 0);
    reinterpret_cast<uint4*>(sm.v)[e] = make_uint4(0, 0, 0, 0);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes before bulk copies
  if (threadIdx.x == 0) {
    for (int s = 0; s < STG; ++s) { mb_init(&sm.full[s], 1); mb_init(&sm.empty[s], 4); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == NCW) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t tile_bytes = (uint32_t)D.bs * HD * 2;
      for (int i = blockIdx.x; i < n_items; i += gridDim.x) {
        const int unit = i / D.kvh, h = i % D.kvh;
        const ItemInfo it = decode_item(pl, D, rows, reqs, unit);
        if (!it.valid) continue;
        for (int s0 = it.t0; s0 < it.t1; s0 += ST_TOK) {
          const int ntok = min(ST_TOK, it.t1 - s0);
          const int nb = (ntok + D.bs - 1) / D.bs;
          mb_wait(&sm.empty[stage], phase ^ 1);
          mb_expect(&sm.full[stage], 2u * nb * tile_bytes);
          for (int j = 0; j < nb; ++j) {
            const long long blk = it.tab[(s0 / D.bs) + j];
            const bf16* kt = pool + kv_tile_off(D, layer, blk, 0, h);
            const bf16* vt = pool + kv_tile_off(D, layer, blk, 1, h);
            bulk_g2s(sm.k[stage] + j * D.bs * HD, kt, tile_bytes, &sm.full[stage]);
            bulk_g2s(sm.v[stage] + j * D.bs * HD, vt, tile_bytes, &sm.full[stage]);
          }
          if (++stage == STG) { stage = 0; phase ^= 1; }
        }
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const int grp = warp >> 2, wg = warp & 3;          // stage group, warp within group
  uint32_t gk = 0;                                   // CTA-global stage counter (same as the producer's)
  for (int i = blockIdx.x; i < n_items; i += gridDim.x) {
    const int unit = i / D.kvh, h = i % D.kvh;
    const ItemInfo it = decode_item(pl, D, rows, reqs, unit);
    if (!it.valid) continue;
    const int mt = it.nq <= 16 ? 1 : (it.nq <= 32 ? 2 : 4);   // m-tiles of 16 query rows
    const int wpt = 4 / mt;                                   // warps per m-tile within a group
    const int mtile = wg % mt;
    const int slice = wg / mt;                                // token slice of the stage
    const int slice_tok = ST_TOK / wpt;                       // 64, 32 or 16 tokens
    // Q fragments of this warp's m-tile (16 rows x HD), zero beyond nq
    uint32_t qa[HD / 16][4];
    {
      const int r0 = mtile * 16 + (lane >> 2), r1 = r0 + 8;
      const bf16* q0 = nullptr;
      const bf16* q1 = nullptr;
      int row, head;
      if (r0 < it.nq) { q_of(pl, D, unit, h, r0, row, head); q0 = q + ((long long)row * D.qh + head) * HD; }
      if (r1 < it.nq) { q_of(pl, D, unit, h, r1, row, head); q1 = q + ((long long)row * D.qh + head) * HD; }
      const int cc = 2 * (lane & 3);
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
        qa[kk][0] = q0 ? *reinterpret_cast<const uint32_t*>(q0 + 16 * kk + cc) : 0u;
        qa[kk][1] = q1 ? *reinterpret_cast<const uint32_t*>(q1 + 16 * kk + cc) : 0u;
        qa[kk][2] = q0 ? *reinterpret_cast<const uint32_t*>(q0 + 16 * kk + 8 + cc) : 0u;
        qa[kk][3] = q1 ? *reinterpret_cast<const uint32_t*>(q1 + 16 * kk + 8 + cc) : 0u;
      }
    }
    float o[HD / 8][4];
#pragma unroll
    for (int nt = 0; nt < HD / 8; ++nt) o[nt][0] = o[nt][1] = o[nt][2] = o[nt][3] = 0.f;
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

    for (int s0 = it.t0; s0 < it.t1; s0 += ST_TOK, ++gk) {
      const int stage = gk % STG;
      const uint32_t phase = (gk / STG) & 1;
      if ((gk & 1) == (uint32_t)grp) {                // the two warp groups take alternate stages
        mb_wait(&sm.full[stage], phase);
        const int ntok = min(ST_TOK, it.t1 - s0);
        const uint32_t kb = s_u32(sm.k[stage]), vb = s_u32(sm.v[stage]);
        for (int sub = slice * slice_tok; sub < slice * slice_tok + slice_tok; sub += 16) {
          if (sub >= ntok) break;
          // S = Q K^T for 16 tokens [sub, sub+16)
          float s[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk) {
            const int mi = lane >> 3;
            const int tok = sub + (lane & 7) + 8 * (mi >> 1);
            const int ch = 2 * kk + (mi & 1);
            uint32_t b0, b1, b2, b3;
            ldsm_x4(kb + tok * (HD * 2) + ((ch ^ (tok & 7)) << 4), b0, b1, b2, b3);
            mma16816(s[0], qa[kk], b0, b1);
            mma16816(s[1], qa[kk], b2, b3);
          }
          // mask tokens beyond the valid range
          const int cbase = sub + 2 * (lane & 3);
#pragma unroll
          for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if (cbase + nt * 8 + (e & 1) >= ntok) s[nt][e] = -INFINITY;
          // online softmax (rows r = lane/4 -> m0/l0, r+8 -> m1/l1)
          float mx0 = fmaxf(fmaxf(s[0][0], s[0][1]), fmaxf(s[1][0], s[1][1]));
          float mx1 = fmaxf(fmaxf(s[0][2], s[0][3]), fmaxf(s[1][2], s[1][3]));
          mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
          mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
          mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
          mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
          const float n0 = fmaxf(m0, mx0), n1 = fmaxf(m1, mx1);
          const float u0 = n0 == -INFINITY ? 0.f : n0, u1 = n1 == -INFINITY ? 0.f : n1;
          const float c0 = exp2f((m0 - u0) * sl2), c1 = exp2f((m1 - u1) * sl2);
          m0 = n0;
          m1 = n1;
          float p[2][4];
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) {
            p[nt][0] = exp2f((s[nt][0] - u0) * sl2);
            p[nt][1] = exp2f((s[nt][1] - u0) * sl2);
            p[nt][2] = exp2f((s[nt][2] - u1) * sl2);
            p[nt][3] = exp2f((s[nt][3] - u1) * sl2);
          }
          l0 = l0 * c0 + p[0][0] + p[0][1] + p[1][0] + p[1][1];
          l1 = l1 * c1 + p[0][2] + p[0][3] + p[1][2] + p[1][3];
#pragma unroll
          for (int nt = 0; nt < HD / 8; ++nt) { o[nt][0] *= c0; o[nt][1] *= c0; o[nt][2] *= c1; o[nt][3] *= c1; }
          uint32_t pa[4];
          pa[0] = pack_bf16(p[0][0], p[0][1]);
          pa[1] = pack_bf16(p[0][2], p[0][3]);
          pa[2] = pack_bf16(p[1][0], p[1][1]);
          pa[3] = pack_bf16(p[1][2], p[1][3]);
          // O += P V : V rows = tokens [sub, sub+16), ldmatrix.trans per pair of hd n-tiles
#pragma unroll
          for (int dp = 0; dp < HD / 16; ++dp) {
            const int mi = lane >> 3;
            const int tok = sub + (lane & 7) + 8 * (mi & 1);
            const int ch = 2 * dp + (mi >> 1);
            uint32_t b0, b1, b2, b3;
            ldsm_x4_t(vb + tok * (HD * 2) + ((ch ^ (tok & 7)) << 4), b0, b1, b2, b3);
            mma16816(o[2 * dp], pa, b0, b1);
            mma16816(o[2 * dp + 1], pa, b2, b3);
          }
        }
        __syncwarp();
        if (lane == 0) mb_arrive(&sm.empty[stage]);
      }
    }
    // ---- per-warp row sums, then cross-warp merge through shared memory
    l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
    l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
    {
      const int r = lane >> 2, cc = 2 * (lane & 3);
#pragma unroll
      for (int nt = 0; nt < HD / 8; ++nt) {
        sm.mo[warp][r][nt * 8 + cc] = o[nt][0];
        sm.mo[warp][r][nt * 8 + cc + 1] = o[nt][1];
        sm.mo[warp][r + 8][nt * 8 + cc] = o[nt][2];
        sm.mo[warp][r + 8][nt * 8 + cc + 1] = o[nt][3];
      }
      if ((lane & 3) == 0) {
        sm.mm[warp][r] = m0; sm.ml[warp][r] = l0;
        sm.mm[warp][r + 8] = m1; sm.ml[warp][r + 8] = l1;
      }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(NCW * 32));
    // merge: warps with the same m-tile are {g*4 + s*mt + mtile}; thread handles (row, col) pairs
    for (int e = threadIdx.x; e < mt * 16 * HD; e += NCW * 32) {
      const int qrow = e / HD, col = e % HD;
      const int mtl = qrow / 16, rr = qrow % 16;
      if (qrow >= it.nq) continue;
      float M = -INFINITY;
      for (int g2 = 0; g2 < 2; ++g2)
        for (int s2 = 0; s2 < wpt; ++s2) M = fmaxf(M, sm.mm[g2 * 4 + s2 * mt + mtl][rr]);
      float L = 0.f, O = 0.f;
      const float Mu = M == -INFINITY ? 0.f : M;
      for (int g2 = 0; g2 < 2; ++g2)
        for (int s2 = 0; s2 < wpt; ++s2) {
          const int w2 = g2 * 4 + s2 * mt + mtl;
          const float wgt = exp2f((sm.mm[w2][rr] - Mu) * sl2);
          L += sm.ml[w2][rr] * wgt;
          O += sm.mo[w2][rr][col] * wgt;
        }
      int row, head;
      q_of(pl, D, unit, h, qrow, row, head);
      const long long pi = ((long long)row * D.qh + head) * pl.nslot + it.slot_idx;
      part_o[pi * HD + col] = O / L;
      if (col == 0) part_lse[pi] = Mu * sl2 + log2f(L);          // log2-domain LSE
    }
    asm volatile("bar.sync 1, %0;" ::"n"(NCW * 32));
  }
}

// merge the partials of each (row, head) in fixed slot order; o (bf16) and optional fp32 debug
template <int HD>
__global__ void k_attn_merge(const float* __restrict__ part_o, const float* __restrict__ part_lse,
                             bf16* __restrict__ out, float* __restrict__ dbg, Dims D, Rows rows, Reqs reqs,
                             AttnPlan pl, int n) {
  const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (wid >= n * D.qh) return;
  const int r = wid / D.qh, head = wid % D.qh;
  if (rows.status[r] != RUNNING_ST) return;
  const int npc = (reqs.P[rows.slot[r]] - 1 + pl.CH - 1) / pl.CH;
  const int nsc = (rows.ell[r] + 1 + pl.CH - 1) / pl.CH;
  const long long base = ((long long)r * D.qh + head) * pl.nslot;
  float M = -INFINITY;
  for (int c = 0; c < npc; ++c) M = fmaxf(M, part_lse[base + c]);
  for (int c = 0; c < nsc; ++c) M = fmaxf(M, part_lse[base + pl.npc_max + c]);
  float acc[HD / 32] = {};
  float L = 0.f;
  auto add = [&](int slot) {
    const float w = exp2f(part_lse[base + slot] - M);
    L += w;
#pragma unroll
    for (int i = 0; i < HD / 32; ++i) acc[i] += w * part_o[(base + slot) * HD + lane + 32 * i];
  };
  for (int c = 0; c < npc; ++c) add(c);
  for (int c = 0; c < nsc; ++c) add(pl.npc_max + c);
#pragma unroll
  for (int i = 0; i < HD / 32; ++i) {
    const float v = acc[i] / L;
    const long long oi = ((long long)r * D.qh + head) * HD + lane + 32 * i;
    out[oi] = __float2bfloat16_rn(v);
    if (dbg) dbg[oi] = v;
  }
}

// ------------------------------------------------------------------ per-window plan
// Units: prefix units first (type 1: group, chunk), then suffix units (type 0: row, chunk).
// Groups: the window's rows of one request in batch order, qr rows per group (cascade) or
// one row per group (flat mode).  Built once per window: rows only change at boundaries.
__global__ void __launch_bounds__(1024) k_attn_plan(Dims D, Rows rows, Reqs reqs, AttnPlan pl, int n, int flat) {
  const int tid = threadIdx.x;
  __shared__ int s_rank[1024], s_nrows[1024];
  const int qr = flat ? 1 : pl.qr_max;
  // rank of each row among the rows of its request (batch order); count at the leader
  for (int r = tid; r < n; r += 1024) {
    const int slot = rows.slot[r];
    int rank = 0, tot = 0;
    for (int r2 = 0; r2 < n; ++r2)
      if (rows.slot[r2] == slot) { rank += r2 < r; ++tot; }
    if (r < 1024) { s_rank[r] = rank; s_nrows[r] = tot; }
  }
  __syncthreads();
  if (tid == 0) {
    // groups in batch order of their leaders; prefix units; suffix units
    int ng = 0, nu = 0;
    for (int r = 0; r < n; ++r) {
      if (s_rank[r] != 0) continue;
      const int slot = rows.slot[r];
      const int npc = (reqs.P[slot] - 1 + pl.CH - 1) / pl.CH;
      const int ngr = (s_nrows[r] + qr - 1) / qr;
      for (int k = 0; k < ngr; ++k) {
        const int gi = ng + k;
        pl.grp_slot[gi] = slot;
        pl.grp_n[gi] = min(qr, s_nrows[r] - k * qr);
        for (int c = 0; c < npc; ++c) pl.units[nu++] = make_int4(1, gi, c, 0);
      }
      // rows of this request in batch order fill the groups
      int k = 0;
      for (int r2 = r; r2 < n; ++r2)
        if (rows.slot[r2] == slot) { pl.grp_rows[(ng + k / qr) * pl.qr_max + k % qr] = r2; ++k; }
      ng += ngr;
    }
    for (int r = 0; r < n; ++r) {
      const int maxlen = min(rows.ell[r] + D.T, D.cap);   // suffix length at the window's last step
      const int nsc = (maxlen + pl.CH - 1) / pl.CH;
      for (int c = 0; c < nsc; ++c) pl.units[nu++] = make_int4(0, r, c, 0);
    }
    *pl.n_units = nu;
  }
}

// algorithmic KV bytes of one step's attention (all layers): prefix once per request with a
// running row, each running suffix once, plus q and o (profiling only)
__global__ void __launch_bounds__(1024) k_attn_account(Dims D, Rows rows, Reqs reqs, AttnPlan pl, int n,
                                                       double* acc) {
  __shared__ double red[32];
  double b = 0.0;
  const double kvtok = 2.0 * D.kvh * D.hd * 2.0;   // K+V bytes per token per layer (bf16)
  for (int r = threadIdx.x; r < n; r += 1024) {
    if (rows.status[r] != RUNNING_ST) continue;
    b += (rows.ell[r] + 1) * kvtok + 2.0 * D.qh * D.hd * 2.0;
    // prefix once per request: counted at the lowest running row of the request
    bool first = true;
    for (int r2 = 0; r2 < r; ++r2)
      if (rows.slot[r2] == rows.slot[r] && rows.status[r2] == RUNNING_ST) { first = false; break; }
    if (first) b += (reqs.P[rows.slot[r]] - 1) * kvtok;
  }
  for (int o = 16; o > 0; o >>= 1) b += __shfl_xor_sync(0xffffffffu, b, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = b;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 32; ++w) t += red[w];
    *acc += t * D.L;
  }
}
}  // namespace

void launch_attn_plan(Dims D, Rows rows, Reqs reqs, AttnPlan pl, int n, int flat, cudaStream_t s) {
  k_attn_plan<<<1, 1024, 0, s>>>(D, rows, reqs, pl, n, flat);
}
void launch_attn_account(Dims D, Rows rows, Reqs reqs, AttnPlan pl, int n, double* acc, cudaStream_t s) {
  k_attn_account<<<1, 1024, 0, s>>>(D, rows, reqs, pl, n, acc);
}

static int g_sms = 0;
void launch_attn_cascade(const bf16* q, const bf16* pool, bf16* out, float* dbg, float* part_o, float* part_lse,
                         Dims D, int layer, Rows rows, Reqs reqs, AttnPlan pl, int n, cudaStream_t s) {
  if (n <= 0) return;
  if (!g_sms) cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, 0);
  if (D.hd == 128) {
    const size_t sm = sizeof(SmemA<128>);
    static bool a = false;
    if (!a) { cudaFuncSetAttribute(k_attn_cascade<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); a = true; }
    k_attn_cascade<128><<<g_sms, NTH, sm, s>>>(q, pool, part_o, part_lse, D, layer, rows, reqs, pl);
    k_attn_merge<128><<<(n * D.qh * 32 + 255) / 256, 256, 0, s>>>(part_o, part_lse, out, dbg, D, rows, reqs, pl, n);
  } else {
    const size_t sm = sizeof(SmemA<64>);
    static bool a = false;
    if (!a) { cudaFuncSetAttribute(k_attn_cascade<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); a = true; }
    k_attn_cascade<64><<<g_sms, NTH, sm, s>>>(q, pool, part_o, part_lse, D, layer, rows, reqs, pl);
    k_attn_merge<64><<<(n * D.qh * 32 + 255) / 256, 256, 0, s>>>(part_o, part_lse, out, dbg, D, rows, reqs, pl, n);
  }
}
