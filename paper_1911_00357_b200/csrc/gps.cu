// PointGoal GPS+Compass actor-critic (configs[1]): goal FC + action embedding -> GRU-512 -> head.
//
// P:L588-593 (App. C): goal [d, cos th, sin th] -> FC 32; 32-d embedding of the previous action
// (start token); recurrent policy; FC -> softmax over 4 actions + value.  PyTorch GRU
// conventions (gate rows r, z, n; n = tanh(W_in x + b_in + r*(W_hn h + b_hn))); the state is
// multiplied by mask_t (episode reset) before step t.
//
// B200 design.  The 128-step recurrence is a dependency chain: per step the whole work is a
// [1536 x 512] x [512 x B] matvec (B = 2 envs per minibatch), so it is latency-bound, not
// FLOP-bound.  One thread-block cluster of 16 CTAs (16 SMs) runs the whole sequence in a
// single persistent launch:
//   * CTA c owns hidden units [32c, 32c+32) and their 96 gate rows of W_hh, held for the whole
//     sequence in REGISTERS as fp16 (fwd) / bf16 (bwd, transposed) mma.sync A-fragments;
//   * per step each CTA multiplies its rows by h_{t-1} (m16n8k16, batch in the n dimension),
//     applies the gate nonlinearity for its own 32 units, and pushes the new h slice into every
//     CTA's shared memory through DSMEM (st.shared::cluster); one split cluster barrier per step
//     (arrive.release right after the DSMEM stores; the global stores of the saved activations
//     and the prefetch of the next step's inputs run while the barrier completes);
//   * the backward pass (BPTT) multiplies by W_hh^T: each CTA forms partial products over its
//     96 rows for all 512 hidden units and sends each 32-unit slice to its owner CTA, which sums
//     the 16 partials in fixed order (deterministic).
// Everything that is NOT on the dependency chain is hoisted out of the recurrence: the input
// projection W_ih x + b_ih for all steps (prologue of the forward kernel) and the weight
// gradients dW_hh = dG_h^T H_in, dW_ih = dG_x^T X, dX = dG_x W_ih (GEMMs after the recurrence),
// all reductions in fixed order.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <string.h>

#include "common.cuh"
#include "ppo_sample.cuh"

namespace {

constexpr int kH = 512, kG = 3 * kH, kIn = 64, kNC = 16, kUPC = kH / kNC /*32*/, kRows = 3 * kUPC /*96*/;
constexpr int kBMax = 8, kA1 = 5, kTMax = 1024, kU = 12;  // U: 9 used columns, padded to 12

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_arrive_release() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_wait_acquire() {
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  cluster_arrive_release();
  cluster_wait_acquire();
}
__device__ __forceinline__ uint32_t map_to_cta(const void* smem_ptr, uint32_t cta) {
  uint32_t a = (uint32_t)__cvta_generic_to_shared(smem_ptr), r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(cta));
  return r;
}
__device__ __forceinline__ void st_cluster_u16(uint32_t addr, uint16_t v) {
  asm volatile("st.shared::cluster.u16 [%0], %1;" ::"r"(addr), "h"(v) : "memory");
}
__device__ __forceinline__ void st_cluster_v2f32(uint32_t addr, float a, float b) {
  asm volatile("st.shared::cluster.v2.f32 [%0], {%1, %2};" ::"r"(addr), "f"(a), "f"(b) : "memory");
}
__device__ __forceinline__ void mma_f16(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void mma_bf16(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_f16(float lo, float hi) {
  __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ float sigmoidf_(float x) { return 1.f / (1.f + __expf(-x)); }
// Single-MUFU forms used on the recurrence's critical path (tanh.approx: ~2^-11 relative error,
// below the fp16 rounding of the broadcast state).
__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float sigmoid_fast(float x) { return fmaf(0.5f, tanh_fast(0.5f * x), 0.5f); }

// Debug-build phase trace of the forward recurrence (CTA 0, thread 0): clock64 at
// 0 = h_{t-1} received, 1 = W_hh h done, 2 = h_t sent.  Compiled out of the product library.
#ifdef DDPPO_TRACE
__device__ long long g_trace[8 * kTMax];
__device__ long long g_trace_b[8 * kTMax];
#define DDPPO_TRACE_POINT(c, tid, t, k) \
  if ((c) == 0 && (tid) == 0 && (t) < kTMax) g_trace[8 * (t) + (k)] = clock64();
#define DDPPO_TRACE_B(c, tid, t, k) \
  if ((c) == 0 && (tid) == 0 && (t) < kTMax) g_trace_b[8 * (t) + (k)] = clock64();
#else
#define DDPPO_TRACE_POINT(c, tid, t, k)
#define DDPPO_TRACE_B(c, tid, t, k)
#endif

// local gate row lr in [0,96) of CTA c -> global row of W (gate-major: r | z | n blocks of 512)
__device__ __forceinline__ int grow_of(int c, int lr) { return (lr / kUPC) * kH + c * kUPC + (lr % kUPC); }

struct GpsPtrs {
  // params
  const float *Wg, *bg, *Emb, *Wih, *Whh, *bih, *bhh, *Wo, *bo;
  // batch
  const float* goal;
  const int32_t* prev_action;
  const float* mask;
  const float* h0;
  const int32_t* env_idx;
  int B, T, ld, T_run;
  // workspace (sample s = b*T_run + t)
  float* X;      // [S][64]
  float* GI;     // [16][T_run][B][96]   CTA-local input projections (incl. b_ih)
  float* Hs;     // [S][512]  h_t
  float* Hin;    // [S][512]  mask_t * h_{t-1}
  float4* RZNG;  // [S][512]  (r, z, n, W_hn h_in + b_hn)
  float* dH;     // [S][512]  dL/dh_t from the head
  float* dGI;    // [S][1536]
  float* dGH;    // [S][1536]
  float* U;      // [S][9]     [goal, 1, onehot(prev_action)]
  float* Q;      // [1536][9]  dG_x^T U
  float* dbhh;   // [1536] b_hh gradient = sum_s dG_h[s], summed by the BPTT kernel (nullable)
  // fused head + PPO loss + head input gradient after the recurrence (learner runtime; on = 0: off)
  struct Loss {
    int on, use_vclip;
    const int32_t *len, *action;
    const float *logp_old, *value_old, *ret, *adv, *mean_invstd;
    float inv_n, eps, vclip_eps, c_v, c_e, n_valid;
    float *dlogits, *dvalues, *stats;
    int* err;
  } loss;
};

// ------------------------------------------------------------------ mbarrier / st.async helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init_cluster() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// The data arrives in this CTA's own shared memory through st.async ... complete_tx, whose
// completion on the local mbarrier makes it visible: the default (CTA-scope) acquire suffices.
// (A .cluster-scope acquire would make ptxas emit an L1 invalidate, CCTL.IVALL, on every poll.)
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void st_async_v4(uint32_t raddr, uint4 v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(raddr),
               "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void st_async_v2f(uint32_t raddr, float a, float b, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];" ::"r"(raddr),
               "f"(a), "f"(b), "r"(rbar)
               : "memory");
}

// ------------------------------------------------------------------ forward recurrence
// tcgen05 formulation (one CTA per 32 hidden units, 16-CTA cluster, 256 threads):
//  * A operand (TMEM, fp16, M = 128 lanes, K = 576 = 512 hidden + 64 input columns):
//      lanes  0..31  r rows: [W_hr | W_ir]     lanes 32..63  z rows: [W_hz | W_iz]
//      lanes 64..95  n rows: [W_hn | 0   ]     lanes 96..127 n rows: [0    | W_in]
//    so ONE accumulation gives r/z pre-activations (input + hidden parts) and the separate
//    W_hn h and W_in x the n gate needs -- the input projection rides on the same MMAs and no
//    per-step input projection is read from HBM;
//  * B operand (smem, fp16 canonical K-major, [16 env rows][576]): the hidden part is filled by
//    every CTA's st.async packets (8 units of one env = one 16-byte core-matrix row, complete_tx
//    on this CTA's mbarrier); the input part x_t = [goal_fc(goal_t), emb(prev_action_t)] is
//    computed locally one step ahead by the otherwise idle warps 4..7;
//  * per step warps 0..3 each issue 9 of the 36 tcgen05.mma (M=128, N=16, K=16) into their own
//    TMEM accumulator (issue cost spread over 4 sub-partitions), commit to one mbarrier, read the
//    four accumulators back (tcgen05.ld.32x32b) and the gate warps finish the GRU cell for the
//    CTA's 32 units, then push the new h slice.  No cluster barrier, no HBM read on the chain.
constexpr int kFwdThreads = 256;
constexpr int kKX = kH + kIn;                  // 576: K of the fused [h; x] operand
constexpr uint32_t kTileSBO = (kKX / 8) * 128; // 9216 B between 8-row groups of a [rows x 576] tile
constexpr int kAcc = 4;                        // MMA warps = independent accumulators
constexpr uint32_t kAccCol0 = kKX / 2;         // TMEM columns [0, 288): A operand (fp16 pairs)
constexpr int kTmemCols = 512;

__device__ __forceinline__ uint32_t ktile_off(int r, int k) {  // canonical K-major, K = 576
  return (uint32_t)((r >> 3) * kTileSBO + (k >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2);
}
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
// kind::f16, D f32, A f16, B f16, K-major, M = 128, N = 16
constexpr uint32_t kIdescF16_M128_N16 = (1u << 4) | (0u << 7) | (0u << 10) | ((16u >> 3) << 17) | ((128u >> 4) << 24);

struct FwdSmem {
  unsigned char h_tile[2][2 * kTileSBO];  // [h_{t-1}; x_t] (fp16) [16 env rows][576], by step parity
  float acc[128][kBMax];                  // the accumulator rows read back from TMEM
  float hown[kBMax][kUPC];                // fp32 state h_in for own units
  unsigned char stage[2][512];            // own new h slice [env][32 units] fp16, by step parity
  float bias[128];                        // r: b_ir+b_hr, z: b_iz+b_hz, n_h: b_hn, n_x: b_in
  float wg[32 * 3 + 32];                  // goal FC
  float emb[kA1 * 32];                    // action embedding
  uint64_t bar[2];                        // "h_tile[t%2] holds h_{t-1}" (tx-count barrier)
  uint64_t mma_bar;                       // "the accumulators hold W [h; x]"
  uint32_t tmem_slot;
};

// x_t for env b into the B tile (k = 512..575) and, from CTA 0, the X / U rows of sample s
__device__ __forceinline__ void fwd_input(const GpsPtrs& p, FwdSmem& sm, unsigned char* tile, int b, int j, int t,
                                          bool write_global) {
  const int n = p.env_idx[b];
  const int T_run = p.T_run;
  const float* gg = p.goal + ((size_t)n * p.T + t) * 3;
  const int act = p.prev_action[(size_t)n * p.ld + t];
  float x;
  if (j < 32) x = sm.wg[j * 3 + 0] * gg[0] + sm.wg[j * 3 + 1] * gg[1] + sm.wg[j * 3 + 2] * gg[2] + sm.wg[96 + j];
  else x = sm.emb[act * 32 + (j - 32)];
  *reinterpret_cast<__half*>(tile + ktile_off(b, kH + j)) = __float2half(x);
  if (write_global) {
    const size_t s = (size_t)b * T_run + t;
    p.X[s * kIn + j] = x;
    if (j < kU) {
      float u;
      if (j < 3) u = gg[j];
      else if (j == 3) u = 1.f;
      else if (j < 9) u = (act == j - 4) ? 1.f : 0.f;
      else u = 0.f;
      p.U[s * kU + j] = u;
    }
  }
}

__global__ void __launch_bounds__(kFwdThreads, 1) gps_gru_fwd_kernel(GpsPtrs p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  FwdSmem& sm = *reinterpret_cast<FwdSmem*>(smem_raw);
  float* smask = reinterpret_cast<float*>(smem_raw + sizeof(FwdSmem));  // [B][T_run]
  const int c = (int)cluster_ctarank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int B = p.B, T_run = p.T_run, S = B * T_run;
  DDPPO_TRACE_POINT(c, tid, kTMax - 1, 5);

  // ---- prologue: operand tiles, biases, masks, barriers, TMEM
  {
    uint4* zz = reinterpret_cast<uint4*>(sm.h_tile);
    for (int i = tid; i < (int)(sizeof(sm.h_tile) / 16); i += blockDim.x) zz[i] = make_uint4(0u, 0u, 0u, 0u);
    uint4* zs = reinterpret_cast<uint4*>(sm.stage);
    for (int i = tid; i < (int)(sizeof(sm.stage) / 16); i += blockDim.x) zs[i] = make_uint4(0u, 0u, 0u, 0u);
  }
  for (int i = tid; i < 128; i += blockDim.x) {
    float bsum;
    if (i < 64) bsum = p.bih[grow_of(c, i)] + p.bhh[grow_of(c, i)];
    else if (i < 96) bsum = p.bhh[grow_of(c, i)];
    else bsum = p.bih[grow_of(c, i - 32)];
    sm.bias[i] = bsum;
  }
  for (int i = tid; i < 128; i += blockDim.x) sm.wg[i] = i < 96 ? p.Wg[i] : p.bg[i - 96];
  for (int i = tid; i < kA1 * 32; i += blockDim.x) sm.emb[i] = p.Emb[i];
  for (int i = tid; i < S; i += blockDim.x) {
    const int b = i / T_run, t = i - b * T_run;
    smask[i] = p.mask[(size_t)p.env_idx[b] * p.ld + t];
  }
  if (tid == 0) {
    mbar_init(&sm.bar[0], 1);
    mbar_init(&sm.bar[1], 1);
    mbar_init(&sm.mma_bar, kAcc);  // one tcgen05.commit per MMA warp
    fence_mbar_init_cluster();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sm.tmem_slot)),
                 "n"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = sm.tmem_slot;
  // A operand -> TMEM.  Warp w and w+4 share lane quarter w%4 (row r = 32(w%4) + lane) and split
  // the 288 packed columns: 8 columns (16 weights) per tcgen05.st.32x32b.x8.
  {
    const int r = (warp & 3) * 32 + lane;
    const int gate_row = r < 96 ? r : r - 32;  // n_x rows reuse the n rows' input weights
    const float* wh = p.Whh + (size_t)grow_of(c, gate_row) * kH;
    const float* wi = p.Wih + (size_t)grow_of(c, gate_row) * kIn;
    const bool has_h = r < 96, has_x = r < 64 || r >= 96;
    const int col_lo = (warp < 4) ? 0 : kAccCol0 / 2;
#pragma unroll 1
    for (int col0 = col_lo; col0 < col_lo + (int)kAccCol0 / 2; col0 += 48) {
      float4 a[24];  // 96 weights = 48 columns: all loads in flight before any conversion
#pragma unroll
      for (int q = 0; q < 24; ++q) {
        const int k = 2 * col0 + 4 * q;
        a[q] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (k < kH) {
          if (has_h) a[q] = *reinterpret_cast<const float4*>(wh + k);
        } else if (has_x) {
          a[q] = *reinterpret_cast<const float4*>(wi + (k - kH));
        }
      }
#pragma unroll
      for (int sblk = 0; sblk < 6; ++sblk) {  // 8 columns per tcgen05.st
        uint32_t v[8];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          v[2 * q] = pack_f16(a[4 * sblk + q].x, a[4 * sblk + q].y);
          v[2 * q + 1] = pack_f16(a[4 * sblk + q].z, a[4 * sblk + q].w);
        }
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(
                         tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(col0 + 8 * sblk)),
                     "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                     : "memory");
      }
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  // initial B tile: h_in_0 = mask_0 * h0 and x_0
  for (int i = tid; i < B * kH; i += blockDim.x) {
    const int b = i / kH, k = i % kH;
    const float h = smask[b * T_run] * p.h0[(size_t)p.env_idx[b] * kH + k];
    *reinterpret_cast<__half*>(sm.h_tile[0] + ktile_off(b, k)) = __float2half(h);
    if (k >= c * kUPC && k < (c + 1) * kUPC) sm.hown[b][k - c * kUPC] = h;
  }
  for (int i = tid; i < B * kIn; i += blockDim.x) fwd_input(p, sm, sm.h_tile[0], i / kIn, i % kIn, 0, c == 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> tensor core
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();  // barriers and tiles initialised everywhere before any remote write
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  DDPPO_TRACE_POINT(c, tid, kTMax - 1, 6);
  DDPPO_TRACE_POINT(c, tid, kTMax - 1, 7);

  // ---- recurrence
  const int gu = lane, gb = warp;  // gate thread: warp b handles env b of the minibatch, lane = unit
  const bool gate_warp = warp < B;
  // st.async packet of this lane: units [8*(lane%4), +8) of env gb (one 16-byte core-matrix row of
  // the peers' B tiles) to CTAs lane/4 and lane/4+8.  (Measured: 128 such packets per step beat
  // 16 cp.async.bulk copies of the whole 512-byte slice -- the bulk path's fixed latency is higher.)
  uint32_t pk_addr[2] = {0u, 0u}, pk_bar[2][2] = {{0u, 0u}, {0u, 0u}};
  const uint32_t tx_bytes = (uint32_t)(kNC * B * kUPC * sizeof(__half));
  if (gate_warp) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const uint32_t q = (uint32_t)(lane / 4 + 8 * j);
      pk_addr[j] = map_to_cta(sm.h_tile[0] + ktile_off(gb, c * kUPC + 8 * (lane % 4)), q);
      pk_bar[j][0] = map_to_cta(&sm.bar[0], q);
      pk_bar[j][1] = map_to_cta(&sm.bar[1], q);
    }
  }
  const uint32_t h_parity_bytes = (uint32_t)sizeof(sm.h_tile[0]);
  const uint32_t h_base0 = smem_u32(sm.h_tile[0]);
  for (int t = 0; t < T_run; ++t) {
    const int cur = t & 1;
    if (warp < kAcc) {  // MMA warps: warp a owns accumulator a and K steps kk = a, a+kAcc, ...;
      // converged warps with warp-uniform operands, one elected lane issues
      if (t > 0) {
        if (tid == 0) mbar_arrive_expect_tx(&sm.bar[cur], tx_bytes);
        mbar_wait_parity(&sm.bar[cur], (uint32_t)(((t - 1) >> 1) & 1));
      }
      DDPPO_TRACE_POINT(c, tid, t, 0);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint64_t bd0 = umma_desc(h_base0 + (uint32_t)cur * h_parity_bytes, 128, kTileSBO);
      const uint32_t d_acc = tmem + kAccCol0 + 16u * (uint32_t)warp;
      // descriptor of K step kk = bd0 + 16*kk (start address advances 256 B); A columns 8*kk
#pragma unroll
      for (int j = 0; j < kKX / 16 / kAcc; ++j) {
        const int kk = warp + kAcc * j;
        asm volatile(
            "{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_acc),
            "r"(tmem + 8u * (uint32_t)kk), "l"(bd0 + (uint64_t)(16 * kk)), "r"(kIdescF16_M128_N16),
            "r"((uint32_t)j)
            : "memory");
      }
      asm volatile(
          "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
          "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(
              smem_u32(&sm.mma_bar))
          : "memory");
      DDPPO_TRACE_POINT(c, tid, t, 3);
      mbar_wait_parity(&sm.mma_bar, (uint32_t)(t & 1));
      DDPPO_TRACE_POINT(c, tid, t, 4);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      uint32_t v[kAcc][8];
#pragma unroll
      for (int a = 0; a < kAcc; ++a)
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                     : "=r"(v[a][0]), "=r"(v[a][1]), "=r"(v[a][2]), "=r"(v[a][3]), "=r"(v[a][4]), "=r"(v[a][5]),
                       "=r"(v[a][6]), "=r"(v[a][7])
                     : "r"(tmem + ((uint32_t)(warp * 32) << 16) + kAccCol0 + 16u * (uint32_t)a));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      DDPPO_TRACE_POINT(c, tid, t, 5);
      float s8[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        float acc = 0.f;
#pragma unroll
        for (int a = 0; a < kAcc; ++a) acc += __uint_as_float(v[a][e]);
        s8[e] = acc;
      }
      const int row = warp * 32 + lane;
      *reinterpret_cast<float4*>(&sm.acc[row][0]) = make_float4(s8[0], s8[1], s8[2], s8[3]);
      *reinterpret_cast<float4*>(&sm.acc[row][4]) = make_float4(s8[4], s8[5], s8[6], s8[7]);
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    } else if (t + 1 < T_run) {
      // warps 4..7: x_{t+1} into the other B tile (its last reader, the MMAs of step t-1, are done)
      for (int i = tid - kAcc * 32; i < B * kIn; i += blockDim.x - kAcc * 32)
        fwd_input(p, sm, sm.h_tile[cur ^ 1], i / kIn, i % kIn, t + 1, c == 0);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    DDPPO_TRACE_POINT(c, tid, t, 1);
    if (gate_warp) {
      const int lr_r = gu, lr_z = kUPC + gu, lr_nh = 2 * kUPC + gu, lr_nx = 3 * kUPC + gu;
      const float pre_r = sm.acc[lr_r][gb] + sm.bias[lr_r];
      const float pre_z = sm.acc[lr_z][gb] + sm.bias[lr_z];
      const float gh_n = sm.acc[lr_nh][gb] + sm.bias[lr_nh];
      const float gi_n = sm.acc[lr_nx][gb] + sm.bias[lr_nx];
      const float h_in = sm.hown[gb][gu];
      const float r = sigmoid_fast(pre_r);
      const float z = sigmoid_fast(pre_z);
      const float nn = tanh_fast(gi_n + r * gh_n);
      const float h = (1.f - z) * nn + z * h_in;
      if (t + 1 < T_run) {
        const float hn = smask[gb * T_run + t + 1] * h;
        sm.hown[gb][gu] = hn;
        __half* st = reinterpret_cast<__half*>(sm.stage[cur]) + gb * kUPC;
        st[gu] = __float2half(hn);
        __syncwarp();
        const uint4 pkt = *reinterpret_cast<const uint4*>(st + 8 * (lane % 4));
        const uint32_t off = (cur ^ 1) * h_parity_bytes;
        st_async_v4(pk_addr[0] + off, pkt, pk_bar[0][cur ^ 1]);
        st_async_v4(pk_addr[1] + off, pkt, pk_bar[1][cur ^ 1]);
      }
      DDPPO_TRACE_POINT(c, tid, t, 2);
      // off the chain: save activations for the head and the backward pass
      const size_t o = ((size_t)gb * T_run + t) * kH + c * kUPC + gu;
      p.Hs[o] = h;
      p.Hin[o] = h_in;
      p.RZNG[o] = make_float4(r, z, nn, gh_n);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();  // no CTA exits while a peer could still address its shared memory
  if (p.loss.on) {
    // ---- fused head + PPO loss + head input gradient (a5 head, a6): the cluster barrier above made
    // every CTA's h_t rows visible; warp per sample over the cluster's 128 warps: logits / value =
    // W_o h + b_o, the sample's loss gradient (ppo_sample), dH = W_o^T [dlogits; dvalue]; loss
    // statistics summed per CTA, then over the 16 CTAs in CTA order (DSMEM) -- deterministic.
    float* wo = reinterpret_cast<float*>(sm.h_tile);  // [5][512] + b_o (the B tiles are free now)
    double* red = reinterpret_cast<double*>(sm.h_tile[1]);      // block_sum scratch [6][8]
    double* cta_part = red + 64;                                   // this CTA's 6 sums
    for (int i = tid; i < 5 * kH; i += blockDim.x) wo[i] = p.Wo[i];
    if (tid < 5) wo[5 * kH + tid] = p.bo[tid];
    __syncthreads();
    const auto& L = p.loss;
    float mu = 0.f, invstd = 1.f;
    if (L.mean_invstd) {
      mu = L.mean_invstd[0];
      invstd = L.mean_invstd[1];
    }
    double acc[6] = {0, 0, 0, 0, 0, 0};
    const int M = B * T_run;
    for (int m = c * (kFwdThreads / 32) + warp; m < M; m += kNC * (kFwdThreads / 32)) {
      const int b = m / T_run, t = m - b * T_run;
      const int n = p.env_idx[b];
      const float* h = p.Hs + (size_t)m * kH;
      float hv[kH / 32];
      float out[5] = {0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int i = 0; i < kH / 32; ++i) {
        hv[i] = h[lane + 32 * i];
#pragma unroll
        for (int o = 0; o < 5; ++o) out[o] += wo[o * kH + lane + 32 * i] * hv[i];
      }
#pragma unroll
      for (int o = 0; o < 5; ++o) out[o] = warp_sum(out[o]) + wo[5 * kH + o];
      float4 dz = make_float4(0.f, 0.f, 0.f, 0.f);
      float dv = 0.f;
      if (t < L.len[n]) {  // (warp-uniform)
        const size_t s = (size_t)n * p.ld + t;
        const float A = L.mean_invstd ? (L.adv[s] - mu) * invstd : L.adv[s];
        const SampleOut o = ppo_sample(make_float4(out[0], out[1], out[2], out[3]), out[4], L.action[s], L.logp_old[s],
                                       L.value_old[s], L.ret[s], A, L.inv_n, L.eps, L.vclip_eps, L.c_v, L.c_e,
                                       L.use_vclip);
        dz = o.dz;
        dv = o.dv;
        if (lane == 0) {
          acc[0] += (double)o.surr;
          acc[1] += (double)o.lv;
          acc[2] += (double)o.H;
          acc[3] += (double)o.clipped;
          acc[4] += (double)o.kl;
        }
      }
      if (lane == 0) {
        *reinterpret_cast<float4*>(L.dlogits + (size_t)m * 4) = dz;
        L.dvalues[m] = dv;
      }
      float* dh = p.dH + (size_t)m * kH;
#pragma unroll
      for (int i = 0; i < kH / 32; ++i) {
        const int k = lane + 32 * i;
        dh[k] = wo[k] * dz.x + wo[kH + k] * dz.y + wo[2 * kH + k] * dz.z + wo[3 * kH + k] * dz.w + wo[4 * kH + k] * dv;
      }
    }
    block_sum<6>(acc, red);
    if (tid == 0)
#pragma unroll
      for (int i = 0; i < 6; ++i) cta_part[i] = acc[i];
    cluster_sync_all();  // every CTA's sums are in place
    if (c == 0 && tid == 0) {
      double fin[6] = {0, 0, 0, 0, 0, 0};
      for (int j = 0; j < kNC; ++j) {
        const uint32_t ra = map_to_cta(cta_part, (uint32_t)j);
#pragma unroll
        for (int i = 0; i < 6; ++i) {
          double v;
          asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(ra + 8u * (uint32_t)i) : "memory");
          fin[i] += v;
        }
      }
      write_stats(fin, L.inv_n, L.c_v, L.c_e, L.n_valid, L.stats, L.err);
    }
    cluster_sync_all();  // CTA 0 has read every peer's sums
  }
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols) : "memory");
}

// ------------------------------------------------------------------ backward recurrence (BPTT)
// tcgen05 formulation.  Iteration i (t = T_run-1-i):
//  * gate warps (warp b = env b, lane = unit) form dG for the CTA's 32 units (local) and write
//    dG_h into the B operand tile (bf16 canonical K-major [16 env rows][96 own gate rows]);
//  * warps 0..3 each issue the 6 tcgen05.mma (M=128 hidden units, N=16, K=16) of one 128-unit
//    tile of W_hh^T (A operand resident in TMEM for the whole sequence, bf16), commit, read the
//    four tiles' lanes they own back with tcgen05.ld and st.async each unit's partial to the
//    unit's owner CTA (complete_tx on its mbarrier);
//  * the owner sums the 16 partials in CTA order (deterministic) -> dL/dh_{t-1}.
constexpr int kBwdThreads = 256;
constexpr uint32_t kDgSBO = (kRows / 8) * 128;  // 1536 B between 8-row groups of the [16 x 96] tile
constexpr uint32_t kBwdD0 = 4 * (kRows / 2);    // TMEM columns [0, 192): 4 tiles x 48 packed columns
constexpr int kBwdTmemCols = 512;  // A (192) + 8 accumulators x 16
// kind::f16, D f32, A bf16, B bf16, K-major, M = 128, N = 16
constexpr uint32_t kIdescBF16_M128_N16 = (1u << 4) | (1u << 7) | (1u << 10) | ((16u >> 3) << 17) | ((128u >> 4) << 24);

struct BwdSmem {
  unsigned char dg_tile[2 * kDgSBO];      // dG_h (bf16) [16 env rows][96 own rows], canonical layout
  float recv[2][kNC][kUPC][kBMax];        // partial W_hh^T dG_h from every CTA, by iteration parity
  uint64_t bar[2];                        // recv[i%2] complete (tx-count)
  uint64_t mma_bar;
  uint32_t tmem_slot;
};

__device__ __forceinline__ uint32_t dg_off(int n, int k) {
  return (uint32_t)((n >> 3) * kDgSBO + (k >> 3) * 128 + (n & 7) * 16 + (k & 7) * 2);
}

__global__ void __launch_bounds__(kBwdThreads, 1) gps_gru_bwd_kernel(GpsPtrs p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  BwdSmem& sm = *reinterpret_cast<BwdSmem*>(smem_raw);
  float* smask = reinterpret_cast<float*>(smem_raw + sizeof(BwdSmem));  // [B][T_run]
  const int c = (int)cluster_ctarank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int B = p.B, T_run = p.T_run, S = B * T_run;
  DDPPO_TRACE_B(c, tid, kTMax - 1, 6);

  {
    uint4* zz = reinterpret_cast<uint4*>(sm.dg_tile);
    for (int i = tid; i < (int)(sizeof(sm.dg_tile) / 16); i += blockDim.x) zz[i] = make_uint4(0u, 0u, 0u, 0u);
  }
  for (int i = tid; i < S; i += blockDim.x) {
    const int b = i / T_run, t = i - b * T_run;
    smask[i] = p.mask[(size_t)p.env_idx[b] * p.ld + t];
  }
  if (tid == 0) {
    mbar_init(&sm.bar[0], 1);
    mbar_init(&sm.bar[1], 1);
    mbar_init(&sm.mma_bar, 8);  // one commit per warp
    fence_mbar_init_cluster();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sm.tmem_slot)),
                 "n"(kBwdTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = sm.tmem_slot;
  // A operand -> TMEM: tile q (hidden units 128q..128q+127), lane = unit, 48 packed columns of the
  // 96 own gate rows: A_q[j][lr] = W_hh[grow(c, lr)][128q + j].  Warps w, w+4 share lane quarter
  // w%4 and split the 4 tiles; loads are coalesced across the warp (consecutive units).
  {
    const int jl = (warp & 3) * 32 + lane;
#pragma unroll 1
    for (int q = (warp < 4 ? 0 : 2); q < (warp < 4 ? 2 : 4); ++q) {
      const float* wcol = p.Whh + 128 * q + jl;
#pragma unroll 1
      for (int lr0 = 0; lr0 < kRows; lr0 += 48) {
        float w[48];
#pragma unroll
        for (int e = 0; e < 48; ++e) w[e] = wcol[(size_t)grow_of(c, lr0 + e) * kH];
#pragma unroll
        for (int sblk = 0; sblk < 3; ++sblk) {
          uint32_t v[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) v[e] = pack_bf16(w[16 * sblk + 2 * e], w[16 * sblk + 2 * e + 1]);
          asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(
                           tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(48 * q + lr0 / 2 + 8 * sblk)),
                       "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                       : "memory");
        }
      }
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  // destinations of this thread's partials: unit j = 128q + 32w + lane is owned by CTA 4q + w;
  // recv is [parity][src CTA][32 units][ustride floats] with ustride = B rounded to 2 / 4 / 8
  const uint32_t unit_bytes = B <= 2 ? 8u : (B <= 4 ? 16u : 32u);
  const int ustride = (int)unit_bytes / 4;
  // Warp w reads lane quarter w%4 of tiles q = 2*(w/4), 2*(w/4)+1 (units 128q + 32(w%4) + lane).
  uint32_t dst[2] = {0u, 0u}, dbar[2][2] = {{0u, 0u}, {0u, 0u}};
#pragma unroll
  for (int qi = 0; qi < 2; ++qi) {
    const int q = 2 * (warp >> 2) + qi;
    const uint32_t owner = (uint32_t)(4 * q + (warp & 3));
    dst[qi] = map_to_cta(&sm.recv[0][0][0][0] + (c * kUPC + lane) * ustride, owner);
    dbar[qi][0] = map_to_cta(&sm.bar[0], owner);
    dbar[qi][1] = map_to_cta(&sm.bar[1], owner);
  }
  const uint32_t recv_parity_bytes = (uint32_t)sizeof(sm.recv[0]);
  const uint32_t tx_bytes = (uint32_t)kNC * kUPC * unit_bytes;
  const uint32_t dg_base = smem_u32(sm.dg_tile);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

  const int gu = lane, gb = warp;
  const bool gate_warp = warp < B;
  float carry = 0.f;  // dL/dh_t flowing back from step t+1 (already multiplied by mask_{t+1})
  float sum_r = 0.f, sum_z = 0.f, sum_n = 0.f;  // this (env, unit)'s dG_h summed over t (-> b_hh grad)
  float dH_t = 0.f, h_in = 0.f;
  float4 rzng = make_float4(0.f, 0.f, 0.f, 0.f);
  if (gate_warp) {
    const size_t o = ((size_t)gb * T_run + T_run - 1) * kH + c * kUPC + gu;
    dH_t = p.dH[o];
    rzng = p.RZNG[o];
    h_in = p.Hin[o];
  }
  DDPPO_TRACE_B(c, tid, kTMax - 1, 7);
  for (int it = 0; it < T_run; ++it) {
    const int t = T_run - 1 - it, par = it & 1;
    DDPPO_TRACE_B(c, tid, it, 0);
    float dzh = 0.f;
    if (gate_warp) {
      const float dh = dH_t + carry;
      const float r = rzng.x, z = rzng.y, nn = rzng.z, ghn = rzng.w;
      const float dn = dh * (1.f - z);
      const float dz = dh * (h_in - nn);
      const float dn_pre = dn * (1.f - nn * nn);
      const float dr = dn_pre * ghn;
      const float dr_pre = dr * r * (1.f - r);
      const float dz_pre = dz * z * (1.f - z);
      *reinterpret_cast<__nv_bfloat16*>(sm.dg_tile + dg_off(gb, gu)) = __float2bfloat16(dr_pre);
      *reinterpret_cast<__nv_bfloat16*>(sm.dg_tile + dg_off(gb, kUPC + gu)) = __float2bfloat16(dz_pre);
      *reinterpret_cast<__nv_bfloat16*>(sm.dg_tile + dg_off(gb, 2 * kUPC + gu)) = __float2bfloat16(dn_pre * r);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      dzh = dh * z;
      // off the chain: save dG, prefetch step t-1
      const size_t og = ((size_t)gb * T_run + t) * kG + c * kUPC + gu;
      p.dGI[og] = dr_pre;
      p.dGI[og + kH] = dz_pre;
      p.dGI[og + 2 * kH] = dn_pre;
      p.dGH[og] = dr_pre;
      p.dGH[og + kH] = dz_pre;
      p.dGH[og + 2 * kH] = dn_pre * r;
      sum_r += dr_pre;
      sum_z += dz_pre;
      sum_n += dn_pre * r;
      if (t > 0) {
        const size_t o = ((size_t)gb * T_run + t - 1) * kH + c * kUPC + gu;
        dH_t = p.dH[o];
        rzng = p.RZNG[o];
        h_in = p.Hin[o];
      }
    }
    __syncthreads();
    DDPPO_TRACE_B(c, tid, it, 1);
    {
      // all 8 warps: warp w issues the 3 K steps 3h..3h+2 (h = w/4) of tile q = w%4 into its own
      // accumulator D[q][h]; then reads D[q'][0] + D[q'][1] of its lane quarter for 2 tiles q'
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int q_mma = warp & 3, h = warp >> 2;
      const uint64_t bd0 = umma_desc(dg_base, 128, kDgSBO);
      const uint32_t d_q = tmem + kBwdD0 + 16u * (uint32_t)(2 * q_mma + h);
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const int kk = 3 * h + j;
        asm volatile(
            "{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_q),
            "r"(tmem + 48u * (uint32_t)q_mma + 8u * (uint32_t)kk), "l"(bd0 + (uint64_t)(16 * kk)),
            "r"(kIdescBF16_M128_N16), "r"((uint32_t)j)
            : "memory");
      }
      asm volatile(
          "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
          "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(
              smem_u32(&sm.mma_bar))
          : "memory");
      DDPPO_TRACE_B(c, tid, it, 2);
      mbar_wait_parity(&sm.mma_bar, (uint32_t)(it & 1));
      DDPPO_TRACE_B(c, tid, it, 3);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t lane_base = tmem + ((uint32_t)((warp & 3) * 32) << 16) + kBwdD0;
      const uint32_t off = (uint32_t)par * recv_parity_bytes;
#pragma unroll
      for (int qi = 0; qi < 2; ++qi) {
        const int q = 2 * (warp >> 2) + qi;
        uint32_t a[8], b[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                     : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]), "=r"(a[4]), "=r"(a[5]), "=r"(a[6]),
                       "=r"(a[7])
                     : "r"(lane_base + 32u * (uint32_t)q));
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                     : "=r"(b[0]), "=r"(b[1]), "=r"(b[2]), "=r"(b[3]), "=r"(b[4]), "=r"(b[5]), "=r"(b[6]),
                       "=r"(b[7])
                     : "r"(lane_base + 32u * (uint32_t)q + 16u));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        float s[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) s[e] = __uint_as_float(a[e]) + __uint_as_float(b[e]);
        if (unit_bytes == 8u) {  // B <= 2: lane pairs send units (l, l+1) as one 16-byte packet
          const float n0 = __shfl_down_sync(0xffffffffu, s[0], 1);
          const float n1 = __shfl_down_sync(0xffffffffu, s[1], 1);
          if ((lane & 1) == 0)
            st_async_v4(dst[qi] + off,
                        make_uint4(__float_as_uint(s[0]), __float_as_uint(s[1]), __float_as_uint(n0),
                                   __float_as_uint(n1)),
                        dbar[qi][par]);
        } else {
          st_async_v4(dst[qi] + off,
                      make_uint4(__float_as_uint(s[0]), __float_as_uint(s[1]), __float_as_uint(s[2]),
                                 __float_as_uint(s[3])),
                      dbar[qi][par]);
          if (unit_bytes == 32u)
            st_async_v4(dst[qi] + off + 16u,
                        make_uint4(__float_as_uint(s[4]), __float_as_uint(s[5]), __float_as_uint(s[6]),
                                   __float_as_uint(s[7])),
                        dbar[qi][par]);
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    }
    DDPPO_TRACE_B(c, tid, it, 4);
    if (gate_warp) {
      if (tid == 0) mbar_arrive_expect_tx(&sm.bar[par], tx_bytes);
      mbar_wait_parity(&sm.bar[par], (uint32_t)((it >> 1) & 1));
      DDPPO_TRACE_B(c, tid, it, 5);
      float s = 0.f;
#pragma unroll
      for (int q = 0; q < kNC; ++q) s += (&sm.recv[par][0][0][0])[(q * kUPC + gu) * ustride + gb];
      carry = smask[gb * T_run + t] * (dzh + s);
    }
    __syncthreads();  // the MMAs of this iteration (done: mma_bar) are the last readers of dg_tile
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();  // no CTA exits while a peer could still address its shared memory
  if (p.dbhh) {
    // b_hh gradient of the CTA's 96 gate rows: per (env, unit) sums over t, then over envs in order
    // (the receive buffers are free: every peer has left the recurrence)
    float* red = &sm.recv[0][0][0][0];  // [B][96]
    if (gate_warp) {
      red[gb * kRows + gu] = sum_r;
      red[gb * kRows + kUPC + gu] = sum_z;
      red[gb * kRows + 2 * kUPC + gu] = sum_n;
    }
    __syncthreads();
    if (tid < kRows) {
      float a = 0.f;
      for (int b = 0; b < B; ++b) a += red[b * kRows + tid];
      p.dbhh[(tid / kUPC) * kH + c * kUPC + tid % kUPC] = a;
    }
  }
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kBwdTmemCols) : "memory");
}

// ------------------------------------------------------------------ head (Linear(512, 5)) fwd/bwd
__global__ void head_fwd_kernel(const float* __restrict__ Wo, const float* __restrict__ bo, const float* __restrict__ Hs,
                                int S, int H, float* __restrict__ logits, float* __restrict__ values) {
  const int warps = blockDim.x >> 5, lane = threadIdx.x & 31;
  for (int s = blockIdx.x * warps + (threadIdx.x >> 5); s < S; s += gridDim.x * warps) {
    const float* h = Hs + (size_t)s * H;
    float acc[kA1] = {0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll 4
    for (int k = 4 * lane; k < H; k += 128) {  // H % 128 == 0: float4 per lane, all loads independent
      const float4 hv = *reinterpret_cast<const float4*>(h + k);
#pragma unroll
      for (int o = 0; o < kA1; ++o) {
        const float4 w = *reinterpret_cast<const float4*>(Wo + o * H + k);
        acc[o] += w.x * hv.x + w.y * hv.y + w.z * hv.z + w.w * hv.w;
      }
    }
#pragma unroll
    for (int o = 0; o < kA1; ++o) acc[o] = warp_sum(acc[o]);
    if (lane == 0) {
      *reinterpret_cast<float4*>(logits + (size_t)s * 4) =
          make_float4(acc[0] + bo[0], acc[1] + bo[1], acc[2] + bo[2], acc[3] + bo[3]);
      values[s] = acc[4] + bo[4];
    }
  }
}

// dH[s][k] = sum_o Wo[o][k] dout[s][o]
__global__ void head_dgrad_kernel(const float* __restrict__ Wo, const float* __restrict__ dlogits,
                                  const float* __restrict__ dvalues, int S, int H, float* __restrict__ dH) {
  const size_t n = (size_t)S * H;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int s = (int)(i / H), k = (int)(i % H);
    const float4 dl = *reinterpret_cast<const float4*>(dlogits + (size_t)s * 4);
    dH[i] = Wo[k] * dl.x + Wo[H + k] * dl.y + Wo[2 * H + k] * dl.z + Wo[3 * H + k] * dl.w +
            Wo[4 * H + k] * dvalues[s];
  }
}

// Fixed-order column reductions: 32 columns per CTA x 8 sample chunks (one warp each), chunk
// partials summed in chunk order.   out[m] = sum_s A[s][m]  (and, for the head, weighted sums).
constexpr int kRedChunks = 8;
__global__ void __launch_bounds__(256) colsum_kernel(const float* __restrict__ A, int lda, int S, int M,
                                                     float* __restrict__ out) {
  __shared__ float part[kRedChunks][32];
  const int m = blockIdx.x * 32 + (threadIdx.x & 31), q = threadIdx.x >> 5;
  const int per = (S + kRedChunks - 1) / kRedChunks;
  float a = 0.f;
  if (m < M)
#pragma unroll 8
    for (int s = q * per; s < min(S, (q + 1) * per); ++s) a += A[(size_t)s * lda + m];
  part[q][threadIdx.x & 31] = a;
  __syncthreads();
  if (threadIdx.x < 32 && m < M) {
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < kRedChunks; ++i) t += part[i][threadIdx.x];
    out[m] = t;
  }
}

// dWo[o][k] = sum_s dout[s][o] Hs[s][k] (32 k per CTA x 8 sample chunks); CTA 0 also does dbo.
__global__ void __launch_bounds__(256) head_wgrad_kernel(const float* __restrict__ Hs,
                                                         const float* __restrict__ dlogits,
                                                         const float* __restrict__ dvalues, int S, int H,
                                                         float* __restrict__ dWo, float* __restrict__ dbo) {
  __shared__ float part[kRedChunks][kA1][33];
  const int kk = threadIdx.x & 31, q = threadIdx.x >> 5, k = blockIdx.x * 32 + kk;
  const int per = (S + kRedChunks - 1) / kRedChunks;
  float a[kA1] = {0.f, 0.f, 0.f, 0.f, 0.f}, bsum[kA1] = {0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll 8
  for (int s = q * per; s < min(S, (q + 1) * per); ++s) {
    const float h = Hs[(size_t)s * H + k];
    const float4 dl = *reinterpret_cast<const float4*>(dlogits + (size_t)s * 4);
    const float dv = dvalues[s];
    a[0] += dl.x * h;
    a[1] += dl.y * h;
    a[2] += dl.z * h;
    a[3] += dl.w * h;
    a[4] += dv * h;
    bsum[0] += dl.x;
    bsum[1] += dl.y;
    bsum[2] += dl.z;
    bsum[3] += dl.w;
    bsum[4] += dv;
  }
#pragma unroll
  for (int o = 0; o < kA1; ++o) part[q][o][kk] = a[o];
  __syncthreads();
  if (threadIdx.x < 32) {
#pragma unroll
    for (int o = 0; o < kA1; ++o) {
      float t = 0.f;
#pragma unroll
      for (int i = 0; i < kRedChunks; ++i) t += part[i][o][kk];
      dWo[o * H + k] = t;
    }
  }
  if (blockIdx.x == 0) {  // biases: chunk partials (identical for every kk) in chunk order
    __syncthreads();
    if (kk == 0) {
#pragma unroll
      for (int o = 0; o < kA1; ++o) part[q][o][32] = bsum[o];
    }
    __syncthreads();
    if (threadIdx.x < kA1) {
      float t = 0.f;
      for (int i = 0; i < kRedChunks; ++i) t += part[i][threadIdx.x][32];
      dbo[threadIdx.x] = t;
    }
  }
}

// Input-layer gradients from Q = dG_x^T U (U = [goal, 1, onehot(prev_action)] per sample):
//   dW_goal[j][c] = sum_row W_ih[row][j] Q[row][c]   (c < 3),  db_goal[j] = ... Q[row][3]
//   dEmb[a][j]    = sum_row W_ih[row][32+j] Q[row][4+a],      db_ih[row] = Q[row][3]
// (chain rule through x = [goal_fc(goal), emb(prev_action)]).  Block j reduces its
// 1536-row dot products in a fixed order (thread partials, then a fixed-order tree).
__global__ void __launch_bounds__(256) input_layer_grads_kernel(const float* __restrict__ Wih,
                                                                const float* __restrict__ Q, float* __restrict__ dWg,
                                                                float* __restrict__ dbg, float* __restrict__ dEmb,
                                                                float* __restrict__ dbih) {
  __shared__ float part[8][kU][33];
  const int j = blockIdx.x;  // 0..63
  float a[kU];
#pragma unroll
  for (int n = 0; n < kU; ++n) a[n] = 0.f;
#pragma unroll 2
  for (int row = threadIdx.x; row < kG; row += 256) {
    const float w = Wih[(size_t)row * kIn + j];
    const float* q = Q + (size_t)row * kU;
#pragma unroll
    for (int n = 0; n < kU; ++n) a[n] += w * q[n];
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int n = 0; n < kU; ++n) part[warp][n][lane] = a[n];
  __syncthreads();
  if (threadIdx.x < kU) {
    const int n = threadIdx.x;
    float t = 0.f;
    for (int w = 0; w < 8; ++w)
      for (int l = 0; l < 32; ++l) t += part[w][n][l];
    if (j < 32) {
      if (n < 3) dWg[j * 3 + n] = t;
      else if (n == 3) dbg[j] = t;
    } else if (n >= 4 && n < 9) {
      dEmb[(n - 4) * 32 + (j - 32)] = t;
    }
  }
  if (j == 0)
    for (int row = threadIdx.x; row < kG; row += 256) dbih[row] = Q[(size_t)row * kU + 3];
}

// ------------------------------------------------------------------ workspace carving
struct GpsWs {
  float *X, *GI, *Hs, *Hin, *RZNG, *dH, *dGI, *dGH, *U, *Q;
};
size_t carve(void* base, int B, int T, GpsWs* w) {
  size_t off = 0;
  const size_t S = (size_t)B * T;
  auto take = [&](size_t n) {
    float* ptr = base ? reinterpret_cast<float*>(reinterpret_cast<char*>(base) + off) : nullptr;
    off = align_up(off + n * sizeof(float), 256);
    return ptr;
  };
  GpsWs tmp;
  tmp.X = take(S * kIn);
  tmp.GI = take(S * kG);
  tmp.Hs = take(S * kH);
  tmp.Hin = take(S * kH);
  tmp.RZNG = take(S * kH * 4);
  tmp.dH = take(S * kH);
  tmp.dGI = take(S * kG);
  tmp.dGH = take(S * kG);
  tmp.U = take(S * kU);
  tmp.Q = take((size_t)kG * kU);
  if (w) *w = tmp;
  return off;
}

GpsPtrs make_ptrs(const ModelLayout& L, const float* params, const ddppo_batch& b, void* ws) {
  GpsPtrs p;
  memset(&p, 0, sizeof(p));  // (loss.on = 0: no fused head / loss unless gps_fwd_loss asks for it)
  p.Wg = params + layout_offset(L, "goal_fc.weight");
  p.bg = params + layout_offset(L, "goal_fc.bias");
  p.Emb = params + layout_offset(L, "act_embed.weight");
  p.Wih = params + layout_offset(L, "rnn.weight_ih");
  p.Whh = params + layout_offset(L, "rnn.weight_hh");
  p.bih = params + layout_offset(L, "rnn.bias_ih");
  p.bhh = params + layout_offset(L, "rnn.bias_hh");
  p.Wo = params + layout_offset(L, "head.weight");
  p.bo = params + layout_offset(L, "head.bias");
  p.goal = b.goal;
  p.prev_action = b.prev_action;
  p.mask = b.mask;
  p.h0 = b.h0;
  p.env_idx = b.env_idx;
  p.B = b.B;
  p.T = b.T;
  p.ld = b.ld;
  p.T_run = b.T_run;
  GpsWs w;
  carve(ws, b.B, b.T_run, &w);
  p.X = w.X;
  p.GI = w.GI;
  p.Hs = w.Hs;
  p.Hin = w.Hin;
  p.RZNG = reinterpret_cast<float4*>(w.RZNG);
  p.dH = w.dH;
  p.dGI = w.dGI;
  p.dGH = w.dGH;
  p.U = w.U;
  p.Q = w.Q;
  return p;
}

template <typename K>
ddppo_status launch_cluster(ddppo_ctx* ctx, K kernel, int threads, size_t smem, const GpsPtrs& p, cudaStream_t st) {
  DDPPO_CUDA_TRY(ctx, cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  DDPPO_CUDA_TRY(ctx, cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kNC, 1, 1);
  cfg.blockDim = dim3(threads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kNC;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  DDPPO_CUDA_TRY(ctx, cudaLaunchKernelEx(&cfg, kernel, p));
  return DDPPO_OK;
}

}  // namespace

size_t gps_workspace(int max_B, int T) { return carve(nullptr, max_B, T, nullptr); }

// h_t of every sample [B*T][512] in a forward's workspace (the act path reads the new state there)
const float* gps_hidden_out(void* ws, int B, int T) {
  GpsWs w;
  carve(ws, B, T, &w);
  return w.Hs;
}

ddppo_status gps_fwd(ddppo_ctx* ctx, const ModelLayout& L, const float* params, const ddppo_batch& b,
                     float* logits, float* values, void* ws, cudaStream_t st, bool skip_head) {
  DDPPO_REQUIRE(ctx, b.B >= 1 && b.B <= kBMax && b.T_run <= kTMax, "gps: minibatch must hold 1..8 envs, T <= 1024");
  GpsPtrs p = make_ptrs(L, params, b, ws);
  const int S = b.B * b.T_run;
  {
    ProfScope ps(ctx, DDPPO_K_NET_FWD, st, 0);
    ProfScope pr(ctx, DDPPO_K_RNN, st, 1);
    if (ctx->prof) ctx->flops[DDPPO_K_RNN] += 2.0 * S * kG * (kH + kIn);
    ddppo_status s =
        launch_cluster(ctx, gps_gru_fwd_kernel, kFwdThreads, sizeof(FwdSmem) + (size_t)S * sizeof(float), p, st);
    if (s != DDPPO_OK) return s;
  }
  if (skip_head) return DDPPO_OK;  // the learner runtime fuses head + loss + head input gradient
  ProfScope ps(ctx, DDPPO_K_HEAD, st, 1);
  head_fwd_kernel<<<grid_for(S, 8, ctx->sm_count * 4), 256, 0, st>>>(p.Wo, p.bo, p.Hs, S, kH, logits, values);
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  return DDPPO_OK;
}

// learner runtime: the recurrence with the head, the PPO loss and the head's input gradient fused
// into its epilogue (dlogits / dvalues / dH / stats written by the same launch)
ddppo_status gps_fwd_loss(ddppo_ctx* ctx, const ModelLayout& L, const float* params, const ddppo_batch& b,
                          const ddppo_loss_inputs& in, const float* mean_invstd, const ddppo_loss_cfg& cfg,
                          float* dlogits, float* dvalues, float* stats, void* ws, cudaStream_t st) {
  DDPPO_REQUIRE(ctx, b.B >= 1 && b.B <= kBMax && b.T_run <= kTMax, "gps: minibatch must hold 1..8 envs, T <= 1024");
  DDPPO_REQUIRE(ctx, b.n_valid >= 1, "loss: need n_valid >= 1");
  DDPPO_REQUIRE(ctx, !cfg.normalize_adv || mean_invstd, "loss: normalize_adv needs mean_invstd");
  DDPPO_REQUIRE(ctx, (uintptr_t)dlogits % 16 == 0, "loss: dlogits must be 16-byte aligned");
  GpsPtrs p = make_ptrs(L, params, b, ws);
  GpsPtrs::Loss& l = p.loss;
  l.on = 1;
  l.use_vclip = cfg.use_value_clip;
  l.len = b.len;
  l.action = in.action;
  l.logp_old = in.logp_old;
  l.value_old = in.value_old;
  l.ret = in.ret;
  l.adv = in.adv;
  l.mean_invstd = cfg.normalize_adv ? mean_invstd : nullptr;
  l.inv_n = 1.f / (float)b.n_valid;
  l.eps = cfg.clip_eps;
  l.vclip_eps = cfg.vclip_eps;
  l.c_v = cfg.c_v;
  l.c_e = cfg.c_e;
  l.n_valid = (float)b.n_valid;
  l.dlogits = dlogits;
  l.dvalues = dvalues;
  l.stats = stats;
  l.err = ctx->d_err;
  const int S = b.B * b.T_run;
  ProfScope ps(ctx, DDPPO_K_NET_FWD, st, 0);
  ProfScope pr(ctx, DDPPO_K_RNN, st, 1);
  if (ctx->prof) ctx->flops[DDPPO_K_RNN] += 2.0 * S * kG * (kH + kIn);
  return launch_cluster(ctx, gps_gru_fwd_kernel, kFwdThreads, sizeof(FwdSmem) + (size_t)S * sizeof(float), p, st);
}

ddppo_status gps_bwd(ddppo_ctx* ctx, const ModelLayout& L, const float* params, const ddppo_batch& b,
                     const float* dlogits, const float* dvalues, float* grad, void* ws, cudaStream_t st,
                     bool dh_ready) {
  DDPPO_REQUIRE(ctx, b.B >= 1 && b.B <= kBMax && b.T_run <= kTMax, "gps: minibatch must hold 1..8 envs, T <= 1024");
  GpsPtrs p = make_ptrs(L, params, b, ws);
  p.dbhh = grad + layout_offset(L, "rnn.bias_hh");  // summed by the BPTT kernel (no colsum pass)
  const int S = b.B * b.T_run;
  // The recurrence occupies 16 SMs; work off its dependency chain runs beside it on two side
  // streams (fork / join through events on the launching stream).
  cudaStream_t sa = nullptr, sb = nullptr;
  ddppo_status s = ctx_side_streams(ctx, &sa, &sb);
  if (s != DDPPO_OK) return s;
  {
    ProfScope ps(ctx, DDPPO_K_HEAD, st, dh_ready ? 1 : 2);
    if (!dh_ready)
      head_dgrad_kernel<<<grid_for(S * kH, 256, ctx->sm_count * 4), 256, 0, st>>>(p.Wo, dlogits, dvalues, S, kH, p.dH);
    DDPPO_CUDA_TRY(ctx, fork_to(ctx, st, sa));
    head_wgrad_kernel<<<kH / 32, 256, 0, sa>>>(p.Hs, dlogits, dvalues, S, kH, grad + layout_offset(L, "head.weight"),
                                              grad + layout_offset(L, "head.bias"));
    DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  }
  {
    ProfScope ps(ctx, DDPPO_K_NET_BWD, st, 0);
    ProfScope pr(ctx, DDPPO_K_RNN, st, 1);
    if (ctx->prof) ctx->flops[DDPPO_K_RNN] += 2.0 * S * kG * kH;
    s = launch_cluster(ctx, gps_gru_bwd_kernel, kBwdThreads, sizeof(BwdSmem) + (size_t)S * sizeof(float), p, st);
    if (s != DDPPO_OK) return s;
  }
  // weight gradients (off the dependency chain), tcgen05 GEMMs over the S samples:
  //   dW_hh[row][j] = sum_s dG_h[s][row] H_in[s][j];  dW_ih[row][j] = sum_s dG_x[s][row] X[s][j]
  //   Q[row][n]     = sum_s dG_x[s][row] U[s][n]   (-> goal FC, embedding and b_ih gradients)
  // main stream: dW_hh; side a: (head weight gradient,) dW_ih; side b: Q, input-layer gradients
  // (db_hh is summed by the BPTT kernel itself)
  ProfScope ps(ctx, DDPPO_K_WGRAD, st, 2);  // + the 3 GEMMs, counted by launch_gemm_tc
  DDPPO_CUDA_TRY(ctx, fork_to(ctx, st, sa));
  DDPPO_CUDA_TRY(ctx, fork_to(ctx, st, sb));
  s = launch_gemm_tc(ctx, GemmTC{p.dGH, 1, kG, p.Hin, 1, kH, grad + layout_offset(L, "rnn.weight_hh"), kH, kG, kH, S},
                     st);
  if (s != DDPPO_OK) return s;
  s = launch_gemm_tc(ctx, GemmTC{p.dGI, 1, kG, p.X, 1, kIn, grad + layout_offset(L, "rnn.weight_ih"), kIn, kG, kIn, S},
                     sa);
  if (s != DDPPO_OK) return s;
  s = launch_gemm_tc(ctx, GemmTC{p.dGI, 1, kG, p.U, 1, kU, p.Q, kU, kG, kU, S}, sb);
  if (s != DDPPO_OK) return s;
  input_layer_grads_kernel<<<kIn, 256, 0, sb>>>(p.Wih, p.Q, grad + layout_offset(L, "goal_fc.weight"),
                                                grad + layout_offset(L, "goal_fc.bias"),
                                                grad + layout_offset(L, "act_embed.weight"),
                                                grad + layout_offset(L, "rnn.bias_ih"));
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  DDPPO_CUDA_TRY(ctx, fork_to(ctx, sa, st));  // join
  DDPPO_CUDA_TRY(ctx, fork_to(ctx, sb, st));
  return DDPPO_OK;
}

#ifdef DDPPO_TRACE
extern "C" int ddppo_debug_trace(long long* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, g_trace, sizeof(long long) * (size_t)n);
}
extern "C" int ddppo_debug_trace_bwd(long long* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, g_trace_b, sizeof(long long) * (size_t)n);
}
#endif

// ------------------------------------------------------------------ shared launchers (used by depth.cu)
ddppo_status launch_head_fwd(ddppo_ctx* ctx, const float* Wo, const float* bo, const float* Hs, int S, int H,
                             float* logits, float* values, cudaStream_t st) {
  head_fwd_kernel<<<grid_for(S, 8, ctx->sm_count * 4), 256, 0, st>>>(Wo, bo, Hs, S, H, logits, values);
  ctx->count(1);
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  return DDPPO_OK;
}

ddppo_status launch_head_bwd(ddppo_ctx* ctx, const float* Wo, const float* Hs, const float* dlogits,
                             const float* dvalues, int S, int H, float* dH, float* dWo, float* dbo,
                             cudaStream_t st) {
  head_dgrad_kernel<<<grid_for(S * H, 256, ctx->sm_count * 4), 256, 0, st>>>(Wo, dlogits, dvalues, S, H, dH);
  head_wgrad_kernel<<<H / 32, 256, 0, st>>>(Hs, dlogits, dvalues, S, H, dWo, dbo);
  ctx->count(2);
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  return DDPPO_OK;
}

ddppo_status launch_colsum(ddppo_ctx* ctx, const float* A, int lda, int S, int M, float* out, cudaStream_t st) {
  colsum_kernel<<<(M + 31) / 32, 256, 0, st>>>(A, lda, S, M, out);
  ctx->count(1);
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  return DDPPO_OK;
}
