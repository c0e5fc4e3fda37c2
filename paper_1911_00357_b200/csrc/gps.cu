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

#include "common.cuh"

namespace {

constexpr int kH = 512, kG = 3 * kH, kIn = 64, kNC = 16, kUPC = kH / kNC /*32*/, kRows = 3 * kUPC /*96*/;
constexpr int kBMax = 8, kA1 = 5, kTMax = 1024, kU = 12;  // U: 9 used columns, padded to 12
constexpr int kHStride = kH + 8;     // fp16 row stride of the broadcast h buffer (bank-conflict pad)
constexpr int kDgStride = kRows + 8; // bf16 row stride of the dG_h buffer
constexpr int kFwdThreads = 384, kBwdThreads = 512;

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
// acquire at cluster scope: the data came from peer CTAs (st.async ... complete_tx)
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
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
// Per step t: all warps wait on the local mbarrier of buffer t%2 (filled by the 16 CTAs'
// st.async packets of h_{t-1}), 12 warps run the W_hh h MMAs, the gate warps (one per batch
// element) finish the GRU cell for the CTA's 32 units and push the new fp16 slice (4 x 16-byte
// packets per batch element) to every CTA's next buffer with st.async + complete_tx.  No
// cluster-wide barrier and no release fence sit on the chain.
struct FwdSmem {
  __half hbuf[2][kBMax][kHStride];  // broadcast h_in (fp16), double-buffered by step parity
  float ghp[2][kRows][kBMax];       // partial W_hh h products of the two k-halves
  float hown[kBMax][kUPC];          // fp32 state h_in for own units
  __half stage[kBMax][kUPC];        // own new h slice before it is packed into st.async packets
  float bhh[kRows];
  float bih[kRows];
  uint64_t bar[2];                  // "buffer t%2 holds h_{t-1}" (tx-count barrier)
};

__global__ void __launch_bounds__(kFwdThreads, 1) gps_gru_fwd_kernel(GpsPtrs p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  FwdSmem& sm = *reinterpret_cast<FwdSmem*>(smem_raw);
  float* smask = reinterpret_cast<float*>(smem_raw + sizeof(FwdSmem));  // [B][T_run]
  const int c = (int)cluster_ctarank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int B = p.B, T_run = p.T_run, S = B * T_run;
  const int g = lane >> 2, tq = lane & 3;

  // ---- prologue 1: zero the h buffers, stage own biases and masks, X slice (samples s % 16 == c)
  for (int i = tid; i < 2 * kBMax * kHStride; i += blockDim.x) (&sm.hbuf[0][0][0])[i] = __float2half(0.f);
  for (int i = tid; i < kRows; i += blockDim.x) {
    sm.bhh[i] = p.bhh[grow_of(c, i)];
    sm.bih[i] = p.bih[grow_of(c, i)];
  }
  for (int i = tid; i < S; i += blockDim.x) {
    const int b = i / T_run, t = i - b * T_run;
    smask[i] = p.mask[(size_t)p.env_idx[b] * p.ld + t];
  }
  if (tid == 0) {
    mbar_init(&sm.bar[0], 1);
    mbar_init(&sm.bar[1], 1);
    fence_mbar_init_cluster();
  }
  for (int i = tid; i < ((S + kNC - 1 - c) / kNC) * kIn; i += blockDim.x) {
    const int s = c + (i / kIn) * kNC, k = i % kIn;
    const int b = s / T_run, t = s - b * T_run;
    const int n = p.env_idx[b];
    float x;
    if (k < 32) {
      const float* gg = p.goal + ((size_t)n * p.T + t) * 3;
      x = p.Wg[k * 3 + 0] * gg[0] + p.Wg[k * 3 + 1] * gg[1] + p.Wg[k * 3 + 2] * gg[2] + p.bg[k];
    } else {
      x = p.Emb[p.prev_action[(size_t)n * p.ld + t] * 32 + (k - 32)];
    }
    p.X[(size_t)s * kIn + k] = x;
  }
  // U[s] = [goal (3), 1, onehot(prev_action) (5)]: the per-sample inputs of the goal FC and the
  // embedding, so that their gradients (and db_ih) come out of one GEMM Q = dG_x^T U in the bwd
  for (int i = tid; i < ((S + kNC - 1 - c) / kNC) * kU; i += blockDim.x) {
    const int s = c + (i / kU) * kNC, k = i % kU;
    const int b = s / T_run, t = s - b * T_run;
    const int n = p.env_idx[b];
    float u;
    if (k < 3) u = p.goal[((size_t)n * p.T + t) * 3 + k];
    else if (k == 3) u = 1.f;
    else if (k < 9) u = (p.prev_action[(size_t)n * p.ld + t] == k - 4) ? 1.f : 0.f;
    else u = 0.f;
    p.U[(size_t)s * kU + k] = u;
  }
  __syncthreads();
  // initial state h_in_0 = mask_0 * h0 (full vector for the MMA operand, own slice in fp32)
  for (int i = tid; i < B * kH; i += blockDim.x) {
    const int b = i / kH, k = i % kH;
    const float h = smask[b * T_run] * p.h0[(size_t)p.env_idx[b] * kH + k];
    sm.hbuf[0][b][k] = __float2half(h);
    if (k >= c * kUPC && k < (c + 1) * kUPC) sm.hown[b][k - c * kUPC] = h;
  }
  // W_hh A-fragments: warp w -> m-tile mt = w/2 (16 local rows), k-half kh = w%2 (16 k-tiles)
  const int mt = warp >> 1, kh = warp & 1;
  uint32_t afr[16][4];
  {
    const int r0 = grow_of(c, mt * 16 + g), r1 = grow_of(c, mt * 16 + g + 8);
    const float2* w0 = reinterpret_cast<const float2*>(p.Whh + (size_t)r0 * kH);
    const float2* w1 = reinterpret_cast<const float2*>(p.Whh + (size_t)r1 * kH);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int k2 = ((kh * 16 + j) * 16 + 2 * tq) / 2;
      const float2 a = w0[k2], b = w1[k2], cc = w0[k2 + 4], d = w1[k2 + 4];
      afr[j][0] = pack_f16(a.x, a.y);
      afr[j][1] = pack_f16(b.x, b.y);
      afr[j][2] = pack_f16(cc.x, cc.y);
      afr[j][3] = pack_f16(d.x, d.y);
    }
  }
  __threadfence();
  cluster_sync_all();  // X visible cluster-wide; barriers/buffers initialised before remote writes

  // ---- prologue 2: GI[c][t][b][lr] = W_ih[row] . X[s] + b_ih[row] with m16n8k16 tiles
  // (6 m-tiles of own rows x S/8 sample tiles x 4 k-tiles; off the dependency chain)
  {
    const int mt2 = warp % 6, half = warp / 6;
    uint32_t wa[4][4];
    const float2* w0 = reinterpret_cast<const float2*>(p.Wih + (size_t)grow_of(c, mt2 * 16 + g) * kIn);
    const float2* w1 = reinterpret_cast<const float2*>(p.Wih + (size_t)grow_of(c, mt2 * 16 + g + 8) * kIn);
#pragma unroll
    for (int kt = 0; kt < 4; ++kt) {
      const int k2 = (kt * 16 + 2 * tq) / 2;
      const float2 a = w0[k2], b = w1[k2], cc = w0[k2 + 4], d = w1[k2 + 4];
      wa[kt][0] = pack_f16(a.x, a.y);
      wa[kt][1] = pack_f16(b.x, b.y);
      wa[kt][2] = pack_f16(cc.x, cc.y);
      wa[kt][3] = pack_f16(d.x, d.y);
    }
    const int n_tiles = (S + 7) / 8;
    for (int nt = half; nt < n_tiles; nt += 2) {
      const int sb = nt * 8 + g;  // sample of this lane's B-fragment column
      const float2* xr = reinterpret_cast<const float2*>(p.X + (size_t)min(sb, S - 1) * kIn);
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int kt = 0; kt < 4; ++kt) {
        float2 x0 = xr[(kt * 16 + 2 * tq) / 2], x1 = xr[(kt * 16 + 8 + 2 * tq) / 2];
        if (sb >= S) x0 = x1 = make_float2(0.f, 0.f);
        mma_f16(acc, wa[kt], pack_f16(x0.x, x0.y), pack_f16(x1.x, x1.y));
      }
      const int lr0 = mt2 * 16 + g;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int lr = lr0 + (e >> 1) * 8, s = nt * 8 + 2 * tq + (e & 1);
        if (s < S) {
          const int b = s / T_run, t = s - b * T_run;
          p.GI[(((size_t)c * T_run + t) * B + b) * kRows + lr] = acc[e] + sm.bih[lr];
        }
      }
    }
  }
  __syncthreads();

  // ---- recurrence
  const int gu = lane, gb = warp;  // gate thread: warp b handles batch element b, lane = unit
  const bool gate_warp = warp < B;
  // st.async packet of this lane: units [8*(lane%4), +8) of batch gb to CTAs lane/4 and lane/4+8
  uint32_t pk_addr[2] = {0u, 0u}, pk_bar[2][2] = {{0u, 0u}, {0u, 0u}};
  float gi_r = 0.f, gi_z = 0.f, gi_n = 0.f;
  const uint32_t tx_bytes = (uint32_t)(kNC * B * kUPC * sizeof(__half));
  if (gate_warp) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const uint32_t q = (uint32_t)(lane / 4 + 8 * j);
      pk_addr[j] = map_to_cta(&sm.hbuf[0][gb][c * kUPC + 8 * (lane % 4)], q);
      pk_bar[j][0] = map_to_cta(&sm.bar[0], q);
      pk_bar[j][1] = map_to_cta(&sm.bar[1], q);
    }
    const float* gi = p.GI + ((size_t)c * T_run * B + gb) * kRows;
    gi_r = gi[gu];
    gi_z = gi[kUPC + gu];
    gi_n = gi[2 * kUPC + gu];
  }
  const uint32_t hbuf_parity_bytes = (uint32_t)sizeof(sm.hbuf[0]);
  for (int t = 0; t < T_run; ++t) {
    const int cur = t & 1;
    if (t > 0) {
      if (tid == 0) mbar_arrive_expect_tx(&sm.bar[cur], tx_bytes);
      mbar_wait_parity(&sm.bar[cur], (uint32_t)(((t - 1) >> 1) & 1));
    }
    {
      float c0[4] = {0.f, 0.f, 0.f, 0.f}, c1[4] = {0.f, 0.f, 0.f, 0.f};
      const uint32_t* hb = reinterpret_cast<const uint32_t*>(&sm.hbuf[cur][g][0]);
#pragma unroll
      for (int j = 0; j < 16; j += 2) {
        const int kt0 = kh * 16 + j, kt1 = kt0 + 1;
        mma_f16(c0, afr[j], hb[kt0 * 8 + tq], hb[kt0 * 8 + 4 + tq]);
        mma_f16(c1, afr[j + 1], hb[kt1 * 8 + tq], hb[kt1 * 8 + 4 + tq]);
      }
      // C layout: c[0],c[1] -> (row g, cols 2tq, 2tq+1); c[2],c[3] -> (row g+8, same cols)
      const int row = mt * 16 + g;
      *reinterpret_cast<float2*>(&sm.ghp[kh][row][2 * tq]) = make_float2(c0[0] + c1[0], c0[1] + c1[1]);
      *reinterpret_cast<float2*>(&sm.ghp[kh][row + 8][2 * tq]) = make_float2(c0[2] + c1[2], c0[3] + c1[3]);
    }
    __syncthreads();
    if (gate_warp) {
      const int lr_r = gu, lr_z = kUPC + gu, lr_n = 2 * kUPC + gu;
      const float gh_r = sm.ghp[0][lr_r][gb] + sm.ghp[1][lr_r][gb] + sm.bhh[lr_r];
      const float gh_z = sm.ghp[0][lr_z][gb] + sm.ghp[1][lr_z][gb] + sm.bhh[lr_z];
      const float gh_n = sm.ghp[0][lr_n][gb] + sm.ghp[1][lr_n][gb] + sm.bhh[lr_n];
      const float h_in = sm.hown[gb][gu];
      const float r = sigmoidf_(gi_r + gh_r);
      const float z = sigmoidf_(gi_z + gh_z);
      const float nn = tanhf(gi_n + r * gh_n);
      const float h = (1.f - z) * nn + z * h_in;
      if (t + 1 < T_run) {
        const float hn = smask[gb * T_run + t + 1] * h;
        sm.hown[gb][gu] = hn;
        sm.stage[gb][gu] = __float2half(hn);
        __syncwarp();
        const uint4 pkt = *reinterpret_cast<const uint4*>(&sm.stage[gb][8 * (lane % 4)]);
        const uint32_t off = (cur ^ 1) * hbuf_parity_bytes;
        st_async_v4(pk_addr[0] + off, pkt, pk_bar[0][cur ^ 1]);
        st_async_v4(pk_addr[1] + off, pkt, pk_bar[1][cur ^ 1]);
      }
      // off the chain: save activations, prefetch the next step's input projections
      const size_t o = ((size_t)gb * T_run + t) * kH + c * kUPC + gu;
      p.Hs[o] = h;
      p.Hin[o] = h_in;
      p.RZNG[o] = make_float4(r, z, nn, gh_n);
      if (t + 1 < T_run) {
        const float* gi = p.GI + (((size_t)c * T_run + t + 1) * B + gb) * kRows;
        gi_r = gi[gu];
        gi_z = gi[kUPC + gu];
        gi_n = gi[2 * kUPC + gu];
      }
    }
  }
  cluster_sync_all();  // no CTA exits while a peer could still address its shared memory
}

// ------------------------------------------------------------------ backward recurrence (BPTT)
// Iteration i (t = T_run-1-i): gate warps form dG for the CTA's units (local), 16 warps multiply
// by W_hh^T (bf16 m16n8k16) and st.async their 32-unit x B partials to the owning CTA's
// recv[i%2] (complete_tx on its mbarrier); the owner sums the 16 partials in CTA order.
struct BwdSmem {
  __nv_bfloat16 dg[kBMax][kDgStride];    // dG_h of own 96 rows (bf16 MMA operand)
  float recv[2][kNC][kUPC][kBMax];        // partial W_hh^T dG_h from every CTA, by iteration parity
  uint64_t bar[2];
};

__global__ void __launch_bounds__(kBwdThreads, 1) gps_gru_bwd_kernel(GpsPtrs p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  BwdSmem& sm = *reinterpret_cast<BwdSmem*>(smem_raw);
  float* smask = reinterpret_cast<float*>(smem_raw + sizeof(BwdSmem));  // [B][T_run]
  const int c = (int)cluster_ctarank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int B = p.B, T_run = p.T_run, S = B * T_run;
  const int g = lane >> 2, tq = lane & 3;

  for (int i = tid; i < kBMax * kDgStride; i += blockDim.x) (&sm.dg[0][0])[i] = __float2bfloat16(0.f);
  for (int i = tid; i < S; i += blockDim.x) {
    const int b = i / T_run, t = i - b * T_run;
    smask[i] = p.mask[(size_t)p.env_idx[b] * p.ld + t];
  }
  if (tid == 0) {
    mbar_init(&sm.bar[0], 1);
    mbar_init(&sm.bar[1], 1);
    fence_mbar_init_cluster();
  }
  // A-fragments of W_hh^T: warp w -> hidden units j in [32w, 32w+32) (2 m-tiles), k = own 96 rows
  uint32_t afr[2][6][4];
#pragma unroll
  for (int mi = 0; mi < 2; ++mi) {
    const int j0 = warp * 32 + mi * 16 + g, j1 = j0 + 8;
#pragma unroll
    for (int kt = 0; kt < 6; ++kt) {
      const int k0 = kt * 16 + 2 * tq;  // local row index
      const float* wa = p.Whh + (size_t)grow_of(c, k0) * kH;
      const float* wb = p.Whh + (size_t)grow_of(c, k0 + 1) * kH;
      const float* wc = p.Whh + (size_t)grow_of(c, k0 + 8) * kH;
      const float* wd = p.Whh + (size_t)grow_of(c, k0 + 9) * kH;
      afr[mi][kt][0] = pack_bf16(wa[j0], wb[j0]);
      afr[mi][kt][1] = pack_bf16(wa[j1], wb[j1]);
      afr[mi][kt][2] = pack_bf16(wc[j0], wd[j0]);
      afr[mi][kt][3] = pack_bf16(wc[j1], wd[j1]);
    }
  }
  // destination of this warp's partials: CTA `warp` (owner of units [32*warp, 32*warp+32))
  const uint32_t recv_remote = map_to_cta(&sm.recv[0][c][0][0], (uint32_t)warp);
  const uint32_t rbar[2] = {map_to_cta(&sm.bar[0], (uint32_t)warp), map_to_cta(&sm.bar[1], (uint32_t)warp)};
  const uint32_t recv_parity_bytes = (uint32_t)sizeof(sm.recv[0]);
  const int cols = 2 * ((B + 1) / 2);  // columns each source sends (lanes with 2*tq < B, pairs)
  const uint32_t tx_bytes = (uint32_t)(kNC * kUPC * cols * sizeof(float));
  __syncthreads();
  cluster_sync_all();

  const int gu = lane, gb = warp;
  const bool gate_warp = warp < B;
  float carry = 0.f;  // dL/dh_t flowing back from step t+1 (already multiplied by mask_{t+1})
  float dH_t = 0.f, h_in = 0.f;
  float4 rzng = make_float4(0.f, 0.f, 0.f, 0.f);
  if (gate_warp) {
    const size_t o = ((size_t)gb * T_run + T_run - 1) * kH + c * kUPC + gu;
    dH_t = p.dH[o];
    rzng = p.RZNG[o];
    h_in = p.Hin[o];
  }
  for (int it = 0; it < T_run; ++it) {
    const int t = T_run - 1 - it, par = it & 1;
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
      sm.dg[gb][gu] = __float2bfloat16(dr_pre);
      sm.dg[gb][kUPC + gu] = __float2bfloat16(dz_pre);
      sm.dg[gb][2 * kUPC + gu] = __float2bfloat16(dn_pre * r);
      dzh = dh * z;
      // off the chain (issued early, consumed never on this path): save dG, prefetch step t-1
      const size_t og = ((size_t)gb * T_run + t) * kG + c * kUPC + gu;
      p.dGI[og] = dr_pre;
      p.dGI[og + kH] = dz_pre;
      p.dGI[og + 2 * kH] = dn_pre;
      p.dGH[og] = dr_pre;
      p.dGH[og + kH] = dz_pre;
      p.dGH[og + 2 * kH] = dn_pre * r;
      if (t > 0) {
        const size_t o = ((size_t)gb * T_run + t - 1) * kH + c * kUPC + gu;
        dH_t = p.dH[o];
        rzng = p.RZNG[o];
        h_in = p.Hin[o];
      }
    }
    __syncthreads();
    {
      float c0[4] = {0.f, 0.f, 0.f, 0.f}, c1[4] = {0.f, 0.f, 0.f, 0.f};
      const uint32_t* db = reinterpret_cast<const uint32_t*>(&sm.dg[g][0]);
#pragma unroll
      for (int kt = 0; kt < 6; ++kt) {
        const uint32_t b0 = db[kt * 8 + tq], b1 = db[kt * 8 + 4 + tq];
        mma_bf16(c0, afr[0][kt], b0, b1);
        mma_bf16(c1, afr[1][kt], b0, b1);
      }
      // rows (unit within the owner's slice): g, g+8 (m-tile 0), 16+g, 24+g (m-tile 1); cols 2tq, 2tq+1
      if (2 * tq < B) {
        const uint32_t base = recv_remote + par * recv_parity_bytes;
        st_async_v2f(base + (uint32_t)(((g) * kBMax + 2 * tq) * 4), c0[0], c0[1], rbar[par]);
        st_async_v2f(base + (uint32_t)(((g + 8) * kBMax + 2 * tq) * 4), c0[2], c0[3], rbar[par]);
        st_async_v2f(base + (uint32_t)(((16 + g) * kBMax + 2 * tq) * 4), c1[0], c1[1], rbar[par]);
        st_async_v2f(base + (uint32_t)(((24 + g) * kBMax + 2 * tq) * 4), c1[2], c1[3], rbar[par]);
      }
    }
    if (gate_warp) {
      if (tid == 0) mbar_arrive_expect_tx(&sm.bar[par], tx_bytes);
      mbar_wait_parity(&sm.bar[par], (uint32_t)((it >> 1) & 1));
      float s = 0.f;
#pragma unroll
      for (int q = 0; q < kNC; ++q) s += sm.recv[par][q][gu][gb];
      carry = smask[gb * T_run + t] * (dzh + s);
    }
    __syncthreads();  // every warp's MMA has read dg before the gate warps overwrite it
  }
  cluster_sync_all();  // no CTA exits while a peer could still address its shared memory
}

// ------------------------------------------------------------------ head (Linear(512, 5)) fwd/bwd
__global__ void head_fwd_kernel(const float* __restrict__ Wo, const float* __restrict__ bo, const float* __restrict__ Hs,
                                int S, float* __restrict__ logits, float* __restrict__ values) {
  const int warps = blockDim.x >> 5, lane = threadIdx.x & 31;
  for (int s = blockIdx.x * warps + (threadIdx.x >> 5); s < S; s += gridDim.x * warps) {
    const float* h = Hs + (size_t)s * kH;
    float acc[kA1] = {0.f, 0.f, 0.f, 0.f, 0.f};
    for (int k = lane; k < kH; k += 32) {
      const float hv = h[k];
#pragma unroll
      for (int o = 0; o < kA1; ++o) acc[o] += Wo[o * kH + k] * hv;
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
                                  const float* __restrict__ dvalues, int S, float* __restrict__ dH) {
  const size_t n = (size_t)S * kH;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int s = (int)(i / kH), k = (int)(i % kH);
    const float4 dl = *reinterpret_cast<const float4*>(dlogits + (size_t)s * 4);
    dH[i] = Wo[k] * dl.x + Wo[kH + k] * dl.y + Wo[2 * kH + k] * dl.z + Wo[3 * kH + k] * dl.w +
            Wo[4 * kH + k] * dvalues[s];
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
                                                         const float* __restrict__ dvalues, int S,
                                                         float* __restrict__ dWo, float* __restrict__ dbo) {
  __shared__ float part[kRedChunks][kA1][33];
  const int kk = threadIdx.x & 31, q = threadIdx.x >> 5, k = blockIdx.x * 32 + kk;
  const int per = (S + kRedChunks - 1) / kRedChunks;
  float a[kA1] = {0.f, 0.f, 0.f, 0.f, 0.f}, bsum[kA1] = {0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll 8
  for (int s = q * per; s < min(S, (q + 1) * per); ++s) {
    const float h = Hs[(size_t)s * kH + k];
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
      dWo[o * kH + k] = t;
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

ddppo_status gps_fwd(ddppo_ctx* ctx, const ModelLayout& L, const float* params, const ddppo_batch& b,
                     float* logits, float* values, void* ws, cudaStream_t st) {
  DDPPO_REQUIRE(ctx, b.B >= 1 && b.B <= kBMax && b.T_run <= kTMax, "gps: minibatch must hold 1..8 envs, T <= 1024");
  GpsPtrs p = make_ptrs(L, params, b, ws);
  const int S = b.B * b.T_run;
  {
    ProfScope ps(ctx, DDPPO_K_NET_FWD, st, 1);
    ddppo_status s =
        launch_cluster(ctx, gps_gru_fwd_kernel, kFwdThreads, sizeof(FwdSmem) + (size_t)S * sizeof(float), p, st);
    if (s != DDPPO_OK) return s;
  }
  ProfScope ps(ctx, DDPPO_K_HEAD, st, 1);
  head_fwd_kernel<<<grid_for(S, 8, ctx->sm_count * 4), 256, 0, st>>>(p.Wo, p.bo, p.Hs, S, logits, values);
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  return DDPPO_OK;
}

ddppo_status gps_bwd(ddppo_ctx* ctx, const ModelLayout& L, const float* params, const ddppo_batch& b,
                     const float* dlogits, const float* dvalues, float* grad, void* ws, cudaStream_t st) {
  DDPPO_REQUIRE(ctx, b.B >= 1 && b.B <= kBMax && b.T_run <= kTMax, "gps: minibatch must hold 1..8 envs, T <= 1024");
  GpsPtrs p = make_ptrs(L, params, b, ws);
  const int S = b.B * b.T_run;
  {
    ProfScope ps(ctx, DDPPO_K_HEAD, st, 2);
    head_dgrad_kernel<<<grid_for(S * kH, 256, ctx->sm_count * 4), 256, 0, st>>>(p.Wo, dlogits, dvalues, S, p.dH);
    head_wgrad_kernel<<<kH / 32, 256, 0, st>>>(p.Hs, dlogits, dvalues, S, grad + layout_offset(L, "head.weight"),
                                              grad + layout_offset(L, "head.bias"));
    DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  }
  {
    ProfScope ps(ctx, DDPPO_K_NET_BWD, st, 1);
    ddppo_status s =
        launch_cluster(ctx, gps_gru_bwd_kernel, kBwdThreads, sizeof(BwdSmem) + (size_t)S * sizeof(float), p, st);
    if (s != DDPPO_OK) return s;
  }
  // weight gradients (off the dependency chain)
  ProfScope ps(ctx, DDPPO_K_WGRAD, st, 5);
  // tcgen05 GEMMs (bf16 operands, fp32 TMEM accumulation) over the S samples:
  //   dW_hh[row][j] = sum_s dG_h[s][row] H_in[s][j];  dW_ih[row][j] = sum_s dG_x[s][row] X[s][j]
  //   Q[row][n]     = sum_s dG_x[s][row] U[s][n]   (-> goal FC, embedding and b_ih gradients)
  ddppo_status gs = launch_gemm_tc(
      ctx, GemmTC{p.dGH, 1, kG, p.Hin, 1, kH, grad + layout_offset(L, "rnn.weight_hh"), kH, kG, kH, S}, st);
  if (gs != DDPPO_OK) return gs;
  gs = launch_gemm_tc(ctx, GemmTC{p.dGI, 1, kG, p.X, 1, kIn, grad + layout_offset(L, "rnn.weight_ih"), kIn, kG, kIn, S},
                      st);
  if (gs != DDPPO_OK) return gs;
  gs = launch_gemm_tc(ctx, GemmTC{p.dGI, 1, kG, p.U, 1, kU, p.Q, kU, kG, kU, S}, st);
  if (gs != DDPPO_OK) return gs;
  colsum_kernel<<<kG / 32, 256, 0, st>>>(p.dGH, kG, S, kG, grad + layout_offset(L, "rnn.bias_hh"));
  input_layer_grads_kernel<<<kIn, 256, 0, st>>>(p.Wih, p.Q, grad + layout_offset(L, "goal_fc.weight"),
                                                grad + layout_offset(L, "goal_fc.bias"),
                                                grad + layout_offset(L, "act_embed.weight"),
                                                grad + layout_offset(L, "rnn.bias_ih"));
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  return DDPPO_OK;
}
