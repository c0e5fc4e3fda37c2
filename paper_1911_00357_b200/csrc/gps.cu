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
//     CTA's shared memory through DSMEM (st.shared::cluster); one cluster barrier per step;
//   * the backward pass (BPTT) multiplies by W_hh^T: each CTA forms partial products over its
//     96 rows for all 512 hidden units and sends each 32-unit slice to its owner CTA, which sums
//     the 16 partials in fixed order (deterministic).
// Everything that is NOT on the dependency chain is hoisted out of the recurrence: the input
// projection W_ih x + b_ih for all steps (prologue of the forward kernel) and the weight
// gradients dW_hh = dG_h^T H_in, dW_ih = dG_x^T X (plain GEMMs after the backward recurrence).
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "common.cuh"

namespace {

constexpr int kH = 512, kG = 3 * kH, kIn = 64, kNC = 16, kUPC = kH / kNC /*32*/, kRows = 3 * kUPC /*96*/;
constexpr int kBMax = 8, kA1 = 5;
constexpr int kHStride = kH + 8;     // fp16 row stride of the broadcast h buffer (bank-conflict pad)
constexpr int kDgStride = kRows + 8; // bf16 row stride of the dG_h buffer
constexpr int kFwdThreads = 384, kBwdThreads = 512;

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ uint32_t map_to_cta(const void* smem_ptr, uint32_t cta) {
  uint32_t a = (uint32_t)__cvta_generic_to_shared(smem_ptr), r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(cta));
  return r;
}
__device__ __forceinline__ void st_cluster_u16(uint32_t addr, uint16_t v) {
  asm volatile("st.shared::cluster.u16 [%0], %1;" ::"r"(addr), "h"(v) : "memory");
}
__device__ __forceinline__ void st_cluster_f32(uint32_t addr, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
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
  float* X;     // [S][64]
  float* GI;    // [16][T_run][B][96]   CTA-local input projections (incl. b_ih)
  float* Hs;    // [S][512]  h_t
  float* Hin;   // [S][512]  mask_t * h_{t-1}
  float* Rg;    // [S][512]
  float* Zg;    // [S][512]
  float* Ng;    // [S][512]
  float* GHN;   // [S][512]  W_hn h_in + b_hn
  float* dH;    // [S][512]  dL/dh_t from the head
  float* dGI;   // [S][1536]
  float* dGH;   // [S][1536]
  float* dX;    // [S][64]
};

// ------------------------------------------------------------------ forward recurrence
struct FwdSmem {
  __half hbuf[2][kBMax][kHStride];  // broadcast h_in (fp16), double-buffered by step parity
  float ghp[2][kRows][kBMax];       // partial W_hh h products of the two k-halves
  float hown[kBMax][kUPC];          // fp32 state h_in for own units
  float bhh[kRows];
  float wih[kRows][kIn + 1];        // own W_ih rows (prologue)
  float xs[32][kIn];                // X chunk (prologue)
};

__global__ void __launch_bounds__(kFwdThreads, 1) gps_gru_fwd_kernel(GpsPtrs p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  FwdSmem& sm = *reinterpret_cast<FwdSmem*>(smem_raw);
  const int c = (int)cluster_ctarank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int B = p.B, T_run = p.T_run, S = B * T_run;

  // ---- prologue 1: zero the h buffers, stage own rows, compute X slice (samples s % 16 == c)
  for (int i = tid; i < 2 * kBMax * kHStride; i += blockDim.x) (&sm.hbuf[0][0][0])[i] = __float2half(0.f);
  for (int i = tid; i < kRows; i += blockDim.x) sm.bhh[i] = p.bhh[grow_of(c, i)];
  for (int i = tid; i < kRows * kIn; i += blockDim.x) {
    const int lr = i / kIn, k = i % kIn;
    sm.wih[lr][k] = p.Wih[(size_t)grow_of(c, lr) * kIn + k];
  }
  for (int i = tid; i < ((S + kNC - 1 - c) / kNC) * kIn; i += blockDim.x) {
    const int s = c + (i / kIn) * kNC, k = i % kIn;
    const int b = s / T_run, t = s - b * T_run;
    const int n = p.env_idx[b];
    float x;
    if (k < 32) {
      const float* g = p.goal + ((size_t)n * p.T + t) * 3;
      x = p.Wg[k * 3 + 0] * g[0] + p.Wg[k * 3 + 1] * g[1] + p.Wg[k * 3 + 2] * g[2] + p.bg[k];
    } else {
      x = p.Emb[p.prev_action[(size_t)n * p.ld + t] * 32 + (k - 32)];
    }
    p.X[(size_t)s * kIn + k] = x;
  }
  // initial state h_in_0 = mask_0 * h0 (full vector for the MMA operand, own slice in fp32)
  for (int i = tid; i < B * kH; i += blockDim.x) {
    const int b = i / kH, k = i % kH;
    const int n = p.env_idx[b];
    const float h = p.mask[(size_t)n * p.ld] * p.h0[(size_t)n * kH + k];
    sm.hbuf[0][b][k] = __float2half(h);
    if (k >= c * kUPC && k < (c + 1) * kUPC) sm.hown[b][k - c * kUPC] = h;
  }
  // W_hh A-fragments: warp w -> m-tile mt = w/2 (16 local rows), k-half kh = w%2 (16 k-tiles)
  const int mt = warp >> 1, kh = warp & 1;
  const int g = lane >> 2, tq = lane & 3;
  uint32_t afr[16][4];
  if (warp < 12) {
    const int r0 = grow_of(c, mt * 16 + g), r1 = grow_of(c, mt * 16 + g + 8);
    const float* w0 = p.Whh + (size_t)r0 * kH;
    const float* w1 = p.Whh + (size_t)r1 * kH;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int k0 = (kh * 16 + j) * 16 + 2 * tq;
      afr[j][0] = pack_f16(w0[k0], w0[k0 + 1]);
      afr[j][1] = pack_f16(w1[k0], w1[k0 + 1]);
      afr[j][2] = pack_f16(w0[k0 + 8], w0[k0 + 9]);
      afr[j][3] = pack_f16(w1[k0 + 8], w1[k0 + 9]);
    }
  }
  __threadfence();
  cluster_sync_all();  // X visible cluster-wide; every CTA's smem initialised before remote writes

  // ---- prologue 2: GI[c][t][b][lr] = W_ih[row] . X[s] + b_ih[row]  (off the dependency chain)
  for (int s0 = 0; s0 < S; s0 += 32) {
    const int ns = min(32, S - s0);
    for (int i = tid; i < ns * kIn; i += blockDim.x) sm.xs[i / kIn][i % kIn] = p.X[(size_t)(s0 + i / kIn) * kIn + i % kIn];
    __syncthreads();
    for (int i = tid; i < kRows * ns; i += blockDim.x) {
      const int lr = i % kRows, si = i / kRows;
      float acc = p.bih[grow_of(c, lr)];
#pragma unroll 16
      for (int k = 0; k < kIn; ++k) acc += sm.wih[lr][k] * sm.xs[si][k];
      const int s = s0 + si, b = s / T_run, t = s - b * T_run;
      p.GI[(((size_t)c * T_run + t) * B + b) * kRows + lr] = acc;
    }
    __syncthreads();
  }

  // ---- recurrence
  const int gu = tid % kUPC, gb = tid / kUPC;  // gate thread: unit, batch (tid < 32*B)
  const bool gate_thread = tid < kUPC * B;
  uint32_t remote_h[kNC];
  if (gate_thread) {
#pragma unroll
    for (int q = 0; q < kNC; ++q) remote_h[q] = map_to_cta(&sm.hbuf[0][gb][c * kUPC + gu], q);
  }
  const uint32_t hbuf_parity_bytes = (uint32_t)sizeof(sm.hbuf[0]);
  for (int t = 0; t < T_run; ++t) {
    const int cur = t & 1;
    float gi_r = 0.f, gi_z = 0.f, gi_n = 0.f, m_next = 0.f;
    if (gate_thread) {  // prefetch (independent of the chain)
      const float* gi = p.GI + (((size_t)c * T_run + t) * B + gb) * kRows;
      gi_r = gi[gu];
      gi_z = gi[kUPC + gu];
      gi_n = gi[2 * kUPC + gu];
      if (t + 1 < T_run) m_next = p.mask[(size_t)p.env_idx[gb] * p.ld + t + 1];
    }
    if (warp < 12) {
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
      sm.ghp[kh][row][2 * tq] = c0[0] + c1[0];
      sm.ghp[kh][row][2 * tq + 1] = c0[1] + c1[1];
      sm.ghp[kh][row + 8][2 * tq] = c0[2] + c1[2];
      sm.ghp[kh][row + 8][2 * tq + 1] = c0[3] + c1[3];
    }
    __syncthreads();
    if (gate_thread) {
      const int lr_r = gu, lr_z = kUPC + gu, lr_n = 2 * kUPC + gu;
      const float gh_r = sm.ghp[0][lr_r][gb] + sm.ghp[1][lr_r][gb] + sm.bhh[lr_r];
      const float gh_z = sm.ghp[0][lr_z][gb] + sm.ghp[1][lr_z][gb] + sm.bhh[lr_z];
      const float gh_n = sm.ghp[0][lr_n][gb] + sm.ghp[1][lr_n][gb] + sm.bhh[lr_n];
      const float h_in = sm.hown[gb][gu];
      const float r = sigmoidf_(gi_r + gh_r);
      const float z = sigmoidf_(gi_z + gh_z);
      const float nn = tanhf(gi_n + r * gh_n);
      const float h = (1.f - z) * nn + z * h_in;
      const size_t o = ((size_t)gb * T_run + t) * kH + c * kUPC + gu;
      p.Hs[o] = h;
      p.Hin[o] = h_in;
      p.Rg[o] = r;
      p.Zg[o] = z;
      p.Ng[o] = nn;
      p.GHN[o] = gh_n;
      const float hn = m_next * h;
      sm.hown[gb][gu] = hn;
      if (t + 1 < T_run) {
        const uint16_t bits = __half_as_ushort(__float2half(hn));
        const uint32_t off = (cur ^ 1) * hbuf_parity_bytes;
#pragma unroll
        for (int q = 0; q < kNC; ++q) st_cluster_u16(remote_h[q] + off, bits);
      }
    }
    cluster_sync_all();
  }
}

// ------------------------------------------------------------------ backward recurrence (BPTT)
struct BwdSmem {
  __nv_bfloat16 dg[kBMax][kDgStride];    // dG_h of own 96 rows (bf16 MMA operand)
  float recv[2][kNC][kUPC][kBMax];        // partial W_hh^T dG_h from every CTA, by step parity
};

__global__ void __launch_bounds__(kBwdThreads, 1) gps_gru_bwd_kernel(GpsPtrs p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  BwdSmem& sm = *reinterpret_cast<BwdSmem*>(smem_raw);
  const int c = (int)cluster_ctarank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int B = p.B, T_run = p.T_run;
  const int g = lane >> 2, tq = lane & 3;

  for (int i = tid; i < kBMax * kDgStride; i += blockDim.x) (&sm.dg[0][0])[i] = __float2bfloat16(0.f);
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
  const uint32_t recv_parity_bytes = (uint32_t)sizeof(sm.recv[0]);
  __syncthreads();
  cluster_sync_all();

  const int gu = tid % kUPC, gb = tid / kUPC;
  const bool gate_thread = tid < kUPC * B;
  float carry = 0.f;  // dL/dh_{t} flowing back from step t+1 (already multiplied by mask_{t+1})
  for (int t = T_run - 1; t >= 0; --t) {
    const int par = t & 1;
    float dzh = 0.f;
    if (gate_thread) {
      const size_t o = ((size_t)gb * T_run + t) * kH + c * kUPC + gu;
      const float dh = p.dH[o] + carry;
      const float r = p.Rg[o], z = p.Zg[o], nn = p.Ng[o], ghn = p.GHN[o], h_in = p.Hin[o];
      const float dn = dh * (1.f - z);
      const float dz = dh * (h_in - nn);
      const float dn_pre = dn * (1.f - nn * nn);
      const float dr = dn_pre * ghn;
      const float dr_pre = dr * r * (1.f - r);
      const float dz_pre = dz * z * (1.f - z);
      const size_t og = ((size_t)gb * T_run + t) * kG + c * kUPC + gu;
      p.dGI[og] = dr_pre;
      p.dGI[og + kH] = dz_pre;
      p.dGI[og + 2 * kH] = dn_pre;
      const float dgn = dn_pre * r;
      p.dGH[og] = dr_pre;
      p.dGH[og + kH] = dz_pre;
      p.dGH[og + 2 * kH] = dgn;
      sm.dg[gb][gu] = __float2bfloat16(dr_pre);
      sm.dg[gb][kUPC + gu] = __float2bfloat16(dz_pre);
      sm.dg[gb][2 * kUPC + gu] = __float2bfloat16(dgn);
      dzh = dh * z;
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
        st_cluster_v2f32(base + (uint32_t)(((g) * kBMax + 2 * tq) * 4), c0[0], c0[1]);
        st_cluster_v2f32(base + (uint32_t)(((g + 8) * kBMax + 2 * tq) * 4), c0[2], c0[3]);
        st_cluster_v2f32(base + (uint32_t)(((16 + g) * kBMax + 2 * tq) * 4), c1[0], c1[1]);
        st_cluster_v2f32(base + (uint32_t)(((24 + g) * kBMax + 2 * tq) * 4), c1[2], c1[3]);
      }
    }
    cluster_sync_all();
    if (gate_thread) {
      float s = 0.f;
#pragma unroll
      for (int q = 0; q < kNC; ++q) s += sm.recv[par][q][gu][gb];
      const float m_t = p.mask[(size_t)p.env_idx[gb] * p.ld + t];
      carry = m_t * (dzh + s);
    }
  }
  cluster_sync_all();  // nobody exits while a peer may still write into its shared memory
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
      logits[(size_t)s * 4 + 0] = acc[0] + bo[0];
      logits[(size_t)s * 4 + 1] = acc[1] + bo[1];
      logits[(size_t)s * 4 + 2] = acc[2] + bo[2];
      logits[(size_t)s * 4 + 3] = acc[3] + bo[3];
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
    const float* dl = dlogits + (size_t)s * 4;
    dH[i] = Wo[k] * dl[0] + Wo[kH + k] * dl[1] + Wo[2 * kH + k] * dl[2] + Wo[3 * kH + k] * dl[3] +
            Wo[4 * kH + k] * dvalues[s];
  }
}

// dWo[o][k] = sum_s dout[s][o] Hs[s][k];  dbo[o] = sum_s dout[s][o]   (fixed order over s)
__global__ void head_wgrad_kernel(const float* __restrict__ Hs, const float* __restrict__ dlogits,
                                  const float* __restrict__ dvalues, int S, float* __restrict__ dWo,
                                  float* __restrict__ dbo) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < kH) {
    float a[kA1] = {0.f, 0.f, 0.f, 0.f, 0.f};
    for (int s = 0; s < S; ++s) {
      const float h = Hs[(size_t)s * kH + k];
      const float* dl = dlogits + (size_t)s * 4;
      a[0] += dl[0] * h;
      a[1] += dl[1] * h;
      a[2] += dl[2] * h;
      a[3] += dl[3] * h;
      a[4] += dvalues[s] * h;
    }
#pragma unroll
    for (int o = 0; o < kA1; ++o) dWo[o * kH + k] = a[o];
  } else if (k < kH + kA1) {
    const int o = k - kH;
    float a = 0.f;
    for (int s = 0; s < S; ++s) a += o < 4 ? dlogits[(size_t)s * 4 + o] : dvalues[s];
    dbo[o] = a;
  }
}

// ------------------------------------------------------------------ weight-gradient GEMMs
// C[M][N] = sum_s A[s][a_off + m] * Bm[s][n]  (A row stride lda, Bm row stride ldb), fixed s order.
// 64x64 tile per CTA, 256 threads, 4x4 outputs per thread, s in chunks of 16 through smem.
__global__ void __launch_bounds__(256) gemm_atb_kernel(const float* __restrict__ A, int lda,
                                                       const float* __restrict__ Bm, int ldb, int S, int M, int N,
                                                       float* __restrict__ C, int ldc) {
  __shared__ float As[16][64 + 4];
  __shared__ float Bs[16][64 + 4];
  const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  float acc[4][4] = {};
  for (int s0 = 0; s0 < S; s0 += 16) {
    for (int i = threadIdx.x; i < 16 * 64; i += 256) {
      const int ss = i / 64, j = i % 64;
      const int s = s0 + ss;
      As[ss][j] = (s < S && m0 + j < M) ? A[(size_t)s * lda + m0 + j] : 0.f;
      Bs[ss][j] = (s < S && n0 + j < N) ? Bm[(size_t)s * ldb + n0 + j] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int ss = 0; ss < 16; ++ss) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[ss][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[ss][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] += a[i] * b[j];
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int m = m0 + ty * 4 + i, n = n0 + tx * 4 + j;
      if (m < M && n < N) C[(size_t)m * ldc + n] = acc[i][j];
    }
}

// column sums: out[m] = sum_s A[s][m]
__global__ void colsum_kernel(const float* __restrict__ A, int lda, int S, int M, float* __restrict__ out) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= M) return;
  float a = 0.f;
  for (int s = 0; s < S; ++s) a += A[(size_t)s * lda + m];
  out[m] = a;
}

// dX[s][k] = sum_row dGI[s][row] * Wih[row][k]   (one warp per sample; lanes over k pairs)
__global__ void dx_kernel(const float* __restrict__ dGI, const float* __restrict__ Wih, int S, float* __restrict__ dX) {
  const int warps = blockDim.x >> 5, lane = threadIdx.x & 31;
  for (int s = blockIdx.x * warps + (threadIdx.x >> 5); s < S; s += gridDim.x * warps) {
    const float* d = dGI + (size_t)s * kG;
    float a0 = 0.f, a1 = 0.f;
    for (int row = 0; row < kG; ++row) {
      const float dv = d[row];
      a0 += dv * Wih[(size_t)row * kIn + lane];
      a1 += dv * Wih[(size_t)row * kIn + 32 + lane];
    }
    dX[(size_t)s * kIn + lane] = a0;
    dX[(size_t)s * kIn + 32 + lane] = a1;
  }
}

// goal FC and embedding gradients from dX (fixed order over samples)
__global__ void input_grads_kernel(const float* __restrict__ dX, const float* __restrict__ goal,
                                   const int32_t* __restrict__ prev_action, const int32_t* __restrict__ env_idx,
                                   int T, int ld, int T_run, int S, float* __restrict__ dWg, float* __restrict__ dbg,
                                   float* __restrict__ dEmb) {
  const int j = threadIdx.x;  // 0..31 goal units, 32..63 embedding dims
  if (j < 32) {
    float w0 = 0.f, w1 = 0.f, w2 = 0.f, bb = 0.f;
    for (int s = 0; s < S; ++s) {
      const int b = s / T_run, t = s - b * T_run;
      const float* g = goal + ((size_t)env_idx[b] * T + t) * 3;
      const float d = dX[(size_t)s * kIn + j];
      w0 += d * g[0];
      w1 += d * g[1];
      w2 += d * g[2];
      bb += d;
    }
    dWg[j * 3 + 0] = w0;
    dWg[j * 3 + 1] = w1;
    dWg[j * 3 + 2] = w2;
    dbg[j] = bb;
  } else if (j < 64) {
    float e[kA1] = {0.f, 0.f, 0.f, 0.f, 0.f};
    for (int s = 0; s < S; ++s) {
      const int b = s / T_run, t = s - b * T_run;
      const int a = prev_action[(size_t)env_idx[b] * ld + t];
      const float d = dX[(size_t)s * kIn + j];
#pragma unroll
      for (int q = 0; q < kA1; ++q) e[q] += (a == q) ? d : 0.f;
    }
#pragma unroll
    for (int q = 0; q < kA1; ++q) dEmb[q * 32 + (j - 32)] = e[q];
  }
}

// ------------------------------------------------------------------ workspace carving
struct GpsWs {
  float *X, *GI, *Hs, *Hin, *Rg, *Zg, *Ng, *GHN, *dH, *dGI, *dGH, *dX;
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
  tmp.Rg = take(S * kH);
  tmp.Zg = take(S * kH);
  tmp.Ng = take(S * kH);
  tmp.GHN = take(S * kH);
  tmp.dH = take(S * kH);
  tmp.dGI = take(S * kG);
  tmp.dGH = take(S * kG);
  tmp.dX = take(S * kIn);
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
  p.Rg = w.Rg;
  p.Zg = w.Zg;
  p.Ng = w.Ng;
  p.GHN = w.GHN;
  p.dH = w.dH;
  p.dGI = w.dGI;
  p.dGH = w.dGH;
  p.dX = w.dX;
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
  DDPPO_REQUIRE(ctx, b.B >= 1 && b.B <= kBMax, "gps: minibatch must hold 1..8 envs");
  GpsPtrs p = make_ptrs(L, params, b, ws);
  {
    ProfScope ps(ctx, DDPPO_K_NET_FWD, st, 1);
    ddppo_status s = launch_cluster(ctx, gps_gru_fwd_kernel, kFwdThreads, sizeof(FwdSmem), p, st);
    if (s != DDPPO_OK) return s;
  }
  const int S = b.B * b.T_run;
  ProfScope ps(ctx, DDPPO_K_HEAD, st, 1);
  head_fwd_kernel<<<grid_for(S, 8, ctx->sm_count * 4), 256, 0, st>>>(p.Wo, p.bo, p.Hs, S, logits, values);
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  return DDPPO_OK;
}

ddppo_status gps_bwd(ddppo_ctx* ctx, const ModelLayout& L, const float* params, const ddppo_batch& b,
                     const float* dlogits, const float* dvalues, float* grad, void* ws, cudaStream_t st) {
  DDPPO_REQUIRE(ctx, b.B >= 1 && b.B <= kBMax, "gps: minibatch must hold 1..8 envs");
  GpsPtrs p = make_ptrs(L, params, b, ws);
  const int S = b.B * b.T_run;
  {
  ProfScope ps(ctx, DDPPO_K_HEAD, st, 2);
  head_dgrad_kernel<<<grid_for(S * kH, 256, ctx->sm_count * 4), 256, 0, st>>>(p.Wo, dlogits, dvalues, S, p.dH);
  head_wgrad_kernel<<<(kH + kA1 + 127) / 128, 128, 0, st>>>(p.Hs, dlogits, dvalues, S,
                                                            grad + layout_offset(L, "head.weight"),
                                                            grad + layout_offset(L, "head.bias"));
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  }
  {
    ProfScope ps(ctx, DDPPO_K_NET_BWD, st, 1);
    ddppo_status s = launch_cluster(ctx, gps_gru_bwd_kernel, kBwdThreads, sizeof(BwdSmem), p, st);
    if (s != DDPPO_OK) return s;
  }
  // weight gradients (off the dependency chain)
  ProfScope ps(ctx, DDPPO_K_WGRAD, st, 6);
  gemm_atb_kernel<<<dim3(kH / 64, kG / 64), 256, 0, st>>>(p.dGH, kG, p.Hin, kH, S, kG, kH,
                                                         grad + layout_offset(L, "rnn.weight_hh"), kH);
  gemm_atb_kernel<<<dim3(1, kG / 64), 256, 0, st>>>(p.dGI, kG, p.X, kIn, S, kG, kIn,
                                                   grad + layout_offset(L, "rnn.weight_ih"), kIn);
  colsum_kernel<<<kG / 128, 128, 0, st>>>(p.dGH, kG, S, kG, grad + layout_offset(L, "rnn.bias_hh"));
  colsum_kernel<<<kG / 128, 128, 0, st>>>(p.dGI, kG, S, kG, grad + layout_offset(L, "rnn.bias_ih"));
  dx_kernel<<<grid_for(S, 8, ctx->sm_count * 4), 256, 0, st>>>(p.dGI, p.Wih, S, p.dX);
  input_grads_kernel<<<1, 64, 0, st>>>(p.dX, b.goal, b.prev_action, b.env_idx, b.T, b.ld, b.T_run, S,
                                       grad + layout_offset(L, "goal_fc.weight"),
                                       grad + layout_offset(L, "goal_fc.bias"),
                                       grad + layout_offset(L, "act_embed.weight"));
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  return DDPPO_OK;
}
