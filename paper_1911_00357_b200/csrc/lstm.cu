// LSTM-512 recurrences of the Depth agent (configs[2]; P:L214 / P:L593 "LSTM with a 512-dimensional
// hidden state"; PyTorch gate order i, f, g, o; reading Z21: state and cell multiplied by mask_t).
//
// Same B200 structure as the GRU of gps.cu, one 16-CTA cluster per direction, CTA c owning hidden
// units [32c, 32c+32):
//  * forward: the CTA's 128 gate rows (i|f|g|o x 32 units, exactly M = 128) of W_hh stay in TMEM as
//    the fp16 A operand; B = h_{t-1} [16 env rows][512] (fp16, canonical K-major smem tile) is
//    filled by every CTA's 16-byte st.async packets (complete_tx on the receiver's mbarrier);
//    4 warps x 8 tcgen05.mma (M=128, N=16, K=16) per step into 4 TMEM accumulators.  The input
//    projection W_ih x_t (x = [visual 512, goal 32, action 32]) for all steps is one tcgen05 GEMM
//    before the recurrence; the gate threads prefetch it one step ahead.
//  * backward (BPTT): W_hh^T (bf16, 4 tiles of 128 units x 128 own rows) in TMEM; per step the
//    gate warps form dL/d(gates) (the cell gradient carry is CTA-local), 8 warps x 4 MMAs give the
//    partial W_hh^T dG for all 512 units, sent to the owners (16-byte packets), summed in CTA order.
#include "common.cuh"
#include "tc_util.cuh"

using namespace tcu;

namespace {

constexpr int kH = 512, kG4 = 4 * kH, kNC = 16, kUPC = kH / kNC /*32*/, kRows = 4 * kUPC /*128*/;
constexpr int kBMax = 8;
constexpr int kThreads = 256;

__device__ __forceinline__ int grow_of(int c, int lr) { return (lr / kUPC) * kH + c * kUPC + (lr % kUPC); }

// ------------------------------------------------------------------ forward
constexpr uint32_t kHSBO = (kH / 8) * 128;  // 8192 B between 8-row groups of the [16 x 512] B tile
constexpr uint32_t kAcc0 = kH / 2;          // TMEM columns [0, 256): W_hh rows (fp16 pairs)
constexpr int kFwdCols = 512;

__device__ __forceinline__ uint32_t htile_off(int r, int k) {
  return (uint32_t)((r >> 3) * kHSBO + (k >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2);
}

struct FwdSmem {
  unsigned char h_tile[2][2 * kHSBO];  // h_{t-1} fp16 [16 env rows][512], by step parity
  float acc[kRows][kBMax];             // W_hh h_{t-1} for own rows
  float hown[kBMax][kUPC];             // fp32 h_in (masked) for own units
  float cown[kBMax][kUPC];             // fp32 c_in (masked)
  unsigned char stage[2][512];         // own new h slice [env][32] fp16, by parity
  float bias[kRows];                   // b_ih + b_hh of own rows
  uint64_t bar[2];
  uint64_t mma_bar;
  uint32_t tmem_slot;
};

__global__ void __launch_bounds__(kThreads, 1) lstm_fwd_kernel(LstmPtrs p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  FwdSmem& sm = *reinterpret_cast<FwdSmem*>(smem_raw);
  float* smask = reinterpret_cast<float*>(smem_raw + sizeof(FwdSmem));  // [B][T_run]
  const int c = (int)cluster_ctarank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int B = p.B, T_run = p.T_run, S = B * T_run;

  {
    uint4* zz = reinterpret_cast<uint4*>(sm.h_tile);
    for (int i = tid; i < (int)(sizeof(sm.h_tile) / 16); i += blockDim.x) zz[i] = make_uint4(0u, 0u, 0u, 0u);
  }
  for (int i = tid; i < kRows; i += blockDim.x) sm.bias[i] = p.bih[grow_of(c, i)] + p.bhh[grow_of(c, i)];
  for (int i = tid; i < S; i += blockDim.x) {
    const int b = i / T_run, t = i - b * T_run;
    smask[i] = p.mask[(size_t)p.env_idx[b] * p.ld + t];
  }
  if (tid == 0) {
    mbar_init(&sm.bar[0], 1);
    mbar_init(&sm.bar[1], 1);
    mbar_init(&sm.mma_bar, 8);  // one tcgen05.commit per issuing warp
    fence_mbar_init_cluster();
  }
  if (warp == 0) tmem_alloc<kFwdCols>(&sm.tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_slot;
  // A operand: warps w, w+4 share lane quarter w%4 (row r), split the 256 packed columns
  {
    const int r = (warp & 3) * 32 + lane;
    const float* wh = p.Whh + (size_t)grow_of(c, r) * kH;
    const int col_lo = (warp < 4) ? 0 : (int)kAcc0 / 2;
#pragma unroll 1
    for (int col0 = col_lo; col0 < col_lo + (int)kAcc0 / 2; col0 += 32) {
      float4 a[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) a[q] = *reinterpret_cast<const float4*>(wh + 2 * col0 + 4 * q);
#pragma unroll
      for (int sb = 0; sb < 4; ++sb) {
        uint32_t v[8];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          v[2 * q] = pack_f16(a[4 * sb + q].x, a[4 * sb + q].y);
          v[2 * q + 1] = pack_f16(a[4 * sb + q].z, a[4 * sb + q].w);
        }
        tmem_st8(tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(col0 + 8 * sb), v);
      }
    }
    tmem_wait_st();
  }
  for (int i = tid; i < B * kH; i += blockDim.x) {
    const int b = i / kH, k = i % kH;
    const int n = p.env_idx[b];
    const float h = smask[b * T_run] * p.h0[(size_t)n * p.sld + k];
    *reinterpret_cast<__half*>(sm.h_tile[0] + htile_off(b, k)) = __float2half(h);
    if (k >= c * kUPC && k < (c + 1) * kUPC) {
      sm.hown[b][k - c * kUPC] = h;
      sm.cown[b][k - c * kUPC] = smask[b * T_run] * p.c0[(size_t)n * p.sld + k];
    }
  }
  fence_proxy_async();
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();

  const int gu = lane, gb = warp;
  const bool gate_warp = warp < B;
  uint32_t pk_addr[2] = {0u, 0u}, pk_bar[2][2] = {{0u, 0u}, {0u, 0u}};
  const uint32_t tx_bytes = (uint32_t)(kNC * B * kUPC * sizeof(__half));
  float gi[4] = {0.f, 0.f, 0.f, 0.f};
  if (gate_warp) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const uint32_t q = (uint32_t)(lane / 4 + 8 * j);
      pk_addr[j] = map_to_cta(sm.h_tile[0] + htile_off(gb, c * kUPC + 8 * (lane % 4)), q);
      pk_bar[j][0] = map_to_cta(&sm.bar[0], q);
      pk_bar[j][1] = map_to_cta(&sm.bar[1], q);
    }
    const float* g0 = p.GI + (size_t)(gb * T_run) * kG4 + c * kUPC + gu;
#pragma unroll
    for (int q = 0; q < 4; ++q) gi[q] = g0[q * kH];
  }
  const uint32_t h_parity_bytes = (uint32_t)sizeof(sm.h_tile[0]);
  const uint32_t h_base0 = smem_u32(sm.h_tile[0]);
  for (int t = 0; t < T_run; ++t) {
    const int cur = t & 1;
    {  // all 8 warps issue (4 MMAs each, own accumulator: measured 8 x 4 beats 4 x 8, r02_rnn_floor.txt)
      if (t > 0) {
        if (tid == 0) mbar_arrive_expect_tx(&sm.bar[cur], tx_bytes);
        mbar_wait_parity(&sm.bar[cur], (uint32_t)(((t - 1) >> 1) & 1));
      }
      fence_proxy_async();
      tc_fence_after();
      const uint64_t bd0 = umma_desc(h_base0 + (uint32_t)cur * h_parity_bytes, 128, kHSBO);
      const uint32_t d_acc = tmem + kAcc0 + 16u * (uint32_t)warp;
#pragma unroll
      for (int j = 0; j < kH / 16 / 8; ++j) {
        const int kk = warp + 8 * j;
        mma_ts(d_acc, tmem + 8u * (uint32_t)kk, bd0 + (uint64_t)(16 * kk), kIdescF16_M128_N16, (uint32_t)j);
      }
      mma_commit(&sm.mma_bar);
    }
    if (warp < 4) {
      mbar_wait_parity(&sm.mma_bar, (uint32_t)(t & 1));
      tc_fence_after();
      uint32_t v[8][8];
#pragma unroll
      for (int a = 0; a < 8; ++a) tmem_ld8(tmem + ((uint32_t)(warp * 32) << 16) + kAcc0 + 16u * (uint32_t)a, v[a]);
      tmem_wait_ld();
      const int row = warp * 32 + lane;
      float s8[8];
#pragma unroll
      for (int e = 0; e < 8; ++e)
        s8[e] = ((__uint_as_float(v[0][e]) + __uint_as_float(v[1][e])) + (__uint_as_float(v[2][e]) + __uint_as_float(v[3][e]))) +
                ((__uint_as_float(v[4][e]) + __uint_as_float(v[5][e])) + (__uint_as_float(v[6][e]) + __uint_as_float(v[7][e])));
      *reinterpret_cast<float4*>(&sm.acc[row][0]) = make_float4(s8[0], s8[1], s8[2], s8[3]);
      *reinterpret_cast<float4*>(&sm.acc[row][4]) = make_float4(s8[4], s8[5], s8[6], s8[7]);
      tc_fence_before();
    }
    __syncthreads();
    if (gate_warp) {
      const float pi = sm.acc[gu][gb] + gi[0] + sm.bias[gu];
      const float pf = sm.acc[kUPC + gu][gb] + gi[1] + sm.bias[kUPC + gu];
      const float pg = sm.acc[2 * kUPC + gu][gb] + gi[2] + sm.bias[2 * kUPC + gu];
      const float po = sm.acc[3 * kUPC + gu][gb] + gi[3] + sm.bias[3 * kUPC + gu];
      const float ig = sigmoid_fast(pi), fg = sigmoid_fast(pf), gg = tanh_fast(pg), og = sigmoid_fast(po);
      const float h_in = sm.hown[gb][gu], c_in = sm.cown[gb][gu];
      const float cc = fg * c_in + ig * gg;
      const float h = og * tanh_fast(cc);
      if (t + 1 < T_run) {
        const float m = smask[gb * T_run + t + 1];
        sm.hown[gb][gu] = m * h;
        sm.cown[gb][gu] = m * cc;
        __half* stp = reinterpret_cast<__half*>(sm.stage[cur]) + gb * kUPC;
        stp[gu] = __float2half(m * h);
        __syncwarp();
        const uint4 pkt = *reinterpret_cast<const uint4*>(stp + 8 * (lane % 4));
        const uint32_t off = (cur ^ 1) * h_parity_bytes;
        st_async_v4(pk_addr[0] + off, pkt, pk_bar[0][cur ^ 1]);
        st_async_v4(pk_addr[1] + off, pkt, pk_bar[1][cur ^ 1]);
      }
      const size_t o = ((size_t)gb * T_run + t) * kH + c * kUPC + gu;
      p.Hs[o] = h;
      p.Hin[o] = h_in;
      p.Cin[o] = c_in;
      p.Cs[o] = cc;
      p.IFGO[o] = make_float4(ig, fg, gg, og);
      if (t + 1 < T_run) {
        const float* g0 = p.GI + (size_t)(gb * T_run + t + 1) * kG4 + c * kUPC + gu;
#pragma unroll
        for (int q = 0; q < 4; ++q) gi[q] = g0[q * kH];
      }
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 0) tmem_dealloc<kFwdCols>(tmem);
}

// ------------------------------------------------------------------ backward (BPTT)
constexpr uint32_t kDgSBO = (kRows / 8) * 128;  // 2048 B between 8-row groups of the [16 x 128] tile
constexpr uint32_t kBwdD0 = 4 * (kRows / 2);     // TMEM [0, 256): 4 tiles x 64 packed columns
constexpr int kBwdCols = 512;                    // + 8 accumulators x 16

struct BwdSmem {
  unsigned char dg_tile[2 * kDgSBO];  // dL/d(gates) (bf16) [16 env rows][128 own rows]
  float recv[2][kNC][kUPC][kBMax];
  uint64_t bar[2];
  uint64_t mma_bar;
  uint32_t tmem_slot;
};

__device__ __forceinline__ uint32_t dg_off(int n, int k) {
  return (uint32_t)((n >> 3) * kDgSBO + (k >> 3) * 128 + (n & 7) * 16 + (k & 7) * 2);
}

__global__ void __launch_bounds__(kThreads, 1) lstm_bwd_kernel(LstmPtrs p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  BwdSmem& sm = *reinterpret_cast<BwdSmem*>(smem_raw);
  float* smask = reinterpret_cast<float*>(smem_raw + sizeof(BwdSmem));
  const int c = (int)cluster_ctarank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int B = p.B, T_run = p.T_run, S = B * T_run;

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
    mbar_init(&sm.mma_bar, 8);
    fence_mbar_init_cluster();
  }
  if (warp == 0) tmem_alloc<kBwdCols>(&sm.tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_slot;
  // A operand: tile q (units 128q..), lane = unit, 64 packed columns of the 128 own gate rows
  {
    const int jl = (warp & 3) * 32 + lane;
#pragma unroll 1
    for (int q = (warp < 4 ? 0 : 2); q < (warp < 4 ? 2 : 4); ++q) {
      const float* wcol = p.Whh + 128 * q + jl;
#pragma unroll 1
      for (int lr0 = 0; lr0 < kRows; lr0 += 32) {
        float w[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) w[e] = wcol[(size_t)grow_of(c, lr0 + e) * kH];
#pragma unroll
        for (int sb = 0; sb < 2; ++sb) {
          uint32_t v[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) v[e] = pack_bf16(w[16 * sb + 2 * e], w[16 * sb + 2 * e + 1]);
          tmem_st8(tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(64 * q + lr0 / 2 + 8 * sb), v);
        }
      }
    }
    tmem_wait_st();
  }
  const uint32_t unit_bytes = B <= 2 ? 8u : (B <= 4 ? 16u : 32u);
  const int ustride = (int)unit_bytes / 4;
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
  fence_proxy_async();
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();

  const int gu = lane, gb = warp;
  const bool gate_warp = warp < B;
  float carry_h = 0.f, carry_c = 0.f;
  float dH_t = 0.f, c_t = 0.f, c_in = 0.f;
  float4 ifgo = make_float4(0.f, 0.f, 0.f, 0.f);
  if (gate_warp) {
    const size_t o = ((size_t)gb * T_run + T_run - 1) * kH + c * kUPC + gu;
    dH_t = p.dH[o];
    c_t = p.Cs[o];
    c_in = p.Cin[o];
    ifgo = p.IFGO[o];
  }
  for (int it = 0; it < T_run; ++it) {
    const int t = T_run - 1 - it, par = it & 1;
    if (gate_warp) {
      const float dh = dH_t + carry_h;
      const float ig = ifgo.x, fg = ifgo.y, gg = ifgo.z, og = ifgo.w;
      const float tc = tanhf(c_t);
      const float dc = dh * og * (1.f - tc * tc) + carry_c;
      const float d_i = dc * gg * ig * (1.f - ig);
      const float d_f = dc * c_in * fg * (1.f - fg);
      const float d_g = dc * ig * (1.f - gg * gg);
      const float d_o = dh * tc * og * (1.f - og);
      *reinterpret_cast<__nv_bfloat16*>(sm.dg_tile + dg_off(gb, gu)) = __float2bfloat16(d_i);
      *reinterpret_cast<__nv_bfloat16*>(sm.dg_tile + dg_off(gb, kUPC + gu)) = __float2bfloat16(d_f);
      *reinterpret_cast<__nv_bfloat16*>(sm.dg_tile + dg_off(gb, 2 * kUPC + gu)) = __float2bfloat16(d_g);
      *reinterpret_cast<__nv_bfloat16*>(sm.dg_tile + dg_off(gb, 3 * kUPC + gu)) = __float2bfloat16(d_o);
      fence_proxy_async();
      carry_c = smask[gb * T_run + t] * dc * fg;  // d c_{t-1} through c_in = mask_t c_{t-1}
      const size_t og4 = ((size_t)gb * T_run + t) * kG4 + c * kUPC + gu;
      p.dG[og4] = d_i;
      p.dG[og4 + kH] = d_f;
      p.dG[og4 + 2 * kH] = d_g;
      p.dG[og4 + 3 * kH] = d_o;
      if (t > 0) {
        const size_t o = ((size_t)gb * T_run + t - 1) * kH + c * kUPC + gu;
        dH_t = p.dH[o];
        c_t = p.Cs[o];
        c_in = p.Cin[o];
        ifgo = p.IFGO[o];
      }
    }
    __syncthreads();
    {
      tc_fence_after();
      const int q_mma = warp & 3, h = warp >> 2;
      const uint64_t bd0 = umma_desc(dg_base, 128, kDgSBO);
      const uint32_t d_q = tmem + kBwdD0 + 16u * (uint32_t)(2 * q_mma + h);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int kk = 4 * h + j;
        mma_ts(d_q, tmem + 64u * (uint32_t)q_mma + 8u * (uint32_t)kk, bd0 + (uint64_t)(16 * kk), kIdescBF16_M128_N16,
               (uint32_t)j);
      }
      mma_commit(&sm.mma_bar);
      mbar_wait_parity(&sm.mma_bar, (uint32_t)(it & 1));
      tc_fence_after();
      const uint32_t lane_base = tmem + ((uint32_t)((warp & 3) * 32) << 16) + kBwdD0;
      const uint32_t off = (uint32_t)par * recv_parity_bytes;
#pragma unroll
      for (int qi = 0; qi < 2; ++qi) {
        const int q = 2 * (warp >> 2) + qi;
        uint32_t a[8], b[8];
        tmem_ld8(lane_base + 32u * (uint32_t)q, a);
        tmem_ld8(lane_base + 32u * (uint32_t)q + 16u, b);
        tmem_wait_ld();
        float s[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) s[e] = __uint_as_float(a[e]) + __uint_as_float(b[e]);
        if (unit_bytes == 8u) {
          const float n0 = __shfl_down_sync(0xffffffffu, s[0], 1);
          const float n1 = __shfl_down_sync(0xffffffffu, s[1], 1);
          if ((lane & 1) == 0)
            st_async_v4(dst[qi] + off, make_uint4(__float_as_uint(s[0]), __float_as_uint(s[1]), __float_as_uint(n0),
                                                  __float_as_uint(n1)),
                        dbar[qi][par]);
        } else {
          st_async_v4(dst[qi] + off, make_uint4(__float_as_uint(s[0]), __float_as_uint(s[1]), __float_as_uint(s[2]),
                                                __float_as_uint(s[3])),
                      dbar[qi][par]);
          if (unit_bytes == 32u)
            st_async_v4(dst[qi] + off + 16u, make_uint4(__float_as_uint(s[4]), __float_as_uint(s[5]),
                                                        __float_as_uint(s[6]), __float_as_uint(s[7])),
                        dbar[qi][par]);
        }
      }
      tc_fence_before();
    }
    if (gate_warp) {
      if (tid == 0) mbar_arrive_expect_tx(&sm.bar[par], tx_bytes);
      mbar_wait_parity(&sm.bar[par], (uint32_t)((it >> 1) & 1));
      float s = 0.f;
#pragma unroll
      for (int q = 0; q < kNC; ++q) s += (&sm.recv[par][0][0][0])[(q * kUPC + gu) * ustride + gb];
      carry_h = smask[gb * T_run + t] * s;
    }
    __syncthreads();
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 0) tmem_dealloc<kBwdCols>(tmem);
}

template <typename K>
ddppo_status launch_cluster16(ddppo_ctx* ctx, K kernel, size_t smem, const LstmPtrs& p, cudaStream_t st) {
  DDPPO_CUDA_TRY(ctx, cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  DDPPO_CUDA_TRY(ctx, cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kNC, 1, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
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
  ctx->count(1);
  return DDPPO_OK;
}

}  // namespace

// recurrent FLOPs per launch: the W_hh contraction of every step, 2 * B * T * 4H * H
ddppo_status launch_lstm_fwd(ddppo_ctx* ctx, const LstmPtrs& p, cudaStream_t st) {
  DDPPO_REQUIRE(ctx, p.B >= 1 && p.B <= kBMax && p.T_run >= 1 && p.T_run <= 1024, "lstm: 1..8 envs, T <= 1024");
  DDPPO_REQUIRE(ctx, p.H == 512 || p.H == 1024, "lstm: hidden 512 or 1024");
  ProfScope ps(ctx, DDPPO_K_RNN, st, 0);
  if (ctx->prof) ctx->flops[DDPPO_K_RNN] += 2.0 * p.B * p.T_run * 4.0 * p.H * p.H;
  if (p.H == 1024) {
    LstmPtrs q = p;
    q.err = ctx->d_err;
    return launch_lstm1024_fwd(ctx, q, st);
  }
  return launch_cluster16(ctx, lstm_fwd_kernel, sizeof(FwdSmem) + (size_t)p.B * p.T_run * sizeof(float), p, st);
}

ddppo_status launch_lstm_bwd(ddppo_ctx* ctx, const LstmPtrs& p, cudaStream_t st) {
  DDPPO_REQUIRE(ctx, p.B >= 1 && p.B <= kBMax && p.T_run >= 1 && p.T_run <= 1024, "lstm: 1..8 envs, T <= 1024");
  DDPPO_REQUIRE(ctx, p.H == 512 || p.H == 1024, "lstm: hidden 512 or 1024");
  ProfScope ps(ctx, DDPPO_K_RNN, st, 0);
  if (ctx->prof) ctx->flops[DDPPO_K_RNN] += 2.0 * p.B * p.T_run * 4.0 * p.H * p.H;
  if (p.H == 1024) {
    LstmPtrs q = p;
    q.err = ctx->d_err;
    return launch_lstm1024_bwd(ctx, q, st);
  }
  return launch_cluster16(ctx, lstm_bwd_kernel, sizeof(BwdSmem) + (size_t)p.B * p.T_run * sizeof(float), p, st);
}
