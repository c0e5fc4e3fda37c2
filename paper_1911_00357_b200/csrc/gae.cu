// a2 GAE reverse-time scan (K1) and a3 advantage-normalisation finalize (K2).
//
// P:L218 (sec.4 Training): GAE, gamma = 0.99, tau = 0.95.  Per env n (include/ddppo.h):
//   delta_t = r_t + gamma V_{t+1} (1-d_t) - V_t ;  A_t = delta_t + gamma tau (1-d_t) A_{t+1}
// Design: one warp per env column, 128 time steps per warp pass (4 consecutive steps per lane,
// 16-byte loads).  The recurrence is an affine map A_t = D_t + C_t A_{t+1}; each lane composes
// its 4 maps, the warp does a Kogge-Stone suffix scan of (D, C) with __shfl_down_sync, and the
// carry A_{t0+128} links the 128-step chunks (processed last chunk first).  Memory-bound:
// 17 B/element algorithmic (r 4 + V 4 + done 1 + A 4 + R 4).  The epilogue accumulates
// {sum A, sum A^2, n} in fp64 and reduces them deterministically (block order) with the
// last-block pattern, so no second launch is needed.
#include "common.cuh"

namespace {

constexpr int kWarps = 8;  // warps per block

template <bool VEC>
__global__ void __launch_bounds__(kWarps * 32)
gae_kernel(const float* __restrict__ rew, const float* __restrict__ val, const uint8_t* __restrict__ done,
           const int32_t* __restrict__ len, int E, int T, int ld, float gamma, float tau,
           float* __restrict__ adv, float* __restrict__ ret, double* partials, unsigned int* counter,
           double* stats3) {
  pdl_enter();
  __shared__ double red[3 * kWarps];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const float gt = gamma * tau;
  double s = 0.0, q = 0.0, cnt = 0.0;
  const int n_chunks = (T + 127) / 128;
  for (int n = blockIdx.x * kWarps + warp; n < E; n += gridDim.x * kWarps) {
    const int L = min(max(len[n], 0), T);
    const size_t row = (size_t)n * ld;
    float carry = 0.f;  // A at the first step after the chunk
    for (int ch = n_chunks - 1; ch >= 0; --ch) {
      const int t0 = ch * 128 + lane * 4;
      float r[4] = {0.f, 0.f, 0.f, 0.f}, v[5] = {0.f, 0.f, 0.f, 0.f, 0.f};
      uint32_t dd = 0;
      // a lane loads if it holds a valid step or the bootstrap slot V_L
      if (t0 < T && t0 <= L) {
        if (VEC) {  // T % 4 == 0 and ld % 4 == 0: the float4 stays inside the row
          const float4 r4 = *reinterpret_cast<const float4*>(rew + row + t0);
          const float4 v4 = *reinterpret_cast<const float4*>(val + row + t0);
          dd = *reinterpret_cast<const uint32_t*>(done + row + t0);
          r[0] = r4.x; r[1] = r4.y; r[2] = r4.z; r[3] = r4.w;
          v[0] = v4.x; v[1] = v4.y; v[2] = v4.z; v[3] = v4.w;
        } else {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (t0 + k < T) {
              r[k] = rew[row + t0 + k];
              dd |= (uint32_t)done[row + t0 + k] << (8 * k);
            }
            if (t0 + k <= T) v[k] = val[row + t0 + k];
          }
        }
      }
      // V_{t0+4}: the next lane's v[0]; lane 31 and the ragged end load slot t0+4 (<= L <= T)
      float vn = __shfl_down_sync(0xffffffffu, v[0], 1);
      if ((lane == 31 || t0 + 4 >= T) && t0 + 4 <= L) vn = val[row + t0 + 4];
      v[4] = vn;
      float dl[4], c[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int t = t0 + k;
        const bool valid = t < L;
        const float nd = 1.f - (float)((dd >> (8 * k)) & 0xffu);
        const float vnext = (k < 3) ? v[k + 1] : v[4];
        dl[k] = valid ? (r[k] + gamma * vnext * nd - v[k]) : 0.f;
        c[k] = valid ? gt * nd : 0.f;
      }
      // compose the lane's 4 maps: A_{t0} = D + C * A_{t0+4}
      float D = dl[3], C = c[3];
#pragma unroll
      for (int k = 2; k >= 0; --k) {
        D = dl[k] + c[k] * D;
        C = c[k] * C;
      }
      // inclusive suffix scan over lanes: F_l = f_l o f_{l+1} o ... o f_31
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const float D2 = __shfl_down_sync(0xffffffffu, D, off);
        const float C2 = __shfl_down_sync(0xffffffffu, C, off);
        if (lane + off < 32) {
          D = D + C * D2;
          C = C * C2;
        }
      }
      const float a_start = D + C * carry;  // A_{t0}
      float a_next = __shfl_down_sync(0xffffffffu, a_start, 1);
      if (lane == 31) a_next = carry;
      float A[4];
      A[3] = dl[3] + c[3] * a_next;
#pragma unroll
      for (int k = 2; k >= 0; --k) A[k] = dl[k] + c[k] * A[k + 1];
      float R[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const bool valid = t0 + k < L;
        R[k] = valid ? A[k] + v[k] : 0.f;
        if (valid) {
          s += (double)A[k];
          q += (double)A[k] * (double)A[k];
          cnt += 1.0;
        }
      }
      if (t0 < T) {
        if (VEC) {
          *reinterpret_cast<float4*>(adv + row + t0) = make_float4(A[0], A[1], A[2], A[3]);
          *reinterpret_cast<float4*>(ret + row + t0) = make_float4(R[0], R[1], R[2], R[3]);
        } else {
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (t0 + k < T) {
              adv[row + t0 + k] = A[k];
              ret[row + t0 + k] = R[k];
            }
        }
      }
      carry = __shfl_sync(0xffffffffu, a_start, 0);
    }
  }
  if (stats3 == nullptr) return;
  double acc[3] = {s, q, cnt};
  last_block_reduce<3>(acc, partials, counter, stats3, red);
}

// Single-chunk fast path (T <= 128, 16-byte rows): each warp loads TWO env rows (its own and the
// row one grid-stride further) before scanning either, so twice the bytes are in flight per warp.
struct GaeRow {
  float r[4], v[5];
  uint32_t dd;
  int L;
};
__device__ __forceinline__ void gae_load(const float* __restrict__ rew, const float* __restrict__ val,
                                         const uint8_t* __restrict__ done, const int32_t* __restrict__ len, int n,
                                         int E, int T, int ld, int lane, GaeRow& g) {
#pragma unroll
  for (int k = 0; k < 4; ++k) g.r[k] = 0.f;
#pragma unroll
  for (int k = 0; k < 5; ++k) g.v[k] = 0.f;
  g.dd = 0;
  g.L = 0;
  if (n >= E) return;
  g.L = min(max(len[n], 0), T);
  const size_t row = (size_t)n * ld;
  const int t0 = lane * 4;
  if (t0 < T && t0 <= g.L) {
    const float4 r4 = *reinterpret_cast<const float4*>(rew + row + t0);
    const float4 v4 = *reinterpret_cast<const float4*>(val + row + t0);
    g.dd = *reinterpret_cast<const uint32_t*>(done + row + t0);
    g.r[0] = r4.x; g.r[1] = r4.y; g.r[2] = r4.z; g.r[3] = r4.w;
    g.v[0] = v4.x; g.v[1] = v4.y; g.v[2] = v4.z; g.v[3] = v4.w;
  }
  if ((lane == 31 || t0 + 4 >= T) && t0 + 4 <= g.L && t0 < T) g.v[4] = val[row + t0 + 4];  // bootstrap slot
}
__device__ __forceinline__ void gae_scan_store(const GaeRow& g, int n, int E, int T, int ld, int lane, float gamma,
                                               float gt, float* __restrict__ adv, float* __restrict__ ret, double& s,
                                               double& q, double& cnt) {
  const int t0 = lane * 4, L = g.L;
  const size_t row = (size_t)n * ld;
  float vn = __shfl_down_sync(0xffffffffu, g.v[0], 1);
  if (lane == 31 || t0 + 4 >= T) vn = g.v[4];
  float dl[4], c[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const bool valid = t0 + k < L;
    const float nd = 1.f - (float)((g.dd >> (8 * k)) & 0xffu);
    const float vnext = (k < 3) ? g.v[k + 1] : vn;
    dl[k] = valid ? (g.r[k] + gamma * vnext * nd - g.v[k]) : 0.f;
    c[k] = valid ? gt * nd : 0.f;
  }
  float D = dl[3], C = c[3];
#pragma unroll
  for (int k = 2; k >= 0; --k) {
    D = dl[k] + c[k] * D;
    C = c[k] * C;
  }
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const float D2 = __shfl_down_sync(0xffffffffu, D, off);
    const float C2 = __shfl_down_sync(0xffffffffu, C, off);
    if (lane + off < 32) {
      D = D + C * D2;
      C = C * C2;
    }
  }
  float a_next = __shfl_down_sync(0xffffffffu, D, 1);  // A_{t0+4} (carry 0 after the last chunk)
  if (lane == 31) a_next = 0.f;
  float A[4], R[4];
  A[3] = dl[3] + c[3] * a_next;
#pragma unroll
  for (int k = 2; k >= 0; --k) A[k] = dl[k] + c[k] * A[k + 1];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const bool valid = t0 + k < L;
    R[k] = valid ? A[k] + g.v[k] : 0.f;
    if (valid) {
      s += (double)A[k];
      q += (double)A[k] * (double)A[k];
      cnt += 1.0;
    }
  }
  if (n < E && t0 < T) {
    *reinterpret_cast<float4*>(adv + row + t0) = make_float4(A[0], A[1], A[2], A[3]);
    *reinterpret_cast<float4*>(ret + row + t0) = make_float4(R[0], R[1], R[2], R[3]);
  }
}

__global__ void __launch_bounds__(kWarps * 32)
gae1_kernel(const float* __restrict__ rew, const float* __restrict__ val, const uint8_t* __restrict__ done,
            const int32_t* __restrict__ len, int E, int T, int ld, float gamma, float tau, float* __restrict__ adv,
            float* __restrict__ ret, double* partials, unsigned int* counter, double* stats3) {
  pdl_enter();
  __shared__ double red[3 * kWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float gt = gamma * tau;
  double s = 0.0, q = 0.0, cnt = 0.0;
  const int stride = gridDim.x * kWarps;
  for (int n = blockIdx.x * kWarps + warp; n < E; n += 2 * stride) {
    GaeRow g0, g1;
    gae_load(rew, val, done, len, n, E, T, ld, lane, g0);
    gae_load(rew, val, done, len, n + stride, E, T, ld, lane, g1);
    gae_scan_store(g0, n, E, T, ld, lane, gamma, gt, adv, ret, s, q, cnt);
    if (n + stride < E) gae_scan_store(g1, n + stride, E, T, ld, lane, gamma, gt, adv, ret, s, q, cnt);
  }
  if (stats3 == nullptr) return;
  double acc[3] = {s, q, cnt};
  last_block_reduce<3>(acc, partials, counter, stats3, red);
}

__global__ void adv_finalize_kernel(const double* stats3, float eps, float* mean_invstd) {
  pdl_enter();
  if (threadIdx.x != 0) return;
  const double S = stats3[0], Q = stats3[1], n = stats3[2];
  const double mu = n > 0 ? S / n : 0.0;
  double var = n > 1 ? (Q - n * mu * mu) / (n - 1.0) : 0.0;
  if (var < 0) var = 0;
  mean_invstd[0] = (float)mu;
  mean_invstd[1] = (float)(1.0 / (sqrt(var) + (double)eps));
}

}  // namespace

ddppo_status launch_gae(ddppo_ctx* ctx, const float* rew, const float* val, const uint8_t* done,
                        const int32_t* len, int E, int T, int ld, float gamma, float tau, float* adv,
                        float* ret, double* stats3, cudaStream_t st) {
  DDPPO_REQUIRE(ctx, E >= 0 && T >= 1 && ld >= T + 1, "gae: need E >= 0, T >= 1, ld >= T+1");
  if (E == 0) {
    if (stats3) DDPPO_CUDA_TRY(ctx, cudaMemsetAsync(stats3, 0, 3 * sizeof(double), st));
    return DDPPO_OK;
  }
  const bool vec = (ld % 4 == 0) && (T % 4 == 0) && ((uintptr_t)rew % 16 == 0) && ((uintptr_t)val % 16 == 0) &&
                   ((uintptr_t)adv % 16 == 0) && ((uintptr_t)ret % 16 == 0) && ((uintptr_t)done % 4 == 0);
  const int blocks = grid_for(E, kWarps, ctx->sm_count * 8);
  ProfScope ps(ctx, DDPPO_K_GAE, st, 1);
  if (vec && T <= 128)
    launch_k(ctx, gae1_kernel, blocks, kWarps * 32, 0, st, rew, val, done, len, E, T, ld, gamma, tau, adv, ret,
             ctx->d_partials,
                                                ctx->d_counters + CNT_GAE, stats3);
  else if (vec)
    launch_k(ctx, gae_kernel<true>, blocks, kWarps * 32, 0, st, rew, val, done, len, E, T, ld, gamma, tau, adv, ret,
                                                     ctx->d_partials, ctx->d_counters + CNT_GAE, stats3);
  else
    launch_k(ctx, gae_kernel<false>, blocks, kWarps * 32, 0, st, rew, val, done, len, E, T, ld, gamma, tau, adv, ret,
                                                      ctx->d_partials, ctx->d_counters + CNT_GAE, stats3);
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  return DDPPO_OK;
}

ddppo_status launch_adv_finalize(ddppo_ctx* ctx, const double* stats3, float eps, float* mean_invstd,
                                 cudaStream_t st) {
  ProfScope ps(ctx, DDPPO_K_ADV_NORM, st, 1);
  launch_k(ctx, adv_finalize_kernel, 1, 32, 0, st, stats3, eps, mean_invstd);
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  return DDPPO_OK;
}
