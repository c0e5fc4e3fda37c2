// Depth agent (BASELINE configs[2]): 64x64 depth -> half-width ResNet18 with GroupNorm -> 128x2x2
// -> FC 512 + ReLU; x = [visual, goal FC 32, action embedding 32] -> LSTM-512 -> Linear(512, 5).
// (P:L212 half-width backbone with GroupNorm, App. C; readings Z17-Z23 in DESIGN.md.)
//
// Layout: activations fp32 NHWC [frames][H][W][C] in the workspace, frames f = b*T_run + t.
// Convolutions are implicit GEMMs on the tcgen05 kernel of gemm_tc.cu (the im2col matrix is
// gathered while operand tiles are staged, never written; fp32 TMEM accumulation):
//   fprop  Y[q][o]   = sum_kk col(x)[q][kk] Wr[o][kk]          (kk = (u, v, c); bf16x3 operands)
//   dgrad  dX[p][c]  = sum_kk colT(dY)[p][kk] Wd[c][kk]        (kk = (u, v, o); transposed taps)
//   wgrad  dWr[o][kk] = sum_q dY[q][o] col(x)[q][kk]           (split-K over output pixels)
// GroupNorm (G = 16, eps 1e-5) statistics / apply (+ residual, + ReLU) / backward and the 3x3/2
// max-pool are fp32 SIMT kernels (HBM-bound), with every reduction in a fixed order.
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "common.cuh"

namespace {

constexpr int kH = 512, kG4 = 2048, kXin = 576, kA1 = 5, kGroups = 16, kThreads = 256;
constexpr int kImg = 64;  // input resolution (configs[2])

// ------------------------------------------------------------------ kernels
// obs [E][T][1][64][64] (gathered through env_idx) -> x0 [F][64][64][1]
__global__ void gather_obs_kernel(const float* __restrict__ obs, const int32_t* __restrict__ env_idx, int T, int T_run,
                                  int F, float* __restrict__ x0) {
  const size_t per = (size_t)kImg * kImg;
  const size_t n = (size_t)F * per;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int f = (int)(i / per);
    const int b = f / T_run, t = f - b * T_run;
    x0[i] = obs[((size_t)env_idx[b] * T + t) * per + (i % per)];
  }
}

// Weight layouts for the implicit GEMMs.  W [Co][Ci][k][k] (PyTorch) ->
//   Wr [Co][(u, v, c)] as bf16 hi / lo planes (plane = Co*k*k*Ci elements)  (forward B operand)
//   Wd [Ci][(u, v, o)] bf16                                                (input-gradient B operand)
__global__ void weights_bf16_kernel(const float* __restrict__ W, int Co, int Ci, int k, __nv_bfloat16* __restrict__ wr,
                                    __nv_bfloat16* __restrict__ wd) {
  const int n = Co * Ci * k * k;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int o = i / (Ci * k * k), rem = i % (Ci * k * k);
    const int c = rem / (k * k), uv = rem % (k * k);
    const float w = W[i];
    const __nv_bfloat16 hi = __float2bfloat16_rn(w);
    if (wr) {
      wr[o * (k * k * Ci) + uv * Ci + c] = hi;
      wr[n + o * (k * k * Ci) + uv * Ci + c] = __float2bfloat16_rn(w - __bfloat162float(hi));
    }
    if (wd) wd[c * (k * k * Co) + uv * Co + o] = hi;
  }
}
// all convolutions' weights of one minibatch in one launch (blockIdx.y = convolution)
constexpr int kMaxConvs = 24;
struct WeightPrep {
  int n;
  struct Item {
    const float* W;
    __nv_bfloat16 *wr, *wd;
    int Co, Ci, k;
  } it[kMaxConvs];
};
__global__ void weights_prep_kernel(const WeightPrep prep) {
  const WeightPrep::Item& t = prep.it[blockIdx.y];
  const int Co = t.Co, Ci = t.Ci, k = t.k, n = Co * Ci * k * k;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int o = i / (Ci * k * k), rem = i % (Ci * k * k);
    const int c = rem / (k * k), uv = rem % (k * k);
    const float w = t.W[i];
    const __nv_bfloat16 hi = __float2bfloat16_rn(w);
    t.wr[o * (k * k * Ci) + uv * Ci + c] = hi;
    t.wr[n + o * (k * k * Ci) + uv * Ci + c] = __float2bfloat16_rn(w - __bfloat162float(hi));
    t.wd[c * (k * k * Co) + uv * Co + o] = hi;
  }
}
// weight gradient: dWt [(u, v, c)][o] (the wgrad GEMM's output) -> dW [Co][Ci][k][k]
__global__ void wgrad_to_torch_kernel(const float* __restrict__ dwt, int Co, int Ci, int k, float* __restrict__ dw) {
  const int n = Co * Ci * k * k;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int o = i / (Ci * k * k), rem = i % (Ci * k * k);
    const int c = rem / (k * k), uv = rem % (k * k);
    dw[i] = dwt[(size_t)(uv * Ci + c) * Co + o];
  }
}
// fp32 -> bf16 hi / lo planes (plane = n)
__global__ void to_planes_kernel(const float* __restrict__ x, size_t n, __nv_bfloat16* __restrict__ xb) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const __nv_bfloat16 hi = __float2bfloat16_rn(x[i]);
    xb[i] = hi;
    xb[n + i] = __float2bfloat16_rn(x[i] - __bfloat162float(hi));
  }
}
__global__ void to_bf16_kernel(const float* __restrict__ x, size_t n, __nv_bfloat16* __restrict__ xb) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    xb[i] = __float2bfloat16_rn(x[i]);
}

// Single-channel stem convolution in fp32 SIMT (K = k*k taps over 1 channel is too narrow for the
// 16-byte implicit-GEMM pieces): block per frame, the frame and the weights staged in shared
// memory; a thread computes 4 horizontally adjacent pixels x 8 output channels per work item, so
// every weight load (float4 x 2, broadcast) feeds 32 FMAs.
constexpr int kStemCoMax = 32;
__global__ void __launch_bounds__(kThreads) stem_fwd_kernel(const float* __restrict__ x, const float* __restrict__ W,
                                                            int H, int Wd, int Co, int k, int s, int p, int Ho, int Wo,
                                                            float* __restrict__ y) {
  extern __shared__ __align__(16) float sm[];
  const int kk = k * k;
  float* ws = sm;                   // [k*k][Co]   (Co % 8 == 0)
  float* xs = sm + kk * Co;         // [H][Wd]
  const int f = blockIdx.x;
  for (int i = threadIdx.x; i < H * Wd; i += blockDim.x) xs[i] = x[(size_t)f * H * Wd + i];
  for (int i = threadIdx.x; i < Co * kk; i += blockDim.x) ws[(i % kk) * Co + i / kk] = W[i];
  __syncthreads();
  const int og = Co / 8, jg = (Wo + 3) / 4;
  for (int item = threadIdx.x; item < Ho * jg * og; item += blockDim.x) {
    const int o0 = (item % og) * 8, rest = item / og, j0 = (rest % jg) * 4, i = rest / jg;
    float acc[4][8];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int o = 0; o < 8; ++o) acc[a][o] = 0.f;
    for (int u = 0; u < k; ++u) {
      const int yy = i * s - p + u;
      if (yy < 0 || yy >= H) continue;
      for (int v = 0; v < k; ++v) {
        const float4 w0 = *reinterpret_cast<const float4*>(ws + (u * k + v) * Co + o0);
        const float4 w1 = *reinterpret_cast<const float4*>(ws + (u * k + v) * Co + o0 + 4);
        const float wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          const int xx = (j0 + a) * s - p + v;
          const float xv = (xx >= 0 && xx < Wd) ? xs[yy * Wd + xx] : 0.f;
#pragma unroll
          for (int o = 0; o < 8; ++o) acc[a][o] = fmaf(xv, wv[o], acc[a][o]);
        }
      }
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      if (j0 + a >= Wo) break;
      float* yo = y + (((size_t)f * Ho + i) * Wo + j0 + a) * Co + o0;
      *reinterpret_cast<float4*>(yo) = make_float4(acc[a][0], acc[a][1], acc[a][2], acc[a][3]);
      *reinterpret_cast<float4*>(yo + 4) = make_float4(acc[a][4], acc[a][5], acc[a][6], acc[a][7]);
    }
  }
}
// per-frame partial weight gradient of the stem: part[f][o*k*k + tap] = sum_q dy[f][q][o] col[q][tap],
// pixels in chunks of kStemPix: the chunk's im2col rows and dy rows are staged in shared memory;
// lane = output channel, warps stride over taps (pixel order fixed)
constexpr int kStemPix = 128, kStemTapPad = 65;
__global__ void __launch_bounds__(kThreads) stem_wgrad_kernel(const float* __restrict__ x,
                                                              const __nv_bfloat16* __restrict__ dy, int H, int Wd,
                                                              int Co, int k, int s, int p, int Ho, int Wo,
                                                              float* __restrict__ part) {
  extern __shared__ __align__(16) float sm[];
  float* xs = sm;                               // [H][Wd]
  float* cs = xs + H * Wd;                      // [kStemPix][kStemTapPad]
  float* ds = cs + kStemPix * kStemTapPad;      // [kStemPix][Co]
  const int f = blockIdx.x, kk = k * k, lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = threadIdx.x; i < H * Wd; i += blockDim.x) xs[i] = x[(size_t)f * H * Wd + i];
  constexpr int kMaxT = 8;  // taps per warp (k*k <= 64)
  float acc[kMaxT];
#pragma unroll
  for (int t = 0; t < kMaxT; ++t) acc[t] = 0.f;
  for (int q0 = 0; q0 < Ho * Wo; q0 += kStemPix) {
    const int nq = min(kStemPix, Ho * Wo - q0);
    __syncthreads();  // xs staged / previous chunk consumed
    // im2col rows of the chunk: thread pair per pixel (no division in the tap loops)
    for (int e = threadIdx.x; e < 2 * nq; e += blockDim.x) {
      const int q = e >> 1, half = e & 1;
      const int i = (q0 + q) / Wo, j = (q0 + q) - i * Wo;
      for (int u = half; u < k; u += 2) {
        const int yy = i * s - p + u;
        const bool yok = yy >= 0 && yy < H;
        for (int v = 0; v < k; ++v) {
          const int xx = j * s - p + v;
          cs[q * kStemTapPad + u * k + v] = (yok && xx >= 0 && xx < Wd) ? xs[yy * Wd + xx] : 0.f;
        }
      }
    }
    for (int e = threadIdx.x; e < nq * Co; e += blockDim.x)
      ds[e] = __bfloat162float(dy[((size_t)f * Ho * Wo + q0) * Co + e]);
    __syncthreads();
    if (lane < Co) {
      for (int q = 0; q < nq; ++q) {
        const float d = ds[q * Co + lane];
#pragma unroll
        for (int t = 0; t < kMaxT; ++t) {
          const int tap = warp + t * nw;
          if (tap < kk) acc[t] = fmaf(d, cs[q * kStemTapPad + tap], acc[t]);
        }
      }
    }
  }
  if (lane < Co) {
#pragma unroll
    for (int t = 0; t < kMaxT; ++t) {
      const int tap = warp + t * nw;
      if (tap < kk) part[(size_t)f * Co * kk + lane * kk + tap] = acc[t];
    }
  }
}
// dW[i] = sum over frames (fixed order) of part[f][i]
__global__ void __launch_bounds__(kThreads) frame_sum_kernel(const float* __restrict__ part, int F, int n,
                                                             float* __restrict__ out) {
  __shared__ double red[kThreads / 32];
  double acc[1] = {0.0};
  for (int f = threadIdx.x; f < F; f += blockDim.x) acc[0] += part[(size_t)f * n + blockIdx.x];
  block_sum<1>(acc, red);
  if (threadIdx.x == 0) out[blockIdx.x] = (float)acc[0];
}

// GroupNorm (G = 16, eps 1e-5), one block per frame.  The block walks the frame's [HW][C] slab
// contiguously (coalesced); with 256 % C == 0 thread t always sees channel t % C, so per-group and
// per-channel partial sums are per-thread sums combined in a fixed order through shared memory.
constexpr int kGnThreads = 256;

// per-group sums of the threads' (a, b) in fixed order -> out[g] (threads t < 16 write)
__device__ __forceinline__ void gn_group_reduce(double a, double b, int C, double* sa, double* sb, double* out_a,
                                                double* out_b) {
  sa[threadIdx.x] = a;
  sb[threadIdx.x] = b;
  __syncthreads();
  if (threadIdx.x < kGroups) {
    const int cg = C / kGroups, g = threadIdx.x;
    double ra = 0.0, rb = 0.0;
    for (int rep = 0; rep < kGnThreads / C; ++rep)
      for (int cc = 0; cc < cg; ++cc) {
        const int t = rep * C + g * cg + cc;
        ra += sa[t];
        rb += sb[t];
      }
    out_a[g] = ra;
    out_b[g] = rb;
  }
  __syncthreads();
}

// z = (relu)(gamma * (y - mu) * rstd + beta (+ residual)); stats[f][g] = (mu, rstd) (biased variance);
// zb (nullable): z as bf16 hi / lo planes (plane = F*HW*C)
__global__ void __launch_bounds__(kGnThreads) gn_fwd_kernel(const float* __restrict__ y, const float* __restrict__ gamma,
                                                            const float* __restrict__ beta,
                                                            const float* __restrict__ residual, int HW, int C,
                                                            int relu, size_t plane, float* __restrict__ stats,
                                                            float* __restrict__ z, __nv_bfloat16* __restrict__ zb) {
  __shared__ double sa[kGnThreads], sb[kGnThreads], ga[kGroups], gb[kGroups];
  __shared__ float smu[kGroups], srs[kGroups];
  const int f = blockIdx.x, n = HW * C, c = threadIdx.x % C, cg = C / kGroups;
  const size_t base = (size_t)f * n;
  double s1 = 0.0, s2 = 0.0;
  for (int e = threadIdx.x; e < n; e += kGnThreads) {
    const float v = y[base + e];
    s1 += v;
    s2 += (double)v * v;
  }
  gn_group_reduce(s1, s2, C, sa, sb, ga, gb);
  if (threadIdx.x < kGroups) {
    const double cnt = (double)HW * cg, mu = ga[threadIdx.x] / cnt;
    double var = gb[threadIdx.x] / cnt - mu * mu;
    if (var < 0) var = 0;
    smu[threadIdx.x] = (float)mu;
    srs[threadIdx.x] = (float)(1.0 / sqrt(var + 1e-5));
    stats[(f * kGroups + threadIdx.x) * 2] = smu[threadIdx.x];
    stats[(f * kGroups + threadIdx.x) * 2 + 1] = srs[threadIdx.x];
  }
  __syncthreads();
  const float mu = smu[c / cg], rs = srs[c / cg], gm = gamma[c], bt = beta[c];
  for (int e = threadIdx.x; e < n; e += kGnThreads) {
    const size_t i = base + e;
    float v = (y[i] - mu) * rs * gm + bt;
    if (residual) v += residual[i];
    v = relu ? fmaxf(v, 0.f) : v;
    z[i] = v;
    if (zb) {  // bf16 hi / lo planes: the next convolution's operand
      const __nv_bfloat16 hi = __float2bfloat16_rn(v);
      zb[i] = hi;
      zb[plane + i] = __float2bfloat16_rn(v - __bfloat162float(hi));
    }
  }
}

// dy_eff = dz * [z > 0] (relu_z nullable): GN backward per group
//   dx = rstd * (dxhat - mean(dxhat) - xhat * mean(dxhat * xhat)),   dxhat = dy_eff * gamma
// written as bf16 (it only feeds the bf16 gradient GEMMs), plus this frame's per-channel partials
// part[f][c] = (sum dy_eff * xhat, sum dy_eff) for dgamma / dbeta.
__global__ void __launch_bounds__(kGnThreads) gn_bwd_kernel(const float* __restrict__ dz, const float* __restrict__ z,
                                                            const float* __restrict__ y,
                                                            const float* __restrict__ stats,
                                                            const float* __restrict__ gamma, int HW, int C,
                                                            __nv_bfloat16* __restrict__ dx, float* __restrict__ part) {
  __shared__ double sa[kGnThreads], sb[kGnThreads], ga[kGroups], gb[kGroups];
  __shared__ float pc[2][kGnThreads];
  const int f = blockIdx.x, n = HW * C, c = threadIdx.x % C, cg = C / kGroups, g = c / cg;
  const size_t base = (size_t)f * n;
  const float mu = stats[(f * kGroups + g) * 2], rs = stats[(f * kGroups + g) * 2 + 1], gm = gamma[c];
  double a1 = 0.0, a2 = 0.0;
  float pg = 0.f, pb = 0.f;
  for (int e = threadIdx.x; e < n; e += kGnThreads) {
    const size_t i = base + e;
    float d = dz[i];
    if (z && z[i] <= 0.f) d = 0.f;
    const float xh = (y[i] - mu) * rs, dxh = d * gm;
    a1 += dxh;
    a2 += (double)dxh * xh;
    pg += d * xh;
    pb += d;
  }
  pc[0][threadIdx.x] = pg;
  pc[1][threadIdx.x] = pb;
  gn_group_reduce(a1, a2, C, sa, sb, ga, gb);  // (its barriers also publish pc)
  if (threadIdx.x < C) {
    float rg = 0.f, rb = 0.f;
    for (int t = threadIdx.x; t < kGnThreads; t += C) {
      rg += pc[0][t];
      rb += pc[1][t];
    }
    part[((size_t)f * C + threadIdx.x) * 2] = rg;
    part[((size_t)f * C + threadIdx.x) * 2 + 1] = rb;
  }
  const double cnt = (double)HW * cg;
  const float m1 = (float)(ga[g] / cnt), m2 = (float)(gb[g] / cnt);
  for (int e = threadIdx.x; e < n; e += kGnThreads) {
    const size_t i = base + e;
    float d = dz[i];
    if (z && z[i] <= 0.f) d = 0.f;
    const float xh = (y[i] - mu) * rs;
    dx[i] = __float2bfloat16_rn(rs * (d * gm - m1 - xh * m2));
  }
}

// dgamma[c], dbeta[c] = sums over frames (in frame order, blocked: thread t takes frames t, t+256,
// ...; then the fixed-order block reduction) of the per-frame partials
__global__ void __launch_bounds__(kThreads) gn_param_reduce_kernel(const float* __restrict__ part, int F, int C,
                                                                   float* __restrict__ dgamma,
                                                                   float* __restrict__ dbeta) {
  __shared__ double red[2 * (kThreads / 32)];
  const int c = blockIdx.x;
  double acc[2] = {0.0, 0.0};
  for (int f = threadIdx.x; f < F; f += blockDim.x) {
    acc[0] += part[((size_t)f * C + c) * 2];
    acc[1] += part[((size_t)f * C + c) * 2 + 1];
  }
  block_sum<2>(acc, red);
  if (threadIdx.x == 0) {
    dgamma[c] = (float)acc[0];
    dbeta[c] = (float)acc[1];
  }
}

// 3x3 / stride 2 / pad 1 max pool with the first maximum in (u, v) order
__global__ void maxpool_fwd_kernel(const float* __restrict__ x, int F, int H, int W, int C, int Ho, int Wo,
                                   float* __restrict__ y, uint8_t* __restrict__ arg, __nv_bfloat16* __restrict__ yb) {
  const size_t n = (size_t)F * Ho * Wo * C;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    const size_t pix = i / C;
    const int j = (int)(pix % Wo), ii = (int)((pix / Wo) % Ho), f = (int)(pix / ((size_t)Wo * Ho));
    float best = -INFINITY;
    int ba = 0;
    for (int u = 0; u < 3; ++u)
      for (int v = 0; v < 3; ++v) {
        const int yy = 2 * ii - 1 + u, xx = 2 * j - 1 + v;
        if (yy < 0 || yy >= H || xx < 0 || xx >= W) continue;
        const float val = x[(((size_t)f * H + yy) * W + xx) * C + c];
        if (val > best) {
          best = val;
          ba = u * 3 + v;
        }
      }
    y[i] = best;
    arg[i] = (uint8_t)ba;
    if (yb) {
      const __nv_bfloat16 hi = __float2bfloat16_rn(best);
      yb[i] = hi;
      yb[n + i] = __float2bfloat16_rn(best - __bfloat162float(hi));
    }
  }
}
// dx[f][y][x][c] = sum over windows whose argmax is (y, x) of dy (gather, fixed order)
__global__ void maxpool_bwd_kernel(const float* __restrict__ dy, const uint8_t* __restrict__ arg, int F, int H, int W,
                                   int C, int Ho, int Wo, float* __restrict__ dx) {
  const size_t n = (size_t)F * H * W * C;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    const size_t pix = i / C;
    const int xx = (int)(pix % W), y = (int)((pix / W) % H), f = (int)(pix / ((size_t)W * H));
    float acc = 0.f;
    for (int u = 0; u < 3; ++u) {
      const int yy = y + 1 - u;
      if (yy < 0 || (yy & 1)) continue;
      const int ii = yy >> 1;
      if (ii >= Ho) continue;
      for (int v = 0; v < 3; ++v) {
        const int xv = xx + 1 - v;
        if (xv < 0 || (xv & 1)) continue;
        const int j = xv >> 1;
        if (j >= Wo) continue;
        const size_t o = (((size_t)f * Ho + ii) * Wo + j) * C + c;
        if (arg[o] == u * 3 + v) acc += dy[o];
      }
    }
    dx[i] = acc;
  }
}

// NHWC [F][2][2][128] <-> flat [F][512] in (c, h, w) order (PyTorch flatten of NCHW)
__global__ void flatten_kernel(const float* __restrict__ in, int F, float* __restrict__ out, int to_flat) {
  const size_t n = (size_t)F * 512;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int f = (int)(i / 512), q = (int)(i % 512);
    const int c = q / 4, hw = q % 4;
    const size_t nhwc = (size_t)f * 512 + hw * 128 + c;
    if (to_flat) out[i] = in[nhwc];
    else out[nhwc] = in[i];
  }
}

// y[m][n] = act(y[m][n] + bias[n])   (act: 1 = ReLU)
__global__ void bias_act_kernel(float* __restrict__ y, const float* __restrict__ bias, int M, int N, int relu) {
  const size_t n = (size_t)M * N;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float v = y[i] + bias[i % N];
    y[i] = relu ? fmaxf(v, 0.f) : v;
  }
}

// x[s] = [visual (512), goal_fc(goal) (32), emb(prev_action) (32)]
__global__ void lstm_input_kernel(const float* __restrict__ vis, const float* __restrict__ goal,
                                  const int32_t* __restrict__ prev_action, const int32_t* __restrict__ env_idx,
                                  const float* __restrict__ Wg, const float* __restrict__ bg,
                                  const float* __restrict__ Emb, int T, int ld, int T_run, int S, float* __restrict__ x) {
  const size_t n = (size_t)S * kXin;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int s = (int)(i / kXin), k = (int)(i % kXin);
    float v;
    if (k < 512) {
      v = vis[(size_t)s * 512 + k];
    } else {
      const int b = s / T_run, t = s - b * T_run, e = env_idx[b];
      if (k < 544) {
        const int j = k - 512;
        const float* g = goal + ((size_t)e * T + t) * 3;
        v = Wg[j * 3] * g[0] + Wg[j * 3 + 1] * g[1] + Wg[j * 3 + 2] * g[2] + bg[j];
      } else {
        v = Emb[prev_action[(size_t)e * ld + t] * 32 + (k - 544)];
      }
    }
    x[i] = v;
  }
}

// from dx [S][576]: dVpre = dx[:, :512] * [vis > 0] (in place into dvis); goal FC and embedding
// gradients (block per output, fixed-order block reduction over samples)
__global__ void vis_mask_kernel(const float* __restrict__ dx, const float* __restrict__ vis, int S,
                                float* __restrict__ dvis) {
  const size_t n = (size_t)S * 512;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const size_t s = i / 512, k = i % 512;
    dvis[i] = vis[i] > 0.f ? dx[s * kXin + k] : 0.f;
  }
}
__global__ void __launch_bounds__(kThreads) goal_emb_grads_kernel(const float* __restrict__ dx,
                                                                  const float* __restrict__ goal,
                                                                  const int32_t* __restrict__ prev_action,
                                                                  const int32_t* __restrict__ env_idx, int T, int ld,
                                                                  int T_run, int S, float* __restrict__ dWg,
                                                                  float* __restrict__ dbg, float* __restrict__ dEmb) {
  __shared__ double red[kA1 * (kThreads / 32)];
  const int j = blockIdx.x;  // 0..63: 0..31 goal units, 32..63 embedding dims
  double acc[kA1] = {0, 0, 0, 0, 0};
  for (int s = threadIdx.x; s < S; s += blockDim.x) {
    const int b = s / T_run, t = s - b * T_run, e = env_idx[b];
    const float d = dx[(size_t)s * kXin + 512 + j];
    if (j < 32) {
      const float* g = goal + ((size_t)e * T + t) * 3;
      acc[0] += d * g[0];
      acc[1] += d * g[1];
      acc[2] += d * g[2];
      acc[3] += d;
    } else {
      const int a = prev_action[(size_t)e * ld + t];
      acc[a] += d;
    }
  }
  block_sum<kA1>(acc, red);
  if (threadIdx.x == 0) {
    if (j < 32) {
      dWg[j * 3] = (float)acc[0];
      dWg[j * 3 + 1] = (float)acc[1];
      dWg[j * 3 + 2] = (float)acc[2];
      dbg[j] = (float)acc[3];
    } else {
      for (int a = 0; a < kA1; ++a) dEmb[a * 32 + (j - 32)] = (float)acc[a];
    }
  }
}

__global__ void relu_mask_kernel(const float* __restrict__ dz, const float* __restrict__ z, size_t n,
                                 float* __restrict__ out) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    out[i] = z[i] > 0.f ? dz[i] : 0.f;
}


// ------------------------------------------------------------------ network plan
struct ConvGN {
  int Ci, Co, k, s, p, H, W, Ho, Wo;  // input H x W, output Ho x Wo
  int64_t w, gw, gb;                  // parameter offsets (conv weight, GN gamma, GN beta)
  float *x, *y, *z, *stats;           // input (not owned), conv out (pre-GN), GN out, GN stats [F][16][2]
  __nv_bfloat16 *xb, *zb;             // input / output as bf16 hi / lo planes (GEMM operands; zb may be null)
  __nv_bfloat16 *wr_b, *wd_b;         // this minibatch's weights as GEMM operands (Wr planes, Wd)
};

struct Plan {
  int F = 0;
  std::vector<ConvGN> convs;  // stem, per block: conv1, conv2, [down], compress
  struct Block {
    int c1, c2, down;        // indices into convs (down = -1: identity shortcut)
    float *in, *out;         // block input, block output (after residual + ReLU)
  };
  std::vector<Block> blocks;
  float *x0, *pool_out;
  __nv_bfloat16* pool_b;
  uint8_t* pool_arg;
  float *flat, *vis, *xin, *GI;
  float *Hs, *Hin, *Cin, *Cs, *IFGO, *dH, *dG;
  // scratch (reused by every layer)
  __nv_bfloat16 *wr_b, *wd_b, *dyb;   // weights as GEMM operands; GN-backward output (bf16)
  float *dwt, *part, *gn_part, *dz_a, *dz_b, *dz_c, *dxin, *dflat, *dvis;
  size_t bytes = 0;
};

int64_t off_of(const ModelLayout& L, const std::string& n) { return layout_offset(L, n.c_str()); }

constexpr int kMaxSplits = 64;

// Deterministic carve of the workspace (base == nullptr: size only)
void make_plan(const ModelLayout& L, int B, int T_run, void* base, Plan* plan) {
  Plan& P = *plan;
  P = Plan();
  const int F = B * T_run;
  P.F = F;
  size_t off = 0;
  auto take_bytes = [&](size_t bytes) {
    char* p = base ? reinterpret_cast<char*>(base) + off : nullptr;
    off = align_up(off + bytes, 256);
    return p;
  };
  auto take = [&](size_t n) { return reinterpret_cast<float*>(take_bytes(n * sizeof(float))); };
  auto take_b = [&](size_t n) { return reinterpret_cast<__nv_bfloat16*>(take_bytes(n * sizeof(__nv_bfloat16))); };
  size_t max_act = 0, max_w = 0;
  auto add_conv = [&](const std::string& cname, const std::string& gname, int Ci, int Co, int k, int s, int p, int H,
                      int W, float* x, __nv_bfloat16* xb, bool planes_out) {
    ConvGN c;
    c.Ci = Ci;
    c.Co = Co;
    c.k = k;
    c.s = s;
    c.p = p;
    c.H = H;
    c.W = W;
    c.Ho = (H + 2 * p - k) / s + 1;
    c.Wo = (W + 2 * p - k) / s + 1;
    c.w = off_of(L, cname + ".weight");
    c.gw = off_of(L, gname + ".weight");
    c.gb = off_of(L, gname + ".bias");
    c.x = x;
    c.xb = xb;
    const size_t act = (size_t)F * c.Ho * c.Wo * Co;
    c.y = take(act);
    c.z = take(act);
    c.zb = planes_out ? take_b(2 * act) : nullptr;
    c.stats = take((size_t)F * kGroups * 2);
    const size_t nw = (size_t)Co * k * k * Ci;
    c.wr_b = Ci > 1 ? take_b(2 * nw) : nullptr;
    c.wd_b = Ci > 1 ? take_b(nw) : nullptr;
    max_act = std::max(max_act, std::max(act, (size_t)F * H * W * Ci));
    max_w = std::max(max_w, (size_t)Co * k * k * Ci);
    P.convs.push_back(c);
    return (int)P.convs.size() - 1;
  };
  P.x0 = take((size_t)F * kImg * kImg);
  const int stem = add_conv("enc.stem.conv", "enc.stem.gn", 1, 32, 7, 2, 3, kImg, kImg, P.x0, nullptr, false);
  const int hs = P.convs[stem].Ho;  // 32
  const int hp = (hs + 2 - 3) / 2 + 1;  // 16
  P.pool_out = take((size_t)F * hp * hp * 32);
  P.pool_b = take_b((size_t)2 * F * hp * hp * 32);
  P.pool_arg = reinterpret_cast<uint8_t*>(take_bytes((size_t)F * hp * hp * 32));
  float* z = P.pool_out;
  __nv_bfloat16* zb = P.pool_b;
  int H = hp, cin = 32;
  const int widths[4] = {32, 64, 128, 256};
  for (int li = 0; li < 4; ++li) {
    for (int bi = 0; bi < 2; ++bi) {
      const int s = (bi == 0 && li > 0) ? 2 : 1, c = widths[li];
      const std::string pre = "enc.layer" + std::to_string(li + 1) + "." + std::to_string(bi);
      Plan::Block blk;
      blk.in = z;
      blk.c1 = add_conv(pre + ".conv1", pre + ".gn1", cin, c, 3, s, 1, H, H, z, zb, true);
      const int Ho = P.convs[blk.c1].Ho;
      blk.c2 = add_conv(pre + ".conv2", pre + ".gn2", c, c, 3, 1, 1, Ho, Ho, P.convs[blk.c1].z, P.convs[blk.c1].zb,
                        true);
      blk.down = (s != 1 || cin != c)
                     ? add_conv(pre + ".down.conv", pre + ".down.gn", cin, c, 1, s, 0, H, H, z, zb, false)
                     : -1;
      blk.out = P.convs[blk.c2].z;  // conv2's GN output buffer holds relu(gn2 + shortcut)
      P.blocks.push_back(blk);
      z = blk.out;
      zb = P.convs[blk.c2].zb;
      H = Ho;
      cin = c;
    }
  }
  add_conv("enc.compress.conv", "enc.compress.gn", 256, 128, 3, 1, 1, H, H, z, zb, false);
  P.flat = take((size_t)F * 512);
  P.vis = take((size_t)F * 512);
  P.xin = take((size_t)F * kXin);
  P.GI = take((size_t)F * kG4);
  P.Hs = take((size_t)F * kH);
  P.Hin = take((size_t)F * kH);
  P.Cin = take((size_t)F * kH);
  P.Cs = take((size_t)F * kH);
  P.IFGO = take((size_t)F * kH * 4);
  P.dH = take((size_t)F * kH);
  P.dG = take((size_t)F * kG4);
  P.wr_b = take_b(2 * max_w);
  P.wd_b = take_b(max_w);
  P.dyb = take_b(max_act);
  P.dwt = take(max_w);
  P.part = take((size_t)kMaxSplits * max_w);
  P.gn_part = take((size_t)F * 256 * 2);
  P.dz_a = take(max_act);
  P.dz_b = take(max_act);
  P.dz_c = take(max_act);
  P.dxin = take((size_t)F * kXin);
  P.dflat = take((size_t)F * 512);
  P.dvis = take((size_t)F * 512);
  P.bytes = off;
}

inline int blocks_for(ddppo_ctx* ctx, size_t n) {
  return (int)std::min<size_t>((n + kThreads - 1) / kThreads, (size_t)ctx->sm_count * 16);
}

// The forward decides every ReLU / max-pool mask the backward inherits, so its implicit GEMMs take
// bf16 hi / lo operand planes (~16-bit-mantissa products, fp32 accumulation); the FC / LSTM input
// GEMMs likewise run bf16x3 on gemm_tc.  Gradient GEMMs use plain bf16.
constexpr int kPrecFwd = 3;

struct ConvGeom {
  int F, H, W, Ci, Co, k, s, p, Ho, Wo;
  int K() const { return k * k * Ci; }
  int M() const { return F * Ho * Wo; }
};
struct ConvScratch {
  __nv_bfloat16 *wr_b, *wd_b;  // weights as bf16 (hi/lo planes) / bf16
  float *dwt, *part;           // weight-gradient GEMM output [(u,v,c)][o], split-K partials
};

bool is_stem(const ConvGeom& g) { return g.Ci == 1; }

// Implicit-GEMM operands over NHWC bf16 tensors
IgOperand op_pix(const __nv_bfloat16* x, int PH, int PW, int SH, int SW, int SC, const ConvGeom& g, int transposed,
                 int64_t plane) {
  IgOperand o = {};
  o.kind = IG_PIX_K;
  o.x = x;
  o.plane = plane;
  o.g = IGather{x, PH, PW, SH, SW, SC, g.k, g.s, g.p, transposed, 0, 0, 0};
  return o;
}
IgOperand op_dense(int kind, const __nv_bfloat16* x, int64_t ld, int64_t plane) {
  IgOperand o = {};
  o.kind = kind;
  o.x = x;
  o.ld = ld;
  o.plane = plane;
  return o;
}

// y[F][Ho][Wo][Co] = conv(x, W[Co][Ci][k][k]); xb = x as bf16 hi/lo planes (unused by the stem)
ddppo_status conv_fwd(ddppo_ctx* ctx, const ConvGeom& g, const float* x, const __nv_bfloat16* xb, const float* w,
                      const __nv_bfloat16* wr_b, float* y, const ConvScratch& sc, cudaStream_t st) {
  if (is_stem(g)) {
    DDPPO_REQUIRE(ctx, g.Co <= kStemCoMax && g.Co % 8 == 0 && g.k * g.k <= 64, "stem conv: Co in {8,..,32}, k*k <= 64");
    const size_t smem = (size_t)(g.H * g.W + g.Co * g.k * g.k) * sizeof(float);
    DDPPO_REQUIRE(ctx, smem <= 48 * 1024, "stem conv: frame too large for shared memory");
    stem_fwd_kernel<<<g.F, kThreads, smem, st>>>(x, w, g.H, g.W, g.Co, g.k, g.s, g.p, g.Ho, g.Wo, y);
    ctx->count(1);
    DDPPO_CUDA_TRY(ctx, cudaGetLastError());
    return DDPPO_OK;
  }
  const int K = g.K(), M = g.M();
  if (!wr_b) {  // weights not prepared by weights_prep_kernel (diagnostic entry)
    weights_bf16_kernel<<<blocks_for(ctx, (size_t)g.Co * K), kThreads, 0, st>>>(w, g.Co, g.Ci, g.k, sc.wr_b, nullptr);
    ctx->count(1);
    DDPPO_CUDA_TRY(ctx, cudaGetLastError());
    wr_b = sc.wr_b;
  }
  IGemm gm;
  gm.a = op_pix(xb, g.Ho, g.Wo, g.H, g.W, g.Ci, g, 0, (int64_t)g.F * g.H * g.W * g.Ci);
  gm.b = op_dense(IG_DENSE_K, wr_b, K, (int64_t)g.Co * K);
  gm.C = y;
  gm.ldc = g.Co;
  gm.M = M;
  gm.N = g.Co;
  gm.K = K;
  gm.planes = 2;
  gm.partial = sc.part;
  gm.auto_split = 1;
  return launch_igemm(ctx, gm, st);
}

// dy (bf16, gradient wrt the conv output) -> dw (PyTorch order); dx (+)= input gradient (if dx)
ddppo_status conv_bwd(ddppo_ctx* ctx, const ConvGeom& g, const float* x, const __nv_bfloat16* xb, const float* w,
                      const __nv_bfloat16* wd_b, const __nv_bfloat16* dy, float* dw, float* dx, int accumulate_dx,
                      const ConvScratch& sc, cudaStream_t st) {
  if (is_stem(g)) {
    DDPPO_REQUIRE(ctx, dx == nullptr, "stem conv: no input gradient");
    const size_t smem = ((size_t)g.H * g.W + (size_t)kStemPix * (kStemTapPad + g.Co)) * sizeof(float);
    DDPPO_REQUIRE(ctx, smem <= 200 * 1024, "stem conv: frame too large for shared memory");
    static bool attr_set = false;
    if (!attr_set) {
      DDPPO_CUDA_TRY(ctx, cudaFuncSetAttribute(stem_wgrad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               200 * 1024));
      DDPPO_CUDA_TRY(ctx, cudaFuncSetAttribute(stem_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               200 * 1024));
      attr_set = true;
    }
    stem_wgrad_kernel<<<g.F, kThreads, smem, st>>>(x, dy, g.H, g.W, g.Co, g.k, g.s, g.p, g.Ho, g.Wo, sc.part);
    frame_sum_kernel<<<g.Co * g.k * g.k, kThreads, 0, st>>>(sc.part, g.F, g.Co * g.k * g.k, dw);
    ctx->count(2);
    DDPPO_CUDA_TRY(ctx, cudaGetLastError());
    return DDPPO_OK;
  }
  const int K = g.K(), M = g.M();
  // wgrad: dWt[(u,v,c)][o] = sum_q x[tap(q; u, v)][c] dy[q][o]  (k runs over the M output pixels)
  {
    const int splits = std::max(1, std::min(kMaxSplits, M / 2048));
    IGemm gm;
    gm.a = op_pix(xb, g.Ho, g.Wo, g.H, g.W, g.Ci, g, 0, 0);
    gm.a.kind = IG_TAP_MN;
    gm.b = op_dense(IG_DENSE_MN, dy, g.Co, 0);
    gm.C = sc.dwt;
    gm.ldc = g.Co;
    gm.M = K;
    gm.N = g.Co;
    gm.K = M;
    gm.splits = splits;
    gm.partial = sc.part;
    ddppo_status s = launch_igemm(ctx, gm, st);
    if (s != DDPPO_OK) return s;
    wgrad_to_torch_kernel<<<blocks_for(ctx, (size_t)g.Co * K), kThreads, 0, st>>>(sc.dwt, g.Co, g.Ci, g.k, dw);
    ctx->count(1);
  }
  if (dx == nullptr) return DDPPO_OK;
  // dgrad: dx[p][c] (+)= sum_{(u,v,o)} dy[tap^T(p; u, v)][o] W[o][c][u][v]
  if (!wd_b) {
    weights_bf16_kernel<<<blocks_for(ctx, (size_t)g.Co * K), kThreads, 0, st>>>(w, g.Co, g.Ci, g.k, nullptr, sc.wd_b);
    ctx->count(1);
    DDPPO_CUDA_TRY(ctx, cudaGetLastError());
    wd_b = sc.wd_b;
  }
  const int Kd = g.k * g.k * g.Co;
  IGemm gm;
  gm.a = op_pix(dy, g.H, g.W, g.Ho, g.Wo, g.Co, g, 1, 0);
  gm.b = op_dense(IG_DENSE_K, wd_b, Kd, 0);
  gm.C = dx;
  gm.ldc = g.Ci;
  gm.M = g.F * g.H * g.W;
  gm.N = g.Ci;
  gm.K = Kd;
  gm.accumulate = accumulate_dx;
  gm.partial = sc.part;
  gm.auto_split = 1;
  return launch_igemm(ctx, gm, st);
}

// z = (relu)(GN(y) (+ residual)); stats [F][16][2] = (mean, rstd); zb (nullable) = z as bf16 planes
ddppo_status gn_fwd(ddppo_ctx* ctx, int F, int HW, int C, const float* y, const float* gamma, const float* beta,
                    const float* residual, int relu, float* stats, float* z, __nv_bfloat16* zb, cudaStream_t st) {
  DDPPO_REQUIRE(ctx, C >= kGroups && kGnThreads % C == 0, "groupnorm: C must divide 256 (and be >= 16)");
  gn_fwd_kernel<<<F, kGnThreads, 0, st>>>(y, gamma, beta, residual, HW, C, relu, (size_t)F * HW * C, stats, z, zb);
  ctx->count(1);
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  return DDPPO_OK;
}

// dz: gradient wrt z; relu_z: z if a ReLU produced it (mask z > 0), else null.  Writes dy (gradient
// wrt y, bf16), dgamma, dbeta.  part [F][C][2] is scratch.
ddppo_status gn_bwd(ddppo_ctx* ctx, int F, int HW, int C, const float* dz, const float* relu_z, const float* y,
                    const float* stats, const float* gamma, __nv_bfloat16* dy, float* dgamma, float* dbeta,
                    float* part, cudaStream_t st) {
  DDPPO_REQUIRE(ctx, C >= kGroups && kGnThreads % C == 0, "groupnorm: C must divide 256 (and be >= 16)");
  gn_bwd_kernel<<<F, kGnThreads, 0, st>>>(dz, relu_z, y, stats, gamma, HW, C, dy, part);
  ctx->count(1);
  gn_param_reduce_kernel<<<C, kThreads, 0, st>>>(part, F, C, dgamma, dbeta);
  ctx->count(1);
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  return DDPPO_OK;
}

ConvGeom geom_of(const Plan& P, const ConvGN& c) { return ConvGeom{P.F, c.H, c.W, c.Ci, c.Co, c.k, c.s, c.p, c.Ho, c.Wo}; }
ConvScratch scratch_of(const Plan& P) { return ConvScratch{P.wr_b, P.wd_b, P.dwt, P.part}; }

// conv (+GN (+residual) (+ReLU)) forward
ddppo_status conv_gn_fwd(ddppo_ctx* ctx, const float* prm, Plan& P, ConvGN& c, const float* residual, int relu,
                         cudaStream_t st) {
  ddppo_status s = conv_fwd(ctx, geom_of(P, c), c.x, c.xb, prm + c.w, c.wr_b, c.y, scratch_of(P), st);
  if (s != DDPPO_OK) return s;
  return gn_fwd(ctx, P.F, c.Ho * c.Wo, c.Co, c.y, prm + c.gw, prm + c.gb, residual, relu, c.stats, c.z, c.zb, st);
}

// backward of conv+GN: dz = gradient wrt the GN(+residual)(+ReLU) output; relu_z = that output if a
// ReLU followed (its > 0 mask), else null.  Writes dW, dgamma, dbeta into grad; dx (+)= into dx.
ddppo_status conv_gn_bwd(ddppo_ctx* ctx, const float* prm, float* grad, Plan& P, ConvGN& c, const float* dz,
                         const float* relu_z, float* dx, int accumulate_dx, cudaStream_t st) {
  ddppo_status s = gn_bwd(ctx, P.F, c.Ho * c.Wo, c.Co, dz, relu_z, c.y, c.stats, prm + c.gw, P.dyb, grad + c.gw,
                          grad + c.gb, P.gn_part, st);
  if (s != DDPPO_OK) return s;
  return conv_bwd(ctx, geom_of(P, c), c.x, c.xb, prm + c.w, c.wd_b, P.dyb, grad + c.w, dx, accumulate_dx,
                  scratch_of(P), st);
}

// gemm_tc with split-K chosen so that small-M / long-K GEMMs still fill the GPU (partials in P.part)
ddppo_status gemm_split(ddppo_ctx* ctx, GemmTC g, const Plan& P, cudaStream_t st) {
  const int bn = g.N <= 32 ? 32 : (g.N <= 64 || g.prec == 3) ? 64 : 128;
  const long long tiles = (long long)((g.N + bn - 1) / bn) * ((g.M + 127) / 128);
  const int chunks = (g.K + 63) / 64;
  const int splits = (int)std::max(1LL, std::min<long long>({(2LL * ctx->sm_count + tiles - 1) / tiles, chunks / 2, 16}));
  if (splits > 1) {
    g.splits = splits;
    g.partial = P.part;
  }
  return launch_gemm_tc(ctx, g, st);
}

LstmPtrs lstm_ptrs(const ModelLayout& L, const float* prm, const ddppo_batch& b, Plan& P) {
  LstmPtrs q;
  q.Whh = prm + off_of(L, "rnn.weight_hh");
  q.bih = prm + off_of(L, "rnn.bias_ih");
  q.bhh = prm + off_of(L, "rnn.bias_hh");
  q.GI = P.GI;
  q.mask = b.mask;
  q.h0 = b.h0;
  q.c0 = b.c0;
  q.env_idx = b.env_idx;
  q.B = b.B;
  q.T_run = b.T_run;
  q.ld = b.ld;
  q.Hs = P.Hs;
  q.Hin = P.Hin;
  q.Cin = P.Cin;
  q.Cs = P.Cs;
  q.IFGO = reinterpret_cast<float4*>(P.IFGO);
  q.dH = P.dH;
  q.dG = P.dG;
  return q;
}

}  // namespace

size_t depth_workspace(int max_B, int T) {
  ddppo_model_desc d = {};
  d.arch = DDPPO_ARCH_DEPTH_R18_LSTM;
  d.hidden = 512;
  d.num_actions = 4;
  ModelLayout L;
  build_layout(&d, &L);
  Plan P;
  make_plan(L, max_B, T, nullptr, &P);
  return P.bytes;
}

namespace {
// encoder -> visual FC -> LSTM input -> GI GEMM -> LSTM recurrence
ddppo_status depth_fwd_net(ddppo_ctx* ctx, const ModelLayout& L, const float* prm, const ddppo_batch& b, Plan& P,
                           cudaStream_t st) {
  const int F = P.F;
  {
    WeightPrep prep;
    prep.n = 0;
    int max_n = 0;
    for (const ConvGN& c : P.convs) {
      if (c.Ci == 1) continue;
      prep.it[prep.n++] = WeightPrep::Item{prm + c.w, c.wr_b, c.wd_b, c.Co, c.Ci, c.k};
      max_n = std::max(max_n, c.Co * c.Ci * c.k * c.k);
    }
    weights_prep_kernel<<<dim3((max_n + 1023) / 1024, prep.n), 1024, 0, st>>>(prep);
    ctx->count(1);
  }
  gather_obs_kernel<<<blocks_for(ctx, (size_t)F * kImg * kImg), kThreads, 0, st>>>(b.obs, b.env_idx, b.T, b.T_run, F,
                                                                                    P.x0);
  ctx->count(1);
  ddppo_status s = conv_gn_fwd(ctx, prm, P, P.convs[0], nullptr, 1, st);
  if (s != DDPPO_OK) return s;
  {
    ConvGN& c = P.convs[0];
    const int hp = (c.Ho + 2 - 3) / 2 + 1;
    maxpool_fwd_kernel<<<blocks_for(ctx, (size_t)F * hp * hp * 32), kThreads, 0, st>>>(c.z, F, c.Ho, c.Wo, 32, hp, hp,
                                                                                       P.pool_out, P.pool_arg, P.pool_b);
    ctx->count(1);
  }
  for (auto& blk : P.blocks) {
    if ((s = conv_gn_fwd(ctx, prm, P, P.convs[blk.c1], nullptr, 1, st)) != DDPPO_OK) return s;
    const float* sc = blk.in;
    if (blk.down >= 0) {
      if ((s = conv_gn_fwd(ctx, prm, P, P.convs[blk.down], nullptr, 0, st)) != DDPPO_OK) return s;
      sc = P.convs[blk.down].z;
    }
    if ((s = conv_gn_fwd(ctx, prm, P, P.convs[blk.c2], sc, 1, st)) != DDPPO_OK) return s;
  }
  ConvGN& comp = P.convs.back();
  if ((s = conv_gn_fwd(ctx, prm, P, comp, nullptr, 1, st)) != DDPPO_OK) return s;
  flatten_kernel<<<blocks_for(ctx, (size_t)F * 512), kThreads, 0, st>>>(comp.z, F, P.flat, 1);
  ctx->count(1);
  // visual FC + ReLU
  if ((s = gemm_split(ctx, GemmTC{P.flat, 512, 1, prm + off_of(L, "visual_fc.weight"), 512, 1, P.vis, 512, F, 512,
                                      512, 1, nullptr, kPrecFwd}, P,
                          st)) != DDPPO_OK)
    return s;
  bias_act_kernel<<<blocks_for(ctx, (size_t)F * 512), kThreads, 0, st>>>(P.vis, prm + off_of(L, "visual_fc.bias"), F,
                                                                         512, 1);
  ctx->count(1);
  lstm_input_kernel<<<blocks_for(ctx, (size_t)F * kXin), kThreads, 0, st>>>(
      P.vis, b.goal, b.prev_action, b.env_idx, prm + off_of(L, "goal_fc.weight"), prm + off_of(L, "goal_fc.bias"),
      prm + off_of(L, "act_embed.weight"), b.T, b.ld, b.T_run, F, P.xin);
  ctx->count(1);
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  // GI = x W_ih^T (biases are added inside the recurrence)
  if ((s = gemm_split(ctx, GemmTC{P.xin, kXin, 1, prm + off_of(L, "rnn.weight_ih"), kXin, 1, P.GI, kG4, F, kG4,
                                      kXin, 1, nullptr, kPrecFwd}, P,
                          st)) != DDPPO_OK)
    return s;
  return launch_lstm_fwd(ctx, lstm_ptrs(L, prm, b, P), st);
}
}  // namespace

ddppo_status depth_fwd(ddppo_ctx* ctx, const ModelLayout& L, const float* prm, const ddppo_batch& b, float* logits,
                       float* values, void* ws, cudaStream_t st) {
  DDPPO_REQUIRE(ctx, b.obs && b.c0, "depth: batch needs obs and c0");
  DDPPO_REQUIRE(ctx, b.B >= 1 && b.B <= 8 && b.T_run <= 1024, "depth: minibatch must hold 1..8 envs, T <= 1024");
  Plan P;
  make_plan(L, b.B, b.T_run, ws, &P);
  {
    ProfScope ps(ctx, DDPPO_K_NET_FWD, st, 0);
    ddppo_status s = depth_fwd_net(ctx, L, prm, b, P, st);
    if (s != DDPPO_OK) return s;
  }
  ProfScope ps(ctx, DDPPO_K_HEAD, st, 0);
  return launch_head_fwd(ctx, prm + off_of(L, "head.weight"), prm + off_of(L, "head.bias"), P.Hs, P.F, logits, values,
                         st);
}

ddppo_status depth_bwd(ddppo_ctx* ctx, const ModelLayout& L, const float* prm, const ddppo_batch& b,
                       const float* dlogits, const float* dvalues, float* grad, void* ws, cudaStream_t st) {
  Plan P;
  make_plan(L, b.B, b.T_run, ws, &P);
  const int F = P.F;
  ddppo_status s;
  {
    ProfScope ps(ctx, DDPPO_K_HEAD, st, 0);
    s = launch_head_bwd(ctx, prm + off_of(L, "head.weight"), P.Hs, dlogits, dvalues, F, P.dH,
                        grad + off_of(L, "head.weight"), grad + off_of(L, "head.bias"), st);
    if (s != DDPPO_OK) return s;
  }
  ProfScope ps(ctx, DDPPO_K_NET_BWD, st, 0);
  if ((s = launch_lstm_bwd(ctx, lstm_ptrs(L, prm, b, P), st)) != DDPPO_OK) return s;
  // LSTM weight gradients and db (b_ih and b_hh receive the same gradient)
  if ((s = gemm_split(ctx, GemmTC{P.dG, 1, kG4, P.xin, 1, kXin, grad + off_of(L, "rnn.weight_ih"), kXin, kG4, kXin,
                                      F}, P,
                          st)) != DDPPO_OK)
    return s;
  if ((s = gemm_split(ctx, GemmTC{P.dG, 1, kG4, P.Hin, 1, kH, grad + off_of(L, "rnn.weight_hh"), kH, kG4, kH, F}, P,
                          st)) != DDPPO_OK)
    return s;
  if ((s = launch_colsum(ctx, P.dG, kG4, F, kG4, grad + off_of(L, "rnn.bias_ih"), st)) != DDPPO_OK) return s;
  if ((s = launch_colsum(ctx, P.dG, kG4, F, kG4, grad + off_of(L, "rnn.bias_hh"), st)) != DDPPO_OK) return s;
  // dx = dG W_ih  [F][576]
  if ((s = gemm_split(ctx, GemmTC{P.dG, kG4, 1, prm + off_of(L, "rnn.weight_ih"), 1, kXin, P.dxin, kXin, F, kXin,
                                      kG4}, P,
                          st)) != DDPPO_OK)
    return s;
  goal_emb_grads_kernel<<<64, kThreads, 0, st>>>(P.dxin, b.goal, b.prev_action, b.env_idx, b.T, b.ld, b.T_run, F,
                                                 grad + off_of(L, "goal_fc.weight"), grad + off_of(L, "goal_fc.bias"),
                                                 grad + off_of(L, "act_embed.weight"));
  ctx->count(1);
  vis_mask_kernel<<<blocks_for(ctx, (size_t)F * 512), kThreads, 0, st>>>(P.dxin, P.vis, F, P.dvis);
  ctx->count(1);
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  // visual FC: dW = dVpre^T flat, db = colsum(dVpre), dflat = dVpre W
  if ((s = gemm_split(ctx, GemmTC{P.dvis, 1, 512, P.flat, 1, 512, grad + off_of(L, "visual_fc.weight"), 512, 512,
                                      512, F}, P,
                          st)) != DDPPO_OK)
    return s;
  if ((s = launch_colsum(ctx, P.dvis, 512, F, 512, grad + off_of(L, "visual_fc.bias"), st)) != DDPPO_OK) return s;
  if ((s = gemm_split(ctx, GemmTC{P.dvis, 512, 1, prm + off_of(L, "visual_fc.weight"), 1, 512, P.dflat, 512, F,
                                      512, 512}, P,
                          st)) != DDPPO_OK)
    return s;
  // encoder: dz = gradient wrt the current block output; three rotating activation buffers
  ConvGN& comp = P.convs.back();
  float* dz = P.dz_a;
  float* da = P.dz_b;
  float* dn = P.dz_c;
  flatten_kernel<<<blocks_for(ctx, (size_t)F * 512), kThreads, 0, st>>>(P.dflat, F, da, 0);
  ctx->count(1);
  if ((s = conv_gn_bwd(ctx, prm, grad, P, comp, da, comp.z, dz, 0, st)) != DDPPO_OK) return s;
  for (int bi = (int)P.blocks.size() - 1; bi >= 0; --bi) {
    const Plan::Block& blk = P.blocks[bi];
    ConvGN& c1 = P.convs[blk.c1];
    ConvGN& c2 = P.convs[blk.c2];
    // out = relu(gn2(conv2(a)) + shortcut(in)), a = relu(gn1(conv1(in)))
    if ((s = conv_gn_bwd(ctx, prm, grad, P, c2, dz, c2.z, da, 0, st)) != DDPPO_OK) return s;
    if (blk.down >= 0) {
      if ((s = conv_gn_bwd(ctx, prm, grad, P, P.convs[blk.down], dz, c2.z, dn, 0, st)) != DDPPO_OK) return s;
    } else {
      const size_t n = (size_t)F * c2.Ho * c2.Wo * c2.Co;
      relu_mask_kernel<<<blocks_for(ctx, n), kThreads, 0, st>>>(dz, c2.z, n, dn);
      ctx->count(1);
    }
    if ((s = conv_gn_bwd(ctx, prm, grad, P, c1, da, c1.z, dn, 1, st)) != DDPPO_OK) return s;
    std::swap(dz, dn);  // dn (the block input's gradient) becomes the next dz
  }
  // max-pool, then the stem (no input gradient)
  ConvGN& stem = P.convs[0];
  {
    const int hp = (stem.Ho + 2 - 3) / 2 + 1;
    maxpool_bwd_kernel<<<blocks_for(ctx, (size_t)F * stem.Ho * stem.Wo * 32), kThreads, 0, st>>>(
        dz, P.pool_arg, F, stem.Ho, stem.Wo, 32, hp, hp, da);
    ctx->count(1);
  }
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  return conv_gn_bwd(ctx, prm, grad, P, stem, da, stem.z, nullptr, 0, st);
}

// ------------------------------------------------------------------ diagnostic entries (tests)
extern "C" ddppo_status ddppo_debug_conv2d(ddppo_ctx* ctx, const float* x, const float* w, int F, int H, int W,
                                           int Ci, int Co, int k, int s, int p, float* y, const float* dy, float* dx,
                                           float* dw, void* scratch, size_t scratch_bytes, size_t* host_need,
                                           void* stream) {
  if (!ctx) return DDPPO_ERR_CONFIG;
  DDPPO_REQUIRE(ctx, F >= 1 && H >= 1 && W >= 1 && Ci >= 1 && Co >= 1 && k >= 1 && s >= 1 && p >= 0 && H + 2 * p >= k &&
                         W + 2 * p >= k,
                "conv2d: bad geometry");
  DDPPO_REQUIRE(ctx, Ci == 1 || (Ci % 8 == 0 && Co % 8 == 0), "conv2d: Ci == 1 (stem) or Ci, Co multiples of 8");
  const int Ho = (H + 2 * p - k) / s + 1, Wo = (W + 2 * p - k) / s + 1;
  ConvGeom g{F, H, W, Ci, Co, k, s, p, Ho, Wo};
  const size_t nx = (size_t)F * H * W * Ci, ny = (size_t)g.M() * Co, ok = (size_t)Co * g.K();
  const size_t nb = 2 * nx + ny + 2 * ok + ok;  // bf16 elements: x planes, dy, wr planes, wd
  const size_t nf = ok + std::max((size_t)kMaxSplits * ok, (size_t)F * ok);
  const size_t need = nb * 2 + nf * 4 + 8 * 256;
  if (host_need) *host_need = need;
  if (!scratch) return DDPPO_OK;
  DDPPO_REQUIRE(ctx, scratch_bytes >= need, "conv2d: scratch too small");
  char* b = reinterpret_cast<char*>(scratch);
  auto take = [&](size_t bytes) {
    char* r = b;
    b += align_up(bytes, 256);
    return r;
  };
  __nv_bfloat16* xb = reinterpret_cast<__nv_bfloat16*>(take(2 * nx * 2));
  __nv_bfloat16* dyb = reinterpret_cast<__nv_bfloat16*>(take(ny * 2));
  ConvScratch sc;
  sc.wr_b = reinterpret_cast<__nv_bfloat16*>(take(2 * ok * 2));
  sc.wd_b = reinterpret_cast<__nv_bfloat16*>(take(ok * 2));
  sc.dwt = reinterpret_cast<float*>(take(ok * 4));
  sc.part = reinterpret_cast<float*>(take((nf - ok) * 4));
  cudaStream_t st = as_stream(stream);
  ProfScope ps(ctx, DDPPO_K_OTHER, st, 0);
  to_planes_kernel<<<blocks_for(ctx, nx), kThreads, 0, st>>>(x, nx, xb);
  ctx->count(1);
  if (y) {
    ddppo_status r = conv_fwd(ctx, g, x, xb, w, nullptr, y, sc, st);
    if (r != DDPPO_OK) return r;
  }
  if (dy) {
    to_bf16_kernel<<<blocks_for(ctx, ny), kThreads, 0, st>>>(dy, ny, dyb);
    ctx->count(1);
    return conv_bwd(ctx, g, x, xb, w, nullptr, dyb, dw, Ci == 1 ? nullptr : dx, 0, sc, st);
  }
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  return DDPPO_OK;
}

namespace {
__global__ void bf16_to_f32_kernel(const __nv_bfloat16* __restrict__ x, size_t n, float* __restrict__ y) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    y[i] = __bfloat162float(x[i]);
}
}  // namespace

extern "C" ddppo_status ddppo_debug_groupnorm(ddppo_ctx* ctx, const float* y, const float* gamma, const float* beta,
                                              const float* residual, int F, int HW, int C, int relu, float* z,
                                              float* stats, const float* dz, float* dy, float* dgamma, float* dbeta,
                                              float* scratch, void* stream) {
  if (!ctx) return DDPPO_ERR_CONFIG;
  DDPPO_REQUIRE(ctx, F >= 1 && HW >= 1 && C >= kGroups && C % kGroups == 0, "groupnorm: C must be a multiple of 16");
  cudaStream_t st = as_stream(stream);
  ProfScope ps(ctx, DDPPO_K_OTHER, st, 0);
  ddppo_status r = gn_fwd(ctx, F, HW, C, y, gamma, beta, residual, relu, stats, z, nullptr, st);
  if (r != DDPPO_OK || !dz) return r;
  __nv_bfloat16* dyb = reinterpret_cast<__nv_bfloat16*>(scratch + 2 * (size_t)F * C);
  r = gn_bwd(ctx, F, HW, C, dz, relu ? z : nullptr, y, stats, gamma, dyb, dgamma, dbeta, scratch, st);
  if (r != DDPPO_OK) return r;
  bf16_to_f32_kernel<<<blocks_for(ctx, (size_t)F * HW * C), kThreads, 0, st>>>(dyb, (size_t)F * HW * C, dy);
  ctx->count(1);
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  return DDPPO_OK;
}

extern "C" ddppo_status ddppo_debug_maxpool(ddppo_ctx* ctx, const float* x, int F, int H, int W, int C, float* y,
                                            uint8_t* arg, const float* dy, float* dx, void* stream) {
  if (!ctx) return DDPPO_ERR_CONFIG;
  DDPPO_REQUIRE(ctx, F >= 1 && H >= 2 && W >= 2 && C >= 1, "maxpool: bad geometry");
  const int Ho = (H + 2 - 3) / 2 + 1, Wo = (W + 2 - 3) / 2 + 1;
  cudaStream_t st = as_stream(stream);
  ProfScope ps(ctx, DDPPO_K_OTHER, st, 0);
  maxpool_fwd_kernel<<<blocks_for(ctx, (size_t)F * Ho * Wo * C), kThreads, 0, st>>>(x, F, H, W, C, Ho, Wo, y, arg,
                                                                                     nullptr);
  ctx->count(1);
  if (dy) {
    maxpool_bwd_kernel<<<blocks_for(ctx, (size_t)F * H * W * C), kThreads, 0, st>>>(dy, arg, F, H, W, C, Ho, Wo, dx);
    ctx->count(1);
  }
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  return DDPPO_OK;
}

namespace {
__global__ void positive_mask_kernel(const float* __restrict__ z, size_t n, uint8_t* __restrict__ out) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    out[i] = z[i] > 0.f ? 1 : 0;
}
}  // namespace

// The forward's discrete decisions (every ReLU mask and the max-pool argmax), from the workspace of
// the last ddppo_policy_fwd on `batch`, in the order documented in include/ddppo.h.
extern "C" ddppo_status ddppo_debug_depth_decisions(ddppo_ctx* ctx, const ddppo_batch* host_batch, void* ws,
                                                    uint8_t* out, int64_t cap, int64_t* host_n, void* stream) {
  if (!ctx || !host_batch) return DDPPO_ERR_CONFIG;
  ddppo_model_desc d = {};
  d.arch = DDPPO_ARCH_DEPTH_R18_LSTM;
  d.hidden = 512;
  d.num_actions = 4;
  ModelLayout L;
  build_layout(&d, &L);
  Plan P;
  make_plan(L, host_batch->B, host_batch->T_run, ws, &P);
  const int F = P.F;
  std::vector<std::pair<const float*, size_t>> masks;
  const ConvGN& stem = P.convs[0];
  masks.push_back({stem.z, (size_t)F * stem.Ho * stem.Wo * stem.Co});
  const size_t pool_n = (size_t)F * 16 * 16 * 32;
  int64_t total = (int64_t)masks[0].second + (int64_t)pool_n;
  for (const auto& blk : P.blocks) {
    const ConvGN& c1 = P.convs[blk.c1];
    const ConvGN& c2 = P.convs[blk.c2];
    masks.push_back({c1.z, (size_t)F * c1.Ho * c1.Wo * c1.Co});
    masks.push_back({c2.z, (size_t)F * c2.Ho * c2.Wo * c2.Co});
    total += (int64_t)(masks[masks.size() - 2].second + masks.back().second);
  }
  const ConvGN& comp = P.convs.back();
  masks.push_back({comp.z, (size_t)F * comp.Ho * comp.Wo * comp.Co});
  masks.push_back({P.vis, (size_t)F * 512});
  total += (int64_t)(masks[masks.size() - 2].second + masks.back().second);
  if (host_n) *host_n = total;
  if (!out) return DDPPO_OK;
  DDPPO_REQUIRE(ctx, cap >= total, "depth decisions: buffer too small");
  cudaStream_t st = as_stream(stream);
  size_t off = 0;
  for (size_t i = 0; i < masks.size(); ++i) {
    positive_mask_kernel<<<blocks_for(ctx, masks[i].second), kThreads, 0, st>>>(masks[i].first, masks[i].second,
                                                                               out + off);
    off += masks[i].second;
    if (i == 0) {
      DDPPO_CUDA_TRY(ctx, cudaMemcpyAsync(out + off, P.pool_arg, pool_n, cudaMemcpyDeviceToDevice, st));
      off += pool_n;
    }
  }
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  return DDPPO_OK;
}
