// Depth agent (BASELINE configs[2]): 64x64 depth -> half-width ResNet18 with GroupNorm -> 128x2x2
// -> FC 512 + ReLU; x = [visual, goal FC 32, action embedding 32] -> LSTM-512 -> Linear(512, 5).
// (P:L212 half-width backbone with GroupNorm, App. C; readings Z17-Z23 in DESIGN.md.)
//
// Layout: activations fp32 NHWC [frames][H][W][C] in the workspace, frames f = b*T_run + t.
// Convolutions are GEMMs on the tcgen05 kernel of gemm_tc.cu (bf16 operands, fp32 TMEM
// accumulation):  fprop  Y[f,i,j][o] = sum_k col[f,i,j][k] Wr[o][k]     (im2col, k = (u, v, c))
//                 dgrad  dcol = dY Wr  -> col2im (gather, fixed order)
//                 wgrad  dWr[o][k] = sum_m dY[m][o] col[m][k]            (split-K over output pixels)
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

// col[m = (f, i, j)][k = (u*kw + v)*C + c] = x[f][i*s-p+u][j*s-p+v][c] (0 outside)
__global__ void im2col_kernel(const float* __restrict__ x, int F, int H, int W, int C, int k, int s, int p, int Ho,
                              int Wo, float* __restrict__ col) {
  const int K = k * k * C;
  const size_t n = (size_t)F * Ho * Wo * K;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int kk = (int)(i % K);
    const size_t m = i / K;
    const int j = (int)(m % Wo), ii = (int)((m / Wo) % Ho), f = (int)(m / ((size_t)Wo * Ho));
    const int c = kk % C, uv = kk / C, u = uv / k, v = uv % k;
    const int y = ii * s - p + u, xx = j * s - p + v;
    col[i] = (y >= 0 && y < H && xx >= 0 && xx < W) ? x[(((size_t)f * H + y) * W + xx) * C + c] : 0.f;
  }
}

// dx[f][y][x][c] (+)= sum over (u, v) with (y + p - u) % s == 0 ... of dcol[(f, i, j)][(u, v, c)]
__global__ void col2im_kernel(const float* __restrict__ dcol, int F, int H, int W, int C, int k, int s, int p, int Ho,
                              int Wo, float* __restrict__ dx, int accumulate) {
  const int K = k * k * C;
  const size_t n = (size_t)F * H * W * C;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    const size_t pix = i / C;
    const int xx = (int)(pix % W), y = (int)((pix / W) % H), f = (int)(pix / ((size_t)W * H));
    float acc = 0.f;
    for (int u = 0; u < k; ++u) {
      const int yy = y + p - u;
      if (yy < 0 || yy % s) continue;
      const int ii = yy / s;
      if (ii >= Ho) continue;
      for (int v = 0; v < k; ++v) {
        const int xv = xx + p - v;
        if (xv < 0 || xv % s) continue;
        const int j = xv / s;
        if (j >= Wo) continue;
        acc += dcol[(((size_t)f * Ho + ii) * Wo + j) * K + (u * k + v) * C + c];
      }
    }
    dx[i] = accumulate ? dx[i] + acc : acc;
  }
}

// W [Co][Ci][k][k] <-> Wr [Co][k][k][Ci]
__global__ void reorder_w_kernel(const float* __restrict__ W, int Co, int Ci, int k, float* __restrict__ Wr,
                                 int to_r) {
  const int n = Co * Ci * k * k;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int o = i / (Ci * k * k), rem = i % (Ci * k * k);
    const int c = rem / (k * k), uv = rem % (k * k);
    const int ir = o * (k * k * Ci) + uv * Ci + c;
    if (to_r) Wr[ir] = W[i];
    else Wr[i] = W[ir];  // (here W is the reordered gradient, Wr the PyTorch-order output)
  }
}

// per (frame, group): mean and rstd over (H*W) x (C/G) channels, fixed-order block reduction
__global__ void __launch_bounds__(kThreads) gn_stats_kernel(const float* __restrict__ x, int HW, int C,
                                                            float* __restrict__ stats) {
  __shared__ double red[2 * (kThreads / 32)];
  const int f = blockIdx.x / kGroups, g = blockIdx.x % kGroups, cg = C / kGroups;
  const int n = HW * cg;
  const float* base = x + (size_t)f * HW * C + g * cg;
  double acc[2] = {0.0, 0.0};
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const float v = base[(size_t)(i / cg) * C + (i % cg)];
    acc[0] += v;
    acc[1] += (double)v * v;
  }
  block_sum<2>(acc, red);
  if (threadIdx.x == 0) {
    const double mu = acc[0] / n;
    double var = acc[1] / n - mu * mu;
    if (var < 0) var = 0;
    stats[2 * blockIdx.x] = (float)mu;
    stats[2 * blockIdx.x + 1] = (float)(1.0 / sqrt(var + 1e-5));
  }
}

// z = (relu)( gamma * xhat + beta (+ residual) )
__global__ void gn_apply_kernel(const float* __restrict__ x, const float* __restrict__ stats,
                                const float* __restrict__ gamma, const float* __restrict__ beta,
                                const float* __restrict__ residual, int F, int HW, int C, int relu,
                                float* __restrict__ z) {
  const int cg = C / kGroups;
  const size_t n = (size_t)F * HW * C;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    const int f = (int)(i / ((size_t)HW * C));
    const int sidx = 2 * (f * kGroups + c / cg);
    float v = (x[i] - stats[sidx]) * stats[sidx + 1] * gamma[c] + beta[c];
    if (residual) v += residual[i];
    z[i] = relu ? fmaxf(v, 0.f) : v;
  }
}

// dy_eff = dz * [z > 0] (optional): per (frame, group) GN backward:
//   dx = rstd * (dxhat - mean(dxhat) - xhat * mean(dxhat * xhat)),   dxhat = dy * gamma
__global__ void __launch_bounds__(kThreads) gn_bwd_kernel(const float* __restrict__ dz, const float* __restrict__ z,
                                                          const float* __restrict__ x, const float* __restrict__ stats,
                                                          const float* __restrict__ gamma, int HW, int C,
                                                          float* __restrict__ dx, float* __restrict__ dy_out) {
  __shared__ double red[2 * (kThreads / 32)];
  __shared__ float sh[2];
  const int f = blockIdx.x / kGroups, g = blockIdx.x % kGroups, cg = C / kGroups;
  const int n = HW * cg;
  const size_t base = (size_t)f * HW * C + g * cg;
  const float mu = stats[2 * blockIdx.x], rstd = stats[2 * blockIdx.x + 1];
  double acc[2] = {0.0, 0.0};
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const size_t o = base + (size_t)(i / cg) * C + (i % cg);
    float dy = dz[o];
    if (z && z[o] <= 0.f) dy = 0.f;
    const int c = g * cg + (i % cg);
    const float dxh = dy * gamma[c];
    const float xh = (x[o] - mu) * rstd;
    acc[0] += dxh;
    acc[1] += (double)dxh * xh;
    if (dy_out) dy_out[o] = dy;
  }
  block_sum<2>(acc, red);
  if (threadIdx.x == 0) {
    sh[0] = (float)(acc[0] / n);
    sh[1] = (float)(acc[1] / n);
  }
  __syncthreads();
  const float m1 = sh[0], m2 = sh[1];
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const size_t o = base + (size_t)(i / cg) * C + (i % cg);
    float dy = dz[o];
    if (z && z[o] <= 0.f) dy = 0.f;
    const int c = g * cg + (i % cg);
    const float dxh = dy * gamma[c];
    const float xh = (x[o] - mu) * rstd;
    dx[o] = rstd * (dxh - m1 - xh * m2);
  }
}

// dgamma[c] = sum_{f,pix} dy * xhat, dbeta[c] = sum dy  (dy already ReLU-masked): thread per
// (channel, chunk) with a fixed chunk partition, partials reduced in chunk order
constexpr int kGnChunks = 32;
__global__ void gn_param_partial_kernel(const float* __restrict__ dy, const float* __restrict__ x,
                                        const float* __restrict__ stats, int F, int HW, int C,
                                        float* __restrict__ part) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int chunk = blockIdx.y;
  if (c >= C) return;
  const int cg = C / kGroups;
  const size_t rows = (size_t)F * HW;
  const size_t per = (rows + kGnChunks - 1) / kGnChunks;
  float sg = 0.f, sb = 0.f;
  for (size_t r = chunk * per; r < min(rows, (chunk + 1) * per); ++r) {
    const size_t o = r * C + c;
    const int f = (int)(r / HW);
    const int sidx = 2 * (f * kGroups + c / cg);
    const float d = dy[o];
    sg += d * (x[o] - stats[sidx]) * stats[sidx + 1];
    sb += d;
  }
  part[((size_t)chunk * C + c) * 2] = sg;
  part[((size_t)chunk * C + c) * 2 + 1] = sb;
}
__global__ void gn_param_reduce_kernel(const float* __restrict__ part, int C, float* __restrict__ dgamma,
                                       float* __restrict__ dbeta) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  float sg = 0.f, sb = 0.f;
  for (int k = 0; k < kGnChunks; ++k) {
    sg += part[((size_t)k * C + c) * 2];
    sb += part[((size_t)k * C + c) * 2 + 1];
  }
  dgamma[c] = sg;
  dbeta[c] = sb;
}

// 3x3 / stride 2 / pad 1 max pool with the first maximum in (u, v) order
__global__ void maxpool_fwd_kernel(const float* __restrict__ x, int F, int H, int W, int C, int Ho, int Wo,
                                   float* __restrict__ y, uint8_t* __restrict__ arg) {
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

__global__ void add_kernel(float* __restrict__ a, const float* __restrict__ b, size_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) a[i] += b[i];
}

// ------------------------------------------------------------------ network plan
struct ConvGN {
  int Ci, Co, k, s, p, H, W, Ho, Wo;  // input H x W, output Ho x Wo
  int64_t w, gw, gb;                  // parameter offsets (conv weight, GN gamma, GN beta)
  float *x, *y, *z, *stats;           // input (not owned), conv out (pre-GN), GN out, GN stats [F][16][2]
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
  uint8_t* pool_arg;
  float *flat, *vis, *xin, *GI;
  float *Hs, *Hin, *Cin, *Cs, *IFGO, *dH, *dG;
  // scratch (reused by every layer)
  float *col, *wr, *dcol, *dwr, *part, *gn_part, *dz_a, *dz_b, *dz_c, *dtmp, *dxin, *dflat, *dvis;
  size_t bytes = 0;
};

int64_t off_of(const ModelLayout& L, const std::string& n) { return layout_offset(L, n.c_str()); }

// Deterministic carve of the workspace (base == nullptr: size only)
void make_plan(const ModelLayout& L, int B, int T_run, void* base, Plan* plan) {
  Plan& P = *plan;
  P = Plan();
  const int F = B * T_run;
  P.F = F;
  size_t off = 0;
  auto take = [&](size_t n_floats) {
    float* p = base ? reinterpret_cast<float*>(reinterpret_cast<char*>(base) + off) : nullptr;
    off = align_up(off + n_floats * sizeof(float), 256);
    return p;
  };
  size_t max_col = 0, max_act = 0, max_w = 0;
  auto add_conv = [&](const std::string& cname, const std::string& gname, int Ci, int Co, int k, int s, int p, int H,
                      int W, float* x) {
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
    const size_t act = (size_t)F * c.Ho * c.Wo * Co;
    c.y = take(act);
    c.z = take(act);
    c.stats = take((size_t)F * kGroups * 2);
    max_col = std::max(max_col, (size_t)F * c.Ho * c.Wo * k * k * Ci);
    max_act = std::max(max_act, std::max(act, (size_t)F * H * W * Ci));
    max_w = std::max(max_w, (size_t)Co * k * k * Ci);
    P.convs.push_back(c);
    return (int)P.convs.size() - 1;
  };
  P.x0 = take((size_t)F * kImg * kImg);
  const int stem = add_conv("enc.stem.conv", "enc.stem.gn", 1, 32, 7, 2, 3, kImg, kImg, P.x0);
  const int hs = P.convs[stem].Ho;  // 32
  const int hp = (hs + 2 - 3) / 2 + 1;  // 16
  P.pool_out = take((size_t)F * hp * hp * 32);
  P.pool_arg = reinterpret_cast<uint8_t*>(take(((size_t)F * hp * hp * 32 + 3) / 4));
  float* z = P.pool_out;
  int H = hp, cin = 32;
  const int widths[4] = {32, 64, 128, 256};
  for (int li = 0; li < 4; ++li) {
    for (int bi = 0; bi < 2; ++bi) {
      const int s = (bi == 0 && li > 0) ? 2 : 1, c = widths[li];
      const std::string pre = "enc.layer" + std::to_string(li + 1) + "." + std::to_string(bi);
      Plan::Block blk;
      blk.in = z;
      blk.c1 = add_conv(pre + ".conv1", pre + ".gn1", cin, c, 3, s, 1, H, H, z);
      const int Ho = P.convs[blk.c1].Ho;
      blk.c2 = add_conv(pre + ".conv2", pre + ".gn2", c, c, 3, 1, 1, Ho, Ho, P.convs[blk.c1].z);
      blk.down = (s != 1 || cin != c) ? add_conv(pre + ".down.conv", pre + ".down.gn", cin, c, 1, s, 0, H, H, z) : -1;
      blk.out = P.convs[blk.c2].z;  // conv2's GN output buffer holds relu(gn2 + shortcut)
      P.blocks.push_back(blk);
      z = blk.out;
      H = Ho;
      cin = c;
    }
  }
  const int comp = add_conv("enc.compress.conv", "enc.compress.gn", 256, 128, 3, 1, 1, H, H, z);
  (void)comp;
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
  P.col = take(max_col);
  P.dcol = take(max_col);
  P.wr = take(std::max(max_w, (size_t)kG4 * kXin));
  P.dwr = take(std::max(max_w, (size_t)kG4 * kXin));
  P.part = take((size_t)64 * std::max(max_w, (size_t)512 * 512));
  P.gn_part = take((size_t)kGnChunks * 256 * 2);
  P.dz_a = take(max_act);
  P.dz_b = take(max_act);
  P.dz_c = take(max_act);
  P.dtmp = take(max_act);
  P.dxin = take((size_t)F * kXin);
  P.dflat = take((size_t)F * 512);
  P.dvis = take((size_t)F * 512);
  P.bytes = off;
}

inline int blocks_for(ddppo_ctx* ctx, size_t n) {
  return (int)std::min<size_t>((n + kThreads - 1) / kThreads, (size_t)ctx->sm_count * 16);
}

// Operand precision of the encoder GEMMs: the forward decides every ReLU / max-pool mask that
// the backward inherits, so it runs on bf16x3 operands (~fp32 products); the gradient GEMMs use
// plain bf16.
constexpr int kPrecFwd = 3, kPrecBwd = 1;

struct ConvGeom {
  int F, H, W, Ci, Co, k, s, p, Ho, Wo;
  int K() const { return k * k * Ci; }
  int M() const { return F * Ho * Wo; }
  bool direct() const { return k == 1 && s == 1 && p == 0; }  // the input is already the im2col matrix
};
struct ConvScratch {
  float *col, *wr, *dcol, *dwr, *part;
};

// y[F][Ho][Wo][Co] = conv(x[F][H][W][Ci], W[Co][Ci][k][k])
ddppo_status conv_fwd(ddppo_ctx* ctx, const ConvGeom& g, const float* x, const float* w, float* y,
                      const ConvScratch& sc, cudaStream_t st) {
  const int K = g.K(), M = g.M();
  reorder_w_kernel<<<blocks_for(ctx, (size_t)g.Co * K), kThreads, 0, st>>>(w, g.Co, g.Ci, g.k, sc.wr, 1);
  ctx->count(1);
  const float* A = x;
  if (!g.direct()) {
    im2col_kernel<<<blocks_for(ctx, (size_t)M * K), kThreads, 0, st>>>(x, g.F, g.H, g.W, g.Ci, g.k, g.s, g.p, g.Ho,
                                                                       g.Wo, sc.col);
    ctx->count(1);
    A = sc.col;
  }
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  return launch_gemm_tc(ctx, GemmTC{A, K, 1, sc.wr, K, 1, y, g.Co, M, g.Co, K, 1, nullptr, kPrecFwd}, st);
}

// dw (PyTorch order) = weight gradient; dx (+)= input gradient (skipped if dx == null)
ddppo_status conv_bwd(ddppo_ctx* ctx, const ConvGeom& g, const float* x, const float* w, const float* dy, float* dw,
                      float* dx, int accumulate_dx, const ConvScratch& sc, cudaStream_t st) {
  const int K = g.K(), M = g.M();
  // wgrad: dWr[o][k] = sum_m dy[m][o] col[m][k]   (split-K over the M output pixels)
  const float* colp = x;
  if (!g.direct()) {
    im2col_kernel<<<blocks_for(ctx, (size_t)M * K), kThreads, 0, st>>>(x, g.F, g.H, g.W, g.Ci, g.k, g.s, g.p, g.Ho,
                                                                       g.Wo, sc.col);
    ctx->count(1);
    colp = sc.col;
  }
  const int splits = std::max(1, std::min(64, M / 2048));
  ddppo_status s =
      launch_gemm_tc(ctx, GemmTC{dy, 1, g.Co, colp, 1, K, sc.dwr, K, g.Co, K, M, splits, sc.part, kPrecBwd}, st);
  if (s != DDPPO_OK) return s;
  reorder_w_kernel<<<blocks_for(ctx, (size_t)g.Co * K), kThreads, 0, st>>>(sc.dwr, g.Co, g.Ci, g.k, dw, 0);
  ctx->count(1);
  if (dx == nullptr) return DDPPO_OK;
  // dgrad: dcol[m][k] = sum_o dy[m][o] Wr[o][k]; then col2im (a gather: fixed order)
  reorder_w_kernel<<<blocks_for(ctx, (size_t)g.Co * K), kThreads, 0, st>>>(w, g.Co, g.Ci, g.k, sc.wr, 1);
  ctx->count(1);
  if (g.direct() && !accumulate_dx) {
    s = launch_gemm_tc(ctx, GemmTC{dy, g.Co, 1, sc.wr, 1, K, dx, K, M, K, g.Co, 1, nullptr, kPrecBwd}, st);
    if (s != DDPPO_OK) return s;
  } else {
    s = launch_gemm_tc(ctx, GemmTC{dy, g.Co, 1, sc.wr, 1, K, sc.dcol, K, M, K, g.Co, 1, nullptr, kPrecBwd}, st);
    if (s != DDPPO_OK) return s;
    col2im_kernel<<<blocks_for(ctx, (size_t)g.F * g.H * g.W * g.Ci), kThreads, 0, st>>>(
        sc.dcol, g.F, g.H, g.W, g.Ci, g.k, g.s, g.p, g.Ho, g.Wo, dx, accumulate_dx);
    ctx->count(1);
  }
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  return DDPPO_OK;
}

// z = (relu)(GN(y) (+ residual)); stats [F][16][2] = (mean, rstd)
ddppo_status gn_fwd(ddppo_ctx* ctx, int F, int HW, int C, const float* y, const float* gamma, const float* beta,
                    const float* residual, int relu, float* stats, float* z, cudaStream_t st) {
  gn_stats_kernel<<<F * kGroups, kThreads, 0, st>>>(y, HW, C, stats);
  ctx->count(1);
  gn_apply_kernel<<<blocks_for(ctx, (size_t)F * HW * C), kThreads, 0, st>>>(y, stats, gamma, beta, residual, F, HW, C,
                                                                            relu, z);
  ctx->count(1);
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  return DDPPO_OK;
}

// dz: gradient wrt z; relu_z: z if a ReLU produced it (mask z > 0), else null.  Writes dy (gradient
// wrt y), dgamma, dbeta.  dzm [F*HW*C] and part [32][C][2] are scratch.
ddppo_status gn_bwd(ddppo_ctx* ctx, int F, int HW, int C, const float* dz, const float* relu_z, const float* y,
                    const float* stats, const float* gamma, float* dy, float* dgamma, float* dbeta, float* dzm,
                    float* part, cudaStream_t st) {
  gn_bwd_kernel<<<F * kGroups, kThreads, 0, st>>>(dz, relu_z, y, stats, gamma, HW, C, dy, dzm);
  ctx->count(1);
  gn_param_partial_kernel<<<dim3((C + 127) / 128, kGnChunks), 128, 0, st>>>(dzm, y, stats, F, HW, C, part);
  ctx->count(1);
  gn_param_reduce_kernel<<<(C + 127) / 128, 128, 0, st>>>(part, C, dgamma, dbeta);
  ctx->count(1);
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  return DDPPO_OK;
}

ConvGeom geom_of(const Plan& P, const ConvGN& c) { return ConvGeom{P.F, c.H, c.W, c.Ci, c.Co, c.k, c.s, c.p, c.Ho, c.Wo}; }
ConvScratch scratch_of(const Plan& P) { return ConvScratch{P.col, P.wr, P.dcol, P.dwr, P.part}; }

// conv (+GN (+residual) (+ReLU)) forward
ddppo_status conv_gn_fwd(ddppo_ctx* ctx, const float* prm, Plan& P, ConvGN& c, const float* residual, int relu,
                         cudaStream_t st) {
  ddppo_status s = conv_fwd(ctx, geom_of(P, c), c.x, prm + c.w, c.y, scratch_of(P), st);
  if (s != DDPPO_OK) return s;
  return gn_fwd(ctx, P.F, c.Ho * c.Wo, c.Co, c.y, prm + c.gw, prm + c.gb, residual, relu, c.stats, c.z, st);
}

// backward of conv+GN: dz = gradient wrt the GN(+residual)(+ReLU) output; relu_z = that output if a
// ReLU followed (its > 0 mask), else null.  Writes dW, dgamma, dbeta into grad; dx (+)= into dx.
// The masked dz for dgamma / dbeta lives in P.dcol, free until the dgrad GEMM.
ddppo_status conv_gn_bwd(ddppo_ctx* ctx, const float* prm, float* grad, Plan& P, ConvGN& c, const float* dz,
                         const float* relu_z, float* dx, int accumulate_dx, cudaStream_t st) {
  ddppo_status s = gn_bwd(ctx, P.F, c.Ho * c.Wo, c.Co, dz, relu_z, c.y, c.stats, prm + c.gw, P.dtmp, grad + c.gw,
                          grad + c.gb, P.dcol, P.gn_part, st);
  if (s != DDPPO_OK) return s;
  return conv_bwd(ctx, geom_of(P, c), c.x, prm + c.w, P.dtmp, grad + c.w, dx, accumulate_dx, scratch_of(P), st);
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
  gather_obs_kernel<<<blocks_for(ctx, (size_t)F * kImg * kImg), kThreads, 0, st>>>(b.obs, b.env_idx, b.T, b.T_run, F,
                                                                                    P.x0);
  ctx->count(1);
  ddppo_status s = conv_gn_fwd(ctx, prm, P, P.convs[0], nullptr, 1, st);
  if (s != DDPPO_OK) return s;
  {
    ConvGN& c = P.convs[0];
    const int hp = (c.Ho + 2 - 3) / 2 + 1;
    maxpool_fwd_kernel<<<blocks_for(ctx, (size_t)F * hp * hp * 32), kThreads, 0, st>>>(c.z, F, c.Ho, c.Wo, 32, hp, hp,
                                                                                       P.pool_out, P.pool_arg);
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
  if ((s = launch_gemm_tc(ctx, GemmTC{P.flat, 512, 1, prm + off_of(L, "visual_fc.weight"), 512, 1, P.vis, 512, F, 512,
                                      512, 1, nullptr, kPrecFwd},
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
  if ((s = launch_gemm_tc(ctx, GemmTC{P.xin, kXin, 1, prm + off_of(L, "rnn.weight_ih"), kXin, 1, P.GI, kG4, F, kG4,
                                      kXin, 1, nullptr, kPrecFwd},
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
  if ((s = launch_gemm_tc(ctx, GemmTC{P.dG, 1, kG4, P.xin, 1, kXin, grad + off_of(L, "rnn.weight_ih"), kXin, kG4, kXin,
                                      F},
                          st)) != DDPPO_OK)
    return s;
  if ((s = launch_gemm_tc(ctx, GemmTC{P.dG, 1, kG4, P.Hin, 1, kH, grad + off_of(L, "rnn.weight_hh"), kH, kG4, kH, F},
                          st)) != DDPPO_OK)
    return s;
  if ((s = launch_colsum(ctx, P.dG, kG4, F, kG4, grad + off_of(L, "rnn.bias_ih"), st)) != DDPPO_OK) return s;
  if ((s = launch_colsum(ctx, P.dG, kG4, F, kG4, grad + off_of(L, "rnn.bias_hh"), st)) != DDPPO_OK) return s;
  // dx = dG W_ih  [F][576]
  if ((s = launch_gemm_tc(ctx, GemmTC{P.dG, kG4, 1, prm + off_of(L, "rnn.weight_ih"), 1, kXin, P.dxin, kXin, F, kXin,
                                      kG4},
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
  if ((s = launch_gemm_tc(ctx, GemmTC{P.dvis, 1, 512, P.flat, 1, 512, grad + off_of(L, "visual_fc.weight"), 512, 512,
                                      512, F},
                          st)) != DDPPO_OK)
    return s;
  if ((s = launch_colsum(ctx, P.dvis, 512, F, 512, grad + off_of(L, "visual_fc.bias"), st)) != DDPPO_OK) return s;
  if ((s = launch_gemm_tc(ctx, GemmTC{P.dvis, 512, 1, prm + off_of(L, "visual_fc.weight"), 1, 512, P.dflat, 512, F,
                                      512, 512},
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
  const int Ho = (H + 2 * p - k) / s + 1, Wo = (W + 2 * p - k) / s + 1;
  ConvGeom g{F, H, W, Ci, Co, k, s, p, Ho, Wo};
  const size_t mk = (size_t)g.M() * g.K(), ok = (size_t)Co * g.K();
  const size_t need = (2 * mk + 2 * ok + 64 * ok) * sizeof(float) + 5 * 256;
  if (host_need) *host_need = need;
  if (!scratch) return DDPPO_OK;
  DDPPO_REQUIRE(ctx, scratch_bytes >= need, "conv2d: scratch too small");
  char* b = reinterpret_cast<char*>(scratch);
  auto take = [&](size_t n) {
    float* r = reinterpret_cast<float*>(b);
    b += align_up(n * sizeof(float), 256);
    return r;
  };
  ConvScratch sc;
  sc.col = take(mk);
  sc.dcol = take(mk);
  sc.wr = take(ok);
  sc.dwr = take(ok);
  sc.part = take(64 * ok);
  cudaStream_t st = as_stream(stream);
  ProfScope ps(ctx, DDPPO_K_OTHER, st, 0);
  if (y) {
    ddppo_status r = conv_fwd(ctx, g, x, w, y, sc, st);
    if (r != DDPPO_OK) return r;
  }
  if (dy) return conv_bwd(ctx, g, x, w, dy, dw, dx, 0, sc, st);
  return DDPPO_OK;
}

extern "C" ddppo_status ddppo_debug_groupnorm(ddppo_ctx* ctx, const float* y, const float* gamma, const float* beta,
                                              const float* residual, int F, int HW, int C, int relu, float* z,
                                              float* stats, const float* dz, float* dy, float* dgamma, float* dbeta,
                                              float* scratch, void* stream) {
  if (!ctx) return DDPPO_ERR_CONFIG;
  DDPPO_REQUIRE(ctx, F >= 1 && HW >= 1 && C >= kGroups && C % kGroups == 0, "groupnorm: C must be a multiple of 16");
  cudaStream_t st = as_stream(stream);
  ProfScope ps(ctx, DDPPO_K_OTHER, st, 0);
  ddppo_status r = gn_fwd(ctx, F, HW, C, y, gamma, beta, residual, relu, stats, z, st);
  if (r != DDPPO_OK || !dz) return r;
  return gn_bwd(ctx, F, HW, C, dz, relu ? z : nullptr, y, stats, gamma, dy, dgamma, dbeta, scratch,
                scratch + (size_t)F * HW * C, st);
}

extern "C" ddppo_status ddppo_debug_maxpool(ddppo_ctx* ctx, const float* x, int F, int H, int W, int C, float* y,
                                            uint8_t* arg, const float* dy, float* dx, void* stream) {
  if (!ctx) return DDPPO_ERR_CONFIG;
  DDPPO_REQUIRE(ctx, F >= 1 && H >= 2 && W >= 2 && C >= 1, "maxpool: bad geometry");
  const int Ho = (H + 2 - 3) / 2 + 1, Wo = (W + 2 - 3) / 2 + 1;
  cudaStream_t st = as_stream(stream);
  ProfScope ps(ctx, DDPPO_K_OTHER, st, 0);
  maxpool_fwd_kernel<<<blocks_for(ctx, (size_t)F * Ho * Wo * C), kThreads, 0, st>>>(x, F, H, W, C, Ho, Wo, y, arg);
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
