// Visual agents (P:L212 half-width backbones with GroupNorm, App. C; readings Z17-Z23, R5,
// R7 in DESIGN.md):
//   Depth (configs[2]): 64x64 depth -> ResNet18/2 -> 128x2x2 -> FC 512 + ReLU; x = [visual, goal FC
//     32, action embedding 32] -> LSTM-512 -> Linear(512, 5).
//   RGB-D (configs[3]): 4x256x256 (RGB normalised channel-wise) -> 2x2 avg-pool -> ResNet50/2
//     (bottlenecks 3/4/6/3) -> 128x4x4 -> FC 2048->512 + ReLU; same x -> 2-layer LSTM-512 -> head.
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
#include <map>
#include <utility>
#include <vector>

#include "common.cuh"

namespace {

constexpr int kXin = 576, kA1 = 5, kGroups = 16, kThreads = 256;
constexpr int kImg = 64;        // Depth input resolution (configs[2])
constexpr int kImgRgbd = 256;   // RGB-D input resolution (configs[3])

// ------------------------------------------------------------------ kernels
// obs [E][T][1][64][64] bf16 (gathered through env_idx) -> x0 [F][64][64][1] fp32 (the stem's input)
__global__ void gather_obs_kernel(const __nv_bfloat16* __restrict__ obs, const int32_t* __restrict__ env_idx, int T,
                                  int T_run, int F, float* __restrict__ x0) {
  pdl_enter();
  const size_t per = (size_t)kImg * kImg / 8;  // 8 pixels (16 bytes) per item
  const size_t n = (size_t)F * per;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int f = (int)(i / per);
    const int b = f / T_run, t = f - b * T_run;
    const uint4 raw = reinterpret_cast<const uint4*>(obs + ((size_t)env_idx[b] * T + t) * kImg * kImg)[i % per];
    const __nv_bfloat16* v = reinterpret_cast<const __nv_bfloat16*>(&raw);
    float4* o = reinterpret_cast<float4*>(x0) + 2 * i;
    o[0] = make_float4(__bfloat162float(v[0]), __bfloat162float(v[1]), __bfloat162float(v[2]), __bfloat162float(v[3]));
    o[1] = make_float4(__bfloat162float(v[4]), __bfloat162float(v[5]), __bfloat162float(v[6]), __bfloat162float(v[7]));
  }
}

// RGB-D prologue: camera bytes rgb [E][T][3][256][256] and depth [E][T][1][256][256] (bf16) ->
// channel-wise RGB normalisation, 2x2 average pooling -> x0 [F][128][128][8] fp32 NHWC
// (channels 4..7 zero: the stem's implicit GEMM reads 8 channels per 16-byte piece) and its bf16
// hi / lo planes
__constant__ float kRgbMean[3] = {0.485f * 255.f, 0.456f * 255.f, 0.406f * 255.f};
__constant__ float kRgbStd[3] = {0.229f * 255.f, 0.224f * 255.f, 0.225f * 255.f};
__global__ void rgbd_prologue_kernel(const uint8_t* __restrict__ rgb, const __nv_bfloat16* __restrict__ depth,
                                     const int32_t* __restrict__ env_idx, int T, int T_run, int F, int Hin,
                                     float* __restrict__ x0, __nv_bfloat16* __restrict__ x0b) {
  pdl_enter();
  // thread = (frame, output row, pair of output columns): 4 input columns of 2 rows per channel
  const int Ho = Hin / 2, Wo = Hin / 2, WP = Wo / 2;
  const int item = blockIdx.x * blockDim.x + threadIdx.x;
  if (item >= F * Ho * WP) return;
  const int jp = item % WP, ii = (item / WP) % Ho, f = item / (WP * Ho);
  const int b = f / T_run, t = f - b * T_run;
  const size_t fr = (size_t)env_idx[b] * T + t, px = (size_t)(2 * ii) * Hin + 4 * jp;
  float r0[4][4], r1[4][4];  // [channel][column]
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const uint8_t* s = rgb + (fr * 3 + c) * Hin * Hin + px;
    const uchar4 a = *reinterpret_cast<const uchar4*>(s), bb = *reinterpret_cast<const uchar4*>(s + Hin);
    r0[c][0] = a.x; r0[c][1] = a.y; r0[c][2] = a.z; r0[c][3] = a.w;
    r1[c][0] = bb.x; r1[c][1] = bb.y; r1[c][2] = bb.z; r1[c][3] = bb.w;
  }
  {
    const __nv_bfloat16* s = depth + fr * Hin * Hin + px;
    const uint2 a = *reinterpret_cast<const uint2*>(s), bb = *reinterpret_cast<const uint2*>(s + Hin);
    const __nv_bfloat16* av = reinterpret_cast<const __nv_bfloat16*>(&a);
    const __nv_bfloat16* bv = reinterpret_cast<const __nv_bfloat16*>(&bb);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      r0[3][q] = __bfloat162float(av[q]);
      r1[3][q] = __bfloat162float(bv[q]);
    }
  }
  const size_t n = (size_t)F * Ho * Wo * 8;
#pragma unroll
  for (int h = 0; h < 2; ++h) {  // output pixel (ii, 2*jp + h)
    float v[8];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const float m = c < 3 ? kRgbMean[c] : 0.f, inv = c < 3 ? 1.f / kRgbStd[c] : 1.f;
      const float a0 = r0[c][2 * h], a1 = r0[c][2 * h + 1], b0 = r1[c][2 * h], b1 = r1[c][2 * h + 1];
      v[c] = 0.25f * (((a0 - m) * inv + (a1 - m) * inv) + ((b0 - m) * inv + (b1 - m) * inv));
      v[c + 4] = 0.f;
    }
    const size_t o = (((size_t)f * Ho + ii) * Wo + 2 * jp + h) * 8;
    *reinterpret_cast<float4*>(x0 + o) = make_float4(v[0], v[1], v[2], v[3]);
    *reinterpret_cast<float4*>(x0 + o + 4) = make_float4(0.f, 0.f, 0.f, 0.f);
    __nv_bfloat16 hi[8], lo[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      hi[c] = __float2bfloat16_rn(v[c]);
      lo[c] = __float2bfloat16_rn(v[c] - __bfloat162float(hi[c]));
    }
    *reinterpret_cast<uint4*>(x0b + o) = *reinterpret_cast<const uint4*>(hi);
    *reinterpret_cast<uint4*>(x0b + n + o) = *reinterpret_cast<const uint4*>(lo);
  }
}

// Weight layouts for the implicit GEMMs.  W [Co][Ci][k][k] (PyTorch) ->
//   Wr [Co][(u, v, c)] as bf16 hi / lo planes (plane = Co*k*k*Ci elements)  (forward B operand)
//   Wd [Ci][(u, v, o)] bf16                                                (input-gradient B operand)
__global__ void weights_bf16_kernel(const float* __restrict__ W, int Co, int Ci, int k, __nv_bfloat16* __restrict__ wr,
                                    __nv_bfloat16* __restrict__ wd) {
  pdl_enter();
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
// all convolutions' weights of one minibatch in one launch: the convolutions' Wr index ranges are
// concatenated (off[i] = start of convolution i), one thread per element; Cp >= Ci is the padded
// channel count of the GEMM operand (extra channels get zero weights)
constexpr int kMaxConvs = 128;
struct WeightPrep {
  int n;
  int off[kMaxConvs + 1];   // prefix sums of the Wr block counts (Co per convolution)
  int offd[kMaxConvs + 1];  // prefix sums of the Wd block counts (Ci per convolution; 0 without wd)
  struct Item {
    const float* W;
    __nv_bfloat16 *wr, *wd;  // wd nullable (no input gradient)
    int Co, Ci, Cp, k;
    int wd_planes;           // 2: Wd also as a lo plane (at wd + Co*Cp*k*k), for hi / lo input gradients
    int groups;              // > 1: W is grouped [Co][Ci/groups][k][k]; the dense operand is block diagonal
  } it[kMaxConvs];
};
// W[o][c][uv] of convolution t as a dense [Co][Ci] operand entry (0 off the block diagonal of a grouped conv)
__device__ __forceinline__ float prep_weight(const WeightPrep::Item& t, int o, int c, int uv, int kk) {
  if (t.groups > 1) {
    const int cgi = t.Ci / t.groups, cgo = t.Co / t.groups;
    return c / cgi == o / cgo ? t.W[(o * cgi + c % cgi) * kk + uv] : 0.f;
  }
  return c < t.Ci ? t.W[(o * t.Ci + c) * kk + uv] : 0.f;
}
__device__ __forceinline__ int prep_item(const int* off, int n, int g) {  // off[lo] <= g < off[lo + 1]
  int lo = 0, hi_i = n - 1;
  while (lo < hi_i) {
    const int mid = (lo + hi_i + 1) >> 1;
    if (off[mid] <= g) lo = mid;
    else hi_i = mid - 1;
  }
  return lo;
}
// One block per output row of Wr [Co][(u,v,c)] (blocks [0, off[n]): conv item, o) and one per input
// channel row of Wd [Ci][(u,v,o)] (blocks [off[n], off[n] + offd[n]): item, c), so that every store
// is coalesced; the reads of W [Co][Ci][k][k] stay within one row (Wr) or touch one k*k run per o (Wd).
__global__ void __launch_bounds__(256) weights_prep_kernel(const WeightPrep prep) {
  pdl_enter();
  const int blk = blockIdx.x, nr = prep.off[prep.n];
  const bool is_wr = blk < nr;
  const int* off = is_wr ? prep.off : prep.offd;
  const int bl = is_wr ? blk : blk - nr;
  if (!is_wr && bl >= prep.offd[prep.n]) return;
  const int it = prep_item(off, prep.n, bl);
  const WeightPrep::Item& t = prep.it[it];
  const int kk = t.k * t.k, n = t.Co * t.Cp * kk, row = bl - off[it];
  if (is_wr) {
    const int o = row;
    for (int e = threadIdx.x; e < kk * t.Cp; e += blockDim.x) {
      const int uv = e / t.Cp, c = e - uv * t.Cp;
      const float w = prep_weight(t, o, c, uv, kk);
      const __nv_bfloat16 hi = __float2bfloat16_rn(w);
      t.wr[(size_t)o * kk * t.Cp + e] = hi;
      t.wr[n + (size_t)o * kk * t.Cp + e] = __float2bfloat16_rn(w - __bfloat162float(hi));
    }
  } else {
    const int c = row;
    for (int e = threadIdx.x; e < kk * t.Co; e += blockDim.x) {
      const int uv = e / t.Co, o = e - uv * t.Co;
      const float w = prep_weight(t, o, c, uv, kk);
      const __nv_bfloat16 hi = __float2bfloat16_rn(w);
      t.wd[(size_t)c * kk * t.Co + e] = hi;
      if (t.wd_planes == 2) t.wd[n + (size_t)c * kk * t.Co + e] = __float2bfloat16_rn(w - __bfloat162float(hi));
    }
  }
}
// fp32 -> bf16 hi / lo planes (plane = n)
__global__ void to_planes_kernel(const float* __restrict__ x, size_t n, __nv_bfloat16* __restrict__ xb) {
  pdl_enter();
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const __nv_bfloat16 hi = __float2bfloat16_rn(x[i]);
    xb[i] = hi;
    xb[n + i] = __float2bfloat16_rn(x[i] - __bfloat162float(hi));
  }
}
__global__ void to_bf16_kernel(const float* __restrict__ x, size_t n, __nv_bfloat16* __restrict__ xb) {
  pdl_enter();
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    xb[i] = __float2bfloat16_rn(x[i]);
}

// Single-channel stem convolution in fp32 SIMT (K = k*k taps over 1 channel is too narrow for the
// 16-byte implicit-GEMM pieces): block per frame, the zero-padded frame and the weights staged in
// shared memory (no bounds tests in the tap loops, which unroll: K, S compile-time); a thread computes
// 8 horizontally adjacent pixels x 8 output channels per work item, so every weight load (float4 x
// 2, broadcast) feeds 64 FMAs.
constexpr int kStemCoMax = 32;
template <int K, int S>
__global__ void __launch_bounds__(kThreads) stem_fwd_kernel(const float* __restrict__ x, const float* __restrict__ W,
                                                            int H, int Wd, int Co, int p, int Ho, int Wo,
                                                            float* __restrict__ y) {
  pdl_enter();
  extern __shared__ __align__(16) float sm[];
  constexpr int kk = K * K;
  const int Hp = H + 2 * p, Wp = Wd + 2 * p + 8 * S;  // + a right margin: the last item's unused columns
  float* ws = sm;                                     // [k*k][Co]   (Co % 8 == 0)
  float* xs = sm + kk * Co;                           // [Hp][Wp], zero borders
  const int f = blockIdx.x;
  for (int i = threadIdx.x; i < Hp * Wp; i += blockDim.x) {
    const int r = i / Wp - p, q = i % Wp - p;
    xs[i] = (r >= 0 && r < H && q >= 0 && q < Wd) ? x[((size_t)f * H + r) * Wd + q] : 0.f;
  }
  for (int i = threadIdx.x; i < Co * kk; i += blockDim.x) ws[(i % kk) * Co + i / kk] = W[i];
  __syncthreads();
  constexpr int kPx = 8;  // horizontally adjacent output pixels per work item (x 8 channels: 64 FMAs per tap)
  const int og = Co / 8, jg = (Wo + kPx - 1) / kPx;
  for (int item = threadIdx.x; item < Ho * jg * og; item += blockDim.x) {
    const int o0 = (item % og) * 8, rest = item / og, j0 = (rest % jg) * kPx, i = rest / jg;
    float acc[kPx][8];
#pragma unroll
    for (int a = 0; a < kPx; ++a)
#pragma unroll
      for (int o = 0; o < 8; ++o) acc[a][o] = 0.f;
#pragma unroll 1
    for (int u = 0; u < K; ++u) {
      const float* xr = xs + (i * S + u) * Wp + j0 * S;  // padded coordinates: (i*S - p + u) + p
#pragma unroll
      for (int v = 0; v < K; ++v) {
        const float4 w0 = *reinterpret_cast<const float4*>(ws + (u * K + v) * Co + o0);
        const float4 w1 = *reinterpret_cast<const float4*>(ws + (u * K + v) * Co + o0 + 4);
        const float wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
        for (int a = 0; a < kPx; ++a) {
          const float xv = xr[a * S + v];
#pragma unroll
          for (int o = 0; o < 8; ++o) acc[a][o] = fmaf(xv, wv[o], acc[a][o]);
        }
      }
    }
#pragma unroll
    for (int a = 0; a < kPx; ++a) {
      if (j0 + a >= Wo) break;
      float* yo = y + (((size_t)f * Ho + i) * Wo + j0 + a) * Co + o0;
      *reinterpret_cast<float4*>(yo) = make_float4(acc[a][0], acc[a][1], acc[a][2], acc[a][3]);
      *reinterpret_cast<float4*>(yo + 4) = make_float4(acc[a][4], acc[a][5], acc[a][6], acc[a][7]);
    }
  }
}
// per-frame partial weight gradient of the stem: part[f][o*k*k + tap] = sum_q dy[f][q][o] col[q][tap].
// The frame (zero-padded) and all of its dy rows (bf16) sit in shared memory, loaded once; the
// im2col values are read straight from the padded frame.  Register-blocked outer products: thread
// (half, o-quad, tap-quad) accumulates a 4 x 4 tile over the output rows of its parity; the two
// halves are added in a fixed order at the end.
__global__ void __launch_bounds__(kThreads) stem_wgrad_kernel(const float* __restrict__ x,
                                                              const __nv_bfloat16* __restrict__ dy, int H, int Wd,
                                                              int Co, int k, int s, int p, int Ho, int Wo,
                                                              float* __restrict__ part) {
  pdl_enter();
  extern __shared__ __align__(16) float sm[];
  const int HP = H + 2 * p, WP = Wd + 2 * p;
  __nv_bfloat16* dys = reinterpret_cast<__nv_bfloat16*>(sm);           // [Ho*Wo][Co]
  float* xp = sm + (Ho * Wo * Co / 2 + 3) / 4 * 4;                      // [HP][WP] zero-padded frame
  const int f = blockIdx.x, kk = k * k;
  {
    const uint4* src = reinterpret_cast<const uint4*>(dy + (size_t)f * Ho * Wo * Co);
    uint4* dst = reinterpret_cast<uint4*>(dys);
    for (int i = threadIdx.x; i < Ho * Wo * Co / 8; i += blockDim.x) dst[i] = src[i];
  }
  for (int i = threadIdx.x; i < HP * WP; i += blockDim.x) {
    const int yy = i / WP - p, xx = i % WP - p;
    xp[i] = (yy >= 0 && yy < H && xx >= 0 && xx < Wd) ? x[((size_t)f * H + yy) * Wd + xx] : 0.f;
  }
  __syncthreads();
  const int half = threadIdx.x >> 7, r = threadIdx.x & 127;
  const int oq = Co / 4, o0 = 4 * (r % oq), t0 = 4 * (r / oq);
  const bool active = r < oq * 16;  // 16 tap quads cover k*k <= 64
  int off[4];
#pragma unroll
  for (int kq = 0; kq < 4; ++kq) {
    const int tap = t0 + kq;
    off[kq] = tap < kk ? (tap / k) * WP + (tap % k) : 0;  // taps past k*k: computed, never stored
  }
  float acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b2 = 0; b2 < 4; ++b2) acc[a][b2] = 0.f;
  if (active) {
    for (int i = half; i < Ho; i += 2) {
      const float* xrow = xp + i * s * WP;
      const __nv_bfloat16* drow = dys + (size_t)i * Wo * Co + o0;
#pragma unroll 4
      for (int j = 0; j < Wo; ++j) {
        const float* xb = xrow + j * s;
        const float cv[4] = {xb[off[0]], xb[off[1]], xb[off[2]], xb[off[3]]};
        const uint2 d2 = *reinterpret_cast<const uint2*>(drow + j * Co);
        const float2 d01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&d2.x));
        const float2 d23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&d2.y));
        const float dv[4] = {d01.x, d01.y, d23.x, d23.y};
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b2 = 0; b2 < 4; ++b2) acc[a][b2] = fmaf(dv[a], cv[b2], acc[a][b2]);
      }
    }
  }
  __syncthreads();
  float* red = xp;  // [128][16] partials of the odd half (the frame is no longer needed)
  if (half == 1 && active)
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b2 = 0; b2 < 4; ++b2) red[r * 16 + a * 4 + b2] = acc[a][b2];
  __syncthreads();
  if (half == 0 && active) {
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b2 = 0; b2 < 4; ++b2) {
        const int tap = t0 + b2;
        if (tap < kk) part[(size_t)f * Co * kk + (o0 + a) * kk + tap] = acc[a][b2] + red[r * 16 + a * 4 + b2];
      }
  }
}

// ---- stem on the warp-level tensor path (mma.sync m16n8k16 bf16 -> fp32) ----
// The single-channel stem has K = k*k <= 49 taps: too narrow for the 16-byte TMA / tcgen05 pieces
// (its one-channel im2col cannot be a TMA box) but dense enough for warp MMAs whose fragments are
// gathered straight from the zero-padded frame in shared memory.  The frame is staged as packed
// bf16 (hi | lo << 16) pairs, x = hi + lo to 2^-17, so one 32-bit shared load yields both planes.
__device__ __forceinline__ void mma_bf16_16816(float* d, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
               "{%0,%1,%2,%3};\n"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_hilo(float v) {
  const __nv_bfloat16 hi = __float2bfloat16_rn(v);
  const __nv_bfloat16 lo = __float2bfloat16_rn(v - __bfloat162float(hi));
  return (uint32_t)__bfloat16_as_ushort(hi) | ((uint32_t)__bfloat16_as_ushort(lo) << 16);
}
// zero-padded frame f -> xp[HP][WP] packed hi/lo; returns (block-uniformly, after the barrier)
// whether any lo half is nonzero -- a frame of bf16 values (the Depth observations are stored as
// bf16) has an all-zero lo plane, whose MMAs then add exact zeros and are skipped
// The stem's input frames: x [F][H][W] fp32, or (obs != null) straight from the rollout's bf16
// observations obs [E][T][H][W], frame f = (env b = f / T_run, step t = f % T_run) of env_idx[b]
// (the Depth step then needs no gather pass: the frames are read where they lie)
struct FrameSrc {
  const float* x;
  const __nv_bfloat16* obs;
  const int32_t* env_idx;
  int T, T_run;
};
__device__ __forceinline__ bool stage_frame_hilo(const FrameSrc& fs, int f, int H, int Wd, int p, int HP, int WP,
                                                 uint32_t* xp) {
  int any_lo = 0;
  constexpr int kB = 8;  // loads in flight per thread (the loop is latency-bound otherwise)
  const float* xf = nullptr;
  const __nv_bfloat16* of = nullptr;
  if (fs.obs) {
    const int b = f / fs.T_run, t = f - b * fs.T_run;
    of = fs.obs + ((size_t)fs.env_idx[b] * fs.T + t) * H * Wd;
  } else {
    xf = fs.x + (size_t)f * H * Wd;
  }
  for (int i0 = 0; i0 < HP * WP; i0 += kB * (int)blockDim.x) {
    float v[kB];
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      const int i = i0 + u * blockDim.x + threadIdx.x, r = i / WP - p, q = i % WP - p;
      v[u] = (i < HP * WP && r >= 0 && r < H && q >= 0 && q < Wd) ? (of ? __bfloat162float(of[r * Wd + q]) : xf[r * Wd + q])
                                                                  : 0.f;
    }
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      const int i = i0 + u * blockDim.x + threadIdx.x;
      const uint32_t pk = pack_hilo(v[u]);
      any_lo |= (pk >> 16) & 0x7fff;  // (a -0 lo half would add -0 products: exact no-ops too)
      if (i < HP * WP) xp[i] = pk;
    }
  }
  return __syncthreads_or(any_lo) != 0;
}

// y[f][q][o] = sum_tap col[q][tap] W[o][tap] as an M = pixels x N = Co x K = taps (padded to 16)
// GEMM per frame, bf16x3 (xh Wh + xh Wl + xl Wh, the forward convention of the other convs).  Block
// per frame; warp w takes the 16-pixel m-tiles w, w + 8, ...; the W fragments stay in registers.
// gsum (nullable): the frame's GroupNorm sums [F][16][2] = (sum y, sum y^2) per group (double; the
// per-thread sums in pixel order, then a fixed butterfly over the 8 row lanes and the warps in
// order), so the stem's GroupNorm needs no statistics pass over y.
template <int K, int S, int CO>
__global__ void __launch_bounds__(kThreads, 2) stem_fwd_mma_kernel(const FrameSrc x,
                                                                   const float* __restrict__ W, int H, int Wd,
                                                                   int p, int Ho, int Wo, float* __restrict__ y,
                                                                   double* __restrict__ gsum) {
  constexpr int kk = K * K, KS = (kk + 15) / 16, NT = CO / 8;
  constexpr int CG = CO / kGroups, GE = CG == 2 ? 1 : 2;  // channels per group; groups per (thread, n-tile)
  static_assert(CO % kGroups == 0 && CG <= 2, "stem: 16 or 32 channels");
  extern __shared__ __align__(16) uint32_t smu[];
  __shared__ double gred[kThreads / 32][CO][2];
  const int HP = H + 2 * p, WP = Wd + 2 * p;
  const int f = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  pdl_enter();  // W is the parameter vector the previous step's update writes
  // B fragments (k = tap, n = o): b0 = taps 16ks + 2t, +1; b1 = taps 16ks + 2t + 8, +9; column o = 8nt + g
  uint32_t bh[KS][NT][2], bl[KS][NT][2];
  int toff[KS][4];  // frame offsets of taps 16ks + 2t + {0, 1, 8, 9} (0 past k*k: W is zero there)
#pragma unroll
  for (int ks = 0; ks < KS; ++ks) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int tap = 16 * ks + 2 * t + (e & 1) + (e >> 1) * 8;
      toff[ks][e] = tap < kk ? (tap / K) * WP + tap % K : 0;
    }
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int tap = 16 * ks + 2 * t + 8 * h, o = 8 * nt + g;
        const uint32_t p0 = tap < kk ? pack_hilo(W[o * kk + tap]) : 0u;
        const uint32_t p1 = tap + 1 < kk ? pack_hilo(W[o * kk + tap + 1]) : 0u;
        bh[ks][nt][h] = __byte_perm(p0, p1, 0x5410);
        bl[ks][nt][h] = __byte_perm(p0, p1, 0x7632);
      }
  }
  const bool x_lo = stage_frame_hilo(x, f, H, Wd, p, HP, WP, smu);
  const int M = Ho * Wo;
  double s1[NT][GE], s2[NT][GE];  // group sums of this thread's columns 8nt + 2t (+ 1)
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int e = 0; e < GE; ++e) s1[nt][e] = s2[nt][e] = 0.0;
  for (int m0 = warp * 16; m0 < M; m0 += 16 * (kThreads / 32)) {
    int base[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int q = m0 + g + 8 * h, i = q / Wo, j = q % Wo;
      base[h] = i * S * WP + j * S;
    }
    float acc[NT][4];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[nt][e] = 0.f;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      // A (row = pixel, k = tap): a0 (g, 2t..), a1 (g + 8, 2t..), a2 (g, 2t + 8..), a3 (g + 8, 2t + 8..)
      uint32_t ah[4], al[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int b = base[r & 1], e0 = (r >> 1) * 2;
        const uint32_t p0 = smu[b + toff[ks][e0]], p1 = smu[b + toff[ks][e0 + 1]];
        ah[r] = __byte_perm(p0, p1, 0x5410);
        al[r] = __byte_perm(p0, p1, 0x7632);
      }
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        mma_bf16_16816(acc[nt], ah, bh[ks][nt][0], bh[ks][nt][1]);
        mma_bf16_16816(acc[nt], ah, bl[ks][nt][0], bl[ks][nt][1]);
        if (x_lo) mma_bf16_16816(acc[nt], al, bh[ks][nt][0], bh[ks][nt][1]);
      }
    }
    float* yf = y + (size_t)f * M * CO;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      *reinterpret_cast<float2*>(yf + (size_t)(m0 + g) * CO + 8 * nt + 2 * t) = make_float2(acc[nt][0], acc[nt][1]);
      *reinterpret_cast<float2*>(yf + (size_t)(m0 + g + 8) * CO + 8 * nt + 2 * t) =
          make_float2(acc[nt][2], acc[nt][3]);
    }
    if (gsum) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const double v = acc[nt][e];
          s1[nt][GE == 1 ? 0 : (e & 1)] += v;
          s2[nt][GE == 1 ? 0 : (e & 1)] += v * v;
        }
    }
  }
  if (gsum) {  // (block-uniform)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < GE; ++e)
#pragma unroll
        for (int sh = 4; sh < 32; sh <<= 1) {  // over g (lane bits 2-4)
          s1[nt][e] += __shfl_xor_sync(0xffffffffu, s1[nt][e], sh);
          s2[nt][e] += __shfl_xor_sync(0xffffffffu, s2[nt][e], sh);
        }
    if (g == 0) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < GE; ++e) {
          const int col = 8 * nt + 2 * t + e;  // GE == 1: the group's first channel holds its sums
          gred[warp][col][0] = s1[nt][e];
          gred[warp][col][1] = s2[nt][e];
        }
    }
    __syncthreads();
    if (threadIdx.x < kGroups) {
      double a = 0.0, b = 0.0;
      const int col = threadIdx.x * CG;
      for (int w = 0; w < kThreads / 32; ++w) {
        a += gred[w][col][0];
        b += gred[w][col][1];
      }
      gsum[((size_t)f * kGroups + threadIdx.x) * 2] = a;
      gsum[((size_t)f * kGroups + threadIdx.x) * 2 + 1] = b;
    }
  }
}

// part[f][o*k*k + tap] = sum_q dy[f][q][o] col[q][tap] as an M = Co x N = taps (padded to 8) x
// K = pixels GEMM per frame: A = dy^T by ldmatrix.trans from the frame's dy rows (16-byte chunks
// XOR-swizzled: conflict-free), B = im2col gathered from the packed frame, two MMAs (x hi, x lo) per
// fragment.  Warp w takes the 16-pixel k-steps w, w + 8, ...; the 8 warps' tiles are added in a
// fixed order.
template <int K, int CO>
__global__ void __launch_bounds__(kThreads, 2) stem_wgrad_mma_kernel(const FrameSrc x,
                                                                     const __nv_bfloat16* __restrict__ dy, int H,
                                                                     int Wd, int s, int p, int Ho, int Wo,
                                                                     float* __restrict__ part) {
  constexpr int kk = K * K, NT = (kk + 7) / 8, MT = CO / 16, CPR = CO / 8;  // CPR: 16-byte chunks per dy row
  constexpr int kWarps = kThreads / 32;
  pdl_enter();
  extern __shared__ __align__(16) uint32_t smu[];
  const int HP = H + 2 * p, WP = Wd + 2 * p, M = Ho * Wo;
  const int f = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  const size_t dy_words = (size_t)M * CO / 2 > (size_t)kWarps * CO * NT * 8 ? (size_t)M * CO / 2
                                                                             : (size_t)kWarps * CO * NT * 8;
  uint4* dys = reinterpret_cast<uint4*>(smu);  // [M][CPR] chunks, chunk c of row q at c ^ swz(q)
  uint32_t* xp = smu + dy_words;               // [HP][WP] packed hi/lo
  auto swz = [](int q) { return CPR == 4 ? (q >> 1) & 3 : (q >> 2) & 1; };
  {
    const uint4* src = reinterpret_cast<const uint4*>(dy + (size_t)f * M * CO);
    for (int i = threadIdx.x; i < M * CPR; i += blockDim.x) {  // all of the frame's dy rows in flight
      const int q = i / CPR, c = i % CPR;
      const uint32_t dst = (uint32_t)__cvta_generic_to_shared(dys + q * CPR + (c ^ swz(q)));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src + i) : "memory");
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  const bool x_lo = stage_frame_hilo(x, f, H, Wd, p, HP, WP, xp);
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();
  int toff[NT];  // frame offset of tap 8nt + g (0 past k*k: those columns are computed, never stored)
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const int tap = 8 * nt + g;
    toff[nt] = tap < kk ? (tap / K) * WP + tap % K : 0;
  }
  float acc[MT][NT][4];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[mt][nt][e] = 0.f;
  const uint32_t dys_addr = (uint32_t)__cvta_generic_to_shared(dys);
  for (int q0 = warp * 16; q0 < M; q0 += 16 * kWarps) {
    uint32_t a[MT][4];
    {
      const int q = q0 + (lane & 7) + ((lane >> 4) & 1) * 8;
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const int c = 2 * mt + ((lane >> 3) & 1);
        const uint32_t addr = dys_addr + (uint32_t)(q * CPR + (c ^ swz(q))) * 16u;
        asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                     : "=r"(a[mt][0]), "=r"(a[mt][1]), "=r"(a[mt][2]), "=r"(a[mt][3])
                     : "r"(addr));
      }
    }
    // B (k = pixel, n = tap): b0 = pixels q0 + 2t, +1; b1 = pixels q0 + 2t + 8, +9; column tap 8nt + g
    int base[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int q = q0 + 2 * t + (e & 1) + (e >> 1) * 8, i = q / Wo, j = q % Wo;
      base[e] = i * s * WP + j * s;
    }
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const uint32_t p0 = xp[base[0] + toff[nt]], p1 = xp[base[1] + toff[nt]];
      const uint32_t p2 = xp[base[2] + toff[nt]], p3 = xp[base[3] + toff[nt]];
      const uint32_t h0 = __byte_perm(p0, p1, 0x5410), h1 = __byte_perm(p2, p3, 0x5410);
      const uint32_t l0 = __byte_perm(p0, p1, 0x7632), l1 = __byte_perm(p2, p3, 0x7632);
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        mma_bf16_16816(acc[mt][nt], a[mt], h0, h1);
        if (x_lo) mma_bf16_16816(acc[mt][nt], a[mt], l0, l1);
      }
    }
  }
  __syncthreads();  // dy no longer needed: its space holds the per-warp tiles
  float* red = reinterpret_cast<float*>(smu);  // [warp][CO][NT*8]
  constexpr int NC = NT * 8;
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int o = 16 * mt + g + 8 * (e >> 1), c = 8 * nt + 2 * t + (e & 1);
        red[(warp * CO + o) * NC + c] = acc[mt][nt][e];
      }
  __syncthreads();
  for (int i = threadIdx.x; i < CO * kk; i += blockDim.x) {
    const int o = i / kk, tap = i % kk;
    float v = 0.f;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) v += red[(w * CO + o) * NC + tap];
    part[(size_t)f * CO * kk + i] = v;
  }
}
// dW[i] = sum over frames (fixed order) of part[f][i]
__global__ void __launch_bounds__(kThreads) frame_sum_kernel(const float* __restrict__ part, int F, int n,
                                                             float* __restrict__ out) {
  pdl_enter();
  __shared__ double red[kThreads / 32];
  double acc[1] = {0.0};
  for (int f = threadIdx.x; f < F; f += blockDim.x) acc[0] += part[(size_t)f * n + blockIdx.x];
  block_sum<1>(acc, red);
  if (threadIdx.x == 0) out[blockIdx.x] = (float)acc[0];
}

// GroupNorm (G = 16, eps 1e-5), one block per frame.  The block walks the frame's [HW][C] slab
// contiguously (coalesced); with 256 % C == 0 thread t always sees channel t % C, so per-group and
// per-channel partial sums are per-thread sums combined in a fixed order through shared memory.
constexpr int kGnMaxThreads = 1024;  // blockDim = max(256, C): a multiple of C
constexpr int kMaxConvsGn = 128;
__host__ __device__ inline int gn_threads(int C) { return C > 256 ? C : 256; }
constexpr int kGnChunk = 8192;  // elements per chunk (a multiple of every C): kGnChunk / blockDim per thread
__host__ __device__ inline int gn_chunk(int) { return kGnChunk; }
__host__ __device__ constexpr int gn_bound(int nv) { return kGnChunk / nv < 1024 ? kGnChunk / nv : 1024; }

// per-group sums of the threads' (a, b) in fixed order -> out[g] (threads t < 16 write)
__device__ __forceinline__ void gn_group_reduce(double a, double b, int C, double* sa, double* sb, double* out_a,
                                                double* out_b) {
  sa[threadIdx.x] = a;
  sb[threadIdx.x] = b;
  __syncthreads();
  if (threadIdx.x < kGroups) {
    const int cg = C / kGroups, g = threadIdx.x;
    double ra = 0.0, rb = 0.0;
    for (int rep = 0; rep < (int)blockDim.x / C; ++rep)
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
// zb (nullable): z as bf16 hi / lo planes (plane = F*HW*C).  Thread t holds elements t + i*blockDim
// (i < NV, NV*blockDim >= HW*C) in registers: every load of the slab is in flight at once and the
// slab is read from memory once.
template <int NV>
__global__ void __launch_bounds__(gn_bound(NV)) gn_fwd_kernel(const float* __restrict__ y, const float* __restrict__ gamma,
                                                            const float* __restrict__ beta,
                                                            const float* __restrict__ residual, int HW, int C,
                                                            int relu, size_t plane, float* __restrict__ stats,
                                                            float* __restrict__ z, __nv_bfloat16* __restrict__ zb) {
  pdl_enter();
  __shared__ double sa[gn_bound(NV)], sb[gn_bound(NV)], ga[kGroups], gb[kGroups];
  __shared__ float smu[kGroups], srs[kGroups];
  const int f = blockIdx.x, n = HW * C, c = threadIdx.x % C, cg = C / kGroups;
  const size_t base = (size_t)f * n;
  const float gm = gamma[c], bt = beta[c];  // (issued with the slab's loads, not after the reduction)
  float v[NV], rv[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int e = threadIdx.x + i * blockDim.x;
    v[i] = e < n ? y[base + e] : 0.f;
    rv[i] = (residual && e < n) ? residual[base + e] : 0.f;
  }
  asm volatile("" ::: "memory");  // every load above is issued before any result is consumed
  double s1 = 0.0, s2 = 0.0;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    s1 += v[i];
    s2 += (double)v[i] * v[i];
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
  const float mu = smu[c / cg], rs = srs[c / cg];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int e = threadIdx.x + i * blockDim.x;
    if (e >= n) break;
    const size_t idx = base + e;
    float o = (v[i] - mu) * rs * gm + bt;
    if (residual) o += rv[i];
    o = relu ? fmaxf(o, 0.f) : o;
    z[idx] = o;
    if (zb) {  // bf16 hi / lo planes: the next convolution's operand
      const __nv_bfloat16 hi = __float2bfloat16_rn(o);
      zb[idx] = hi;
      zb[plane + idx] = __float2bfloat16_rn(o - __bfloat162float(hi));
    }
  }
}

// Backward staging: elements [e0, e1) of the block's slab of dz, z (ReLU mask, nullable) and y go
// HBM -> shared memory with 16-byte cp.async (zero-filled past e1), every copy in flight at once and
// no register waiting on a load (register-cached loads let the compiler consume the mask early,
// which serialised the loads); thread t then reads its elements t + i*blockDim from shared memory.
__device__ __forceinline__ void gn_cp16(float* dst, const float* src, bool ok) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(ok ? 16u : 0u) : "memory");
}
__device__ __forceinline__ void gn_stage_bwd(float* s_dz, float* s_z, float* s_y, const float* __restrict__ dz,
                                             const float* __restrict__ z, const float* __restrict__ y, size_t base,
                                             int e0, int e1, int cap) {
  for (int j = threadIdx.x; j < cap / 4; j += blockDim.x) {
    const int e = e0 + 4 * j;
    const bool ok = e < e1;
    const size_t o = ok ? base + e : 0;
    gn_cp16(s_dz + 4 * j, dz + o, ok);
    if (z) gn_cp16(s_z + 4 * j, z + o, ok);
    gn_cp16(s_y + 4 * j, y + o, ok);
  }
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
  __syncthreads();
}
__host__ __device__ constexpr size_t gn_bwd_smem(int nv, int nt) { return (size_t)3 * nv * nt * sizeof(float); }

// the GN input gradient as bf16 (lo == 0), or as hi / lo planes (x = hi + lo; lo plane at +lo elements)
// for the deep encoder's input-gradient chain
__device__ __forceinline__ void put_grad(__nv_bfloat16* dx, size_t lo, size_t i, float v) {
  const __nv_bfloat16 h = __float2bfloat16_rn(v);
  dx[i] = h;
  if (lo) dx[lo + i] = __float2bfloat16_rn(v - __bfloat162float(h));
}

// dy_eff = dz * [z > 0] (relu_z nullable): GN backward per group
//   dx = rstd * (dxhat - mean(dxhat) - xhat * mean(dxhat * xhat)),   dxhat = dy_eff * gamma
// written as bf16 (it only feeds the bf16 gradient GEMMs), plus this frame's per-channel partials
// part[f][c] = (sum dy_eff * xhat, sum dy_eff) for dgamma / dbeta.  One block per frame; the slab is
// read from HBM once (shared-memory staged).
template <int NV>
__global__ void __launch_bounds__(gn_bound(NV)) gn_bwd_kernel(const float* __restrict__ dz, const float* __restrict__ z,
                                                            const float* __restrict__ y,
                                                            const float* __restrict__ stats,
                                                            const float* __restrict__ gamma, int HW, int C,
                                                            __nv_bfloat16* __restrict__ dx, float* __restrict__ part,
                                                            size_t lo) {
  pdl_enter();
  __shared__ double sa[gn_bound(NV)], sb[gn_bound(NV)], ga[kGroups], gb[kGroups];
  __shared__ float pc[2][gn_bound(NV)];
  extern __shared__ __align__(16) float gsm[];
  const int cap = NV * blockDim.x;
  float *s_dz = gsm, *s_z = gsm + cap, *s_y = gsm + 2 * cap;
  const int f = blockIdx.x, n = HW * C, c = threadIdx.x % C, cg = C / kGroups, g = c / cg;
  const size_t base = (size_t)f * n;
  // (the statistics / gamma loads are issued before the staging wait, not after it)
  const float mu = stats[(f * kGroups + g) * 2], rs = stats[(f * kGroups + g) * 2 + 1], gm = gamma[c];
  gn_stage_bwd(s_dz, s_z, s_y, dz, z, y, base, 0, n, cap);
  double a1 = 0.0, a2 = 0.0;
  float pg = 0.f, pb = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int e = threadIdx.x + i * blockDim.x;
    if (e >= n) break;
    float d = s_dz[e];
    if (z && s_z[e] <= 0.f) d = 0.f;
    const float xh = (s_y[e] - mu) * rs, dxh = d * gm;
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
    for (int t = threadIdx.x; t < (int)blockDim.x; t += C) {
      rg += pc[0][t];
      rb += pc[1][t];
    }
    part[((size_t)f * C + threadIdx.x) * 2] = rg;
    part[((size_t)f * C + threadIdx.x) * 2 + 1] = rb;
  }
  const double cnt = (double)HW * cg;
  const float m1 = (float)(ga[g] / cnt), m2 = (float)(gb[g] / cnt);
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int e = threadIdx.x + i * blockDim.x;
    if (e >= n) break;
    float d = s_dz[e];
    if (z && s_z[e] <= 0.f) d = 0.f;
    const float xh = (s_y[e] - mu) * rs;
    put_grad(dx, lo, base + e, rs * (d * gm - m1 - xh * m2));
  }
}

// Large frames: the [HW][C] slab of a frame is split into S chunks of gn_chunk(C) elements, one
// block each (grid (S, F)).  Pass 1 writes per-chunk per-group partial sums (double), pass 2 reduces
// the frame's S partials in chunk order, then normalises / back-propagates its chunk.

template <int NV>
__global__ void __launch_bounds__(gn_bound(NV)) gn_stats_part_kernel(const float* __restrict__ y, int HW, int C,
                                                                      double* __restrict__ gpart) {
  pdl_enter();
  __shared__ double sa[gn_bound(NV)], sb[gn_bound(NV)], ga[kGroups], gb[kGroups];
  const int f = blockIdx.y, S = gridDim.x, n = HW * C, chunk = gn_chunk(C);
  const int e0 = blockIdx.x * chunk, e1 = min(n, e0 + chunk);
  const size_t base = (size_t)f * n;
  float v[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) {  // all loads in flight
    const int e = e0 + threadIdx.x + i * blockDim.x;
    v[i] = e < e1 ? y[base + e] : 0.f;
  }
  asm volatile("" ::: "memory");  // every load above is issued before any result is consumed
  double s1 = 0.0, s2 = 0.0;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    s1 += v[i];
    s2 += (double)v[i] * v[i];
  }
  gn_group_reduce(s1, s2, C, sa, sb, ga, gb);
  if (threadIdx.x < kGroups) {
    double* o = gpart + (((size_t)f * S + blockIdx.x) * kGroups + threadIdx.x) * 2;
    o[0] = ga[threadIdx.x];
    o[1] = gb[threadIdx.x];
  }
}

template <int NV>
__global__ void __launch_bounds__(gn_bound(NV)) gn_apply_part_kernel(const float* __restrict__ y,
                                                                      const double* __restrict__ gpart,
                                                                      const float* __restrict__ gamma,
                                                                      const float* __restrict__ beta,
                                                                      const float* __restrict__ residual, int HW,
                                                                      int C, int relu, size_t plane,
                                                                      float* __restrict__ stats, float* __restrict__ z,
                                                                      __nv_bfloat16* __restrict__ zb, int nparts) {
  pdl_enter();
  __shared__ float smu[kGroups], srs[kGroups];
  // gpart holds nparts partial sums per frame (gn_stats_part: one per chunk; the stem kernel: 1)
  const int f = blockIdx.y, S = nparts, n = HW * C, chunk = gn_chunk(C), cg = C / kGroups;
  const int e0 = blockIdx.x * chunk, e1 = min(n, e0 + chunk);
  const size_t base = (size_t)f * n;
  const int c = threadIdx.x % C;
  const float gm = gamma[c], bt = beta[c];
  float v[NV], rv[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) {  // the chunk's loads first: in flight while the statistics are formed
    const int e = e0 + threadIdx.x + i * blockDim.x;
    v[i] = e < e1 ? y[base + e] : 0.f;
    rv[i] = (residual && e < e1) ? residual[base + e] : 0.f;
  }
  if (threadIdx.x < kGroups) {
    double a = 0.0, b = 0.0;
    for (int s = 0; s < S; ++s) {
      const double* o = gpart + (((size_t)f * S + s) * kGroups + threadIdx.x) * 2;
      a += o[0];
      b += o[1];
    }
    const double cnt = (double)HW * cg, mu = a / cnt;
    double var = b / cnt - mu * mu;
    if (var < 0) var = 0;
    smu[threadIdx.x] = (float)mu;
    srs[threadIdx.x] = (float)(1.0 / sqrt(var + 1e-5));
    if (blockIdx.x == 0) {
      stats[(f * kGroups + threadIdx.x) * 2] = smu[threadIdx.x];
      stats[(f * kGroups + threadIdx.x) * 2 + 1] = srs[threadIdx.x];
    }
  }
  __syncthreads();
  const float mu = smu[c / cg], rs = srs[c / cg];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int e = e0 + threadIdx.x + i * blockDim.x;
    if (e >= e1) break;
    const size_t idx = base + e;
    float o = (v[i] - mu) * rs * gm + bt;
    if (residual) o += rv[i];
    o = relu ? fmaxf(o, 0.f) : o;
    z[idx] = o;
    if (zb) {
      const __nv_bfloat16 hi = __float2bfloat16_rn(o);
      zb[idx] = hi;
      zb[plane + idx] = __float2bfloat16_rn(o - __bfloat162float(hi));
    }
  }
}

// backward pass 1: per chunk, per group (sum dxhat, sum dxhat*xhat) and per channel (sum dy*xhat, sum dy)
template <int NV>
__global__ void __launch_bounds__(gn_bound(NV)) gn_bwd_part_kernel(const float* __restrict__ dz,
                                                                  const float* __restrict__ z,
                                                                  const float* __restrict__ y,
                                                                  const float* __restrict__ stats,
                                                                  const float* __restrict__ gamma, int HW, int C,
                                                                  double* __restrict__ gpart,
                                                                  float* __restrict__ part) {
  pdl_enter();
  __shared__ double sa[gn_bound(NV)], sb[gn_bound(NV)], ga[kGroups], gb[kGroups];
  __shared__ float pc[2][gn_bound(NV)];
  extern __shared__ __align__(16) float gsm[];
  const int cap = NV * blockDim.x;
  float *s_dz = gsm, *s_z = gsm + cap, *s_y = gsm + 2 * cap;
  const int f = blockIdx.y, S = gridDim.x, n = HW * C, chunk = gn_chunk(C), c = threadIdx.x % C, cg = C / kGroups,
            g = c / cg;
  const int e0 = blockIdx.x * chunk, e1 = min(n, e0 + chunk);
  const size_t base = (size_t)f * n;
  // (the statistics / gamma loads are issued before the staging wait, not after it)
  const float mu = stats[(f * kGroups + g) * 2], rs = stats[(f * kGroups + g) * 2 + 1], gm = gamma[c];
  gn_stage_bwd(s_dz, s_z, s_y, dz, z, y, base, e0, e1, cap);
  double a1 = 0.0, a2 = 0.0;
  float pg = 0.f, pb = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int e = threadIdx.x + i * blockDim.x;
    if (e0 + e >= e1) break;
    float d = s_dz[e];
    if (z && s_z[e] <= 0.f) d = 0.f;
    const float xh = (s_y[e] - mu) * rs, dxh = d * gm;
    a1 += dxh;
    a2 += (double)dxh * xh;
    pg += d * xh;
    pb += d;
  }
  pc[0][threadIdx.x] = pg;
  pc[1][threadIdx.x] = pb;
  gn_group_reduce(a1, a2, C, sa, sb, ga, gb);
  if (threadIdx.x < kGroups) {
    double* o = gpart + (((size_t)f * S + blockIdx.x) * kGroups + threadIdx.x) * 2;
    o[0] = ga[threadIdx.x];
    o[1] = gb[threadIdx.x];
  }
  if (threadIdx.x < C) {
    float rg = 0.f, rb = 0.f;
    for (int t = threadIdx.x; t < (int)blockDim.x; t += C) {
      rg += pc[0][t];
      rb += pc[1][t];
    }
    const size_t row = (size_t)f * S + blockIdx.x;  // rows of the dgamma / dbeta reduction
    part[(row * C + threadIdx.x) * 2] = rg;
    part[(row * C + threadIdx.x) * 2 + 1] = rb;
  }
}

template <int NV>
__global__ void __launch_bounds__(gn_bound(NV)) gn_bwd_apply_kernel(const float* __restrict__ dz,
                                                                   const float* __restrict__ z,
                                                                   const float* __restrict__ y,
                                                                   const float* __restrict__ stats,
                                                                   const float* __restrict__ gamma,
                                                                   const double* __restrict__ gpart, int HW, int C,
                                                                   __nv_bfloat16* __restrict__ dx, size_t lo) {
  pdl_enter();
  __shared__ float sm1[kGroups], sm2[kGroups];
  extern __shared__ __align__(16) float gsm[];
  const int cap = NV * blockDim.x;
  float *s_dz = gsm, *s_z = gsm + cap, *s_y = gsm + 2 * cap;
  const int f = blockIdx.y, S = gridDim.x, n = HW * C, chunk = gn_chunk(C), cg = C / kGroups;
  const int e0 = blockIdx.x * chunk, e1 = min(n, e0 + chunk);
  const size_t base = (size_t)f * n;
  // the copies fly while the 16 group sums are reduced
  for (int j = threadIdx.x; j < cap / 4; j += blockDim.x) {
    const int e = e0 + 4 * j;
    const bool ok = e < e1;
    const size_t o = ok ? base + e : 0;
    gn_cp16(s_dz + 4 * j, dz + o, ok);
    if (z) gn_cp16(s_z + 4 * j, z + o, ok);
    gn_cp16(s_y + 4 * j, y + o, ok);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  if (threadIdx.x < kGroups) {
    double a = 0.0, b = 0.0;
    for (int s = 0; s < S; ++s) {
      const double* o = gpart + (((size_t)f * S + s) * kGroups + threadIdx.x) * 2;
      a += o[0];
      b += o[1];
    }
    const double cnt = (double)HW * cg;
    sm1[threadIdx.x] = (float)(a / cnt);
    sm2[threadIdx.x] = (float)(b / cnt);
  }
  const int c = threadIdx.x % C, g = c / cg;
  const float mu = stats[(f * kGroups + g) * 2], rs = stats[(f * kGroups + g) * 2 + 1], gm = gamma[c];
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  const float m1 = sm1[g], m2 = sm2[g];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int e = threadIdx.x + i * blockDim.x;
    if (e0 + e >= e1) break;
    float d = s_dz[e];
    if (z && s_z[e] <= 0.f) d = 0.f;
    const float xh = (s_y[e] - mu) * rs;
    put_grad(dx, lo, base + e0 + e, rs * (d * gm - m1 - xh * m2));
  }
}

// Large frames, one pass: the S chunks of a frame form a thread-block cluster (S <= 16).  Each CTA
// stages its chunk (cp.async), computes its per-group sums and per-channel dgamma / dbeta rows, the
// cluster barrier publishes the group sums, every CTA adds the S of them in CTA order through DSMEM
// (the same order and arithmetic as gn_bwd_apply_kernel's loop over the chunk partials) and writes
// dx from the staged chunk: dz / z / y are read from HBM once instead of twice.
template <int NV>
__global__ void __launch_bounds__(gn_bound(NV)) gn_bwd_cluster_kernel(const float* __restrict__ dz,
                                                                     const float* __restrict__ z,
                                                                     const float* __restrict__ y,
                                                                     const float* __restrict__ stats,
                                                                     const float* __restrict__ gamma, int HW, int C,
                                                                     float* __restrict__ part,
                                                                     __nv_bfloat16* __restrict__ dx, size_t lo) {
  __shared__ double sa[gn_bound(NV)], sb[gn_bound(NV)], ga[kGroups], gb[kGroups];
  __shared__ float pc[2][gn_bound(NV)];
  __shared__ float sm1[kGroups], sm2[kGroups];
  extern __shared__ __align__(16) float gsm[];
  const int cap = NV * blockDim.x;
  float *s_dz = gsm, *s_z = gsm + cap, *s_y = gsm + 2 * cap;
  const int f = blockIdx.y, S = gridDim.x, n = HW * C, chunk = gn_chunk(C), c = threadIdx.x % C, cg = C / kGroups,
            g = c / cg;
  const int e0 = blockIdx.x * chunk, e1 = min(n, e0 + chunk);
  const size_t base = (size_t)f * n;
  // (the statistics / gamma loads are issued before the staging wait, not after it)
  const float mu = stats[(f * kGroups + g) * 2], rs = stats[(f * kGroups + g) * 2 + 1], gm = gamma[c];
  gn_stage_bwd(s_dz, s_z, s_y, dz, z, y, base, e0, e1, cap);
  double a1 = 0.0, a2 = 0.0;
  float pg = 0.f, pb = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int e = threadIdx.x + i * blockDim.x;
    if (e0 + e >= e1) break;
    float d = s_dz[e];
    if (z && s_z[e] <= 0.f) d = 0.f;
    const float xh = (s_y[e] - mu) * rs, dxh = d * gm;
    a1 += dxh;
    a2 += (double)dxh * xh;
    pg += d * xh;
    pb += d;
  }
  pc[0][threadIdx.x] = pg;
  pc[1][threadIdx.x] = pb;
  gn_group_reduce(a1, a2, C, sa, sb, ga, gb);  // ga / gb: this chunk's group sums (its barriers publish pc)
  if (threadIdx.x < C) {
    float rg = 0.f, rb = 0.f;
    for (int t = threadIdx.x; t < (int)blockDim.x; t += C) {
      rg += pc[0][t];
      rb += pc[1][t];
    }
    const size_t row = (size_t)f * S + blockIdx.x;  // rows of the dgamma / dbeta reduction
    part[(row * C + threadIdx.x) * 2] = rg;
    part[(row * C + threadIdx.x) * 2 + 1] = rb;
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  if (threadIdx.x < kGroups) {
    double a = 0.0, b = 0.0;
    const uint32_t la = (uint32_t)__cvta_generic_to_shared(&ga[threadIdx.x]),
                   lb = (uint32_t)__cvta_generic_to_shared(&gb[threadIdx.x]);
    for (int r = 0; r < S; ++r) {
      uint32_t ra, rb2;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(r));
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb2) : "r"(lb), "r"(r));
      double va, vb;
      asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(va) : "r"(ra) : "memory");
      asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(vb) : "r"(rb2) : "memory");
      a += va;
      b += vb;
    }
    const double cnt = (double)HW * cg;
    sm1[threadIdx.x] = (float)(a / cnt);
    sm2[threadIdx.x] = (float)(b / cnt);
  }
  // every CTA has read every peer's group sums before any CTA leaves (or rewrites ga / gb)
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  const float m1 = sm1[g], m2 = sm2[g];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int e = threadIdx.x + i * blockDim.x;
    if (e0 + e >= e1) break;
    float d = s_dz[e];
    if (z && s_z[e] <= 0.f) d = 0.f;
    const float xh = (s_y[e] - mu) * rs;
    put_grad(dx, lo, base + e0 + e, rs * (d * gm - m1 - xh * m2));
  }
}

// dgamma[c], dbeta[c] = sums over frames (in frame order, blocked: thread t takes frames t, t+256,
// ...; then the fixed-order block reduction) of the per-frame partials
__global__ void __launch_bounds__(kThreads) gn_param_reduce_kernel(const float* __restrict__ part, int F, int C,
                                                                   float* __restrict__ dgamma,
                                                                   float* __restrict__ dbeta) {
  pdl_enter();
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

// every GroupNorm layer's dgamma / dbeta of one backward pass in one launch (ch_off[i] = first block
// of layer i)
struct GnParamAll {
  int n;
  int ch_off[kMaxConvsGn + 1];
  struct Item {
    const float* part;
    float *dgamma, *dbeta;
    int rows, C;
  } it[kMaxConvsGn];
};
// block = 32 consecutive channels of one layer (ch_off: first block of each layer), 1024 threads =
// 32 channels x 32 row lanes: a warp reads one row's 32 channel pairs (256 contiguous bytes), lane
// row rl sums rows rl, rl + 32, ... in order, then the 32 row lanes are added in order (fixed,
// deterministic).  (A block per channel read 8 of every 32 bytes it fetched: 21 us per backward.)
constexpr int kGnRedThreads = 1024;
__global__ void __launch_bounds__(kGnRedThreads) gn_param_reduce_all_kernel(const GnParamAll a) {
  pdl_enter();
  __shared__ double red[32][33][2];
  int lo = 0, hi = a.n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (a.ch_off[mid] <= (int)blockIdx.x) lo = mid;
    else hi = mid - 1;
  }
  const GnParamAll::Item& t = a.it[lo];
  const int cl = threadIdx.x & 31, rl = threadIdx.x >> 5, c = 32 * (blockIdx.x - a.ch_off[lo]) + cl;
  double acc0 = 0.0, acc1 = 0.0;
  if (c < t.C) {
    const float2* p = reinterpret_cast<const float2*>(t.part) + c;
    int f = rl;
    for (; f + 3 * 32 < t.rows; f += 4 * 32) {  // 4 rows in flight
      const float2 v0 = p[(size_t)f * t.C], v1 = p[(size_t)(f + 32) * t.C];
      const float2 v2 = p[(size_t)(f + 64) * t.C], v3 = p[(size_t)(f + 96) * t.C];
      acc0 += v0.x; acc1 += v0.y;
      acc0 += v1.x; acc1 += v1.y;
      acc0 += v2.x; acc1 += v2.y;
      acc0 += v3.x; acc1 += v3.y;
    }
    for (; f < t.rows; f += 32) {
      const float2 v = p[(size_t)f * t.C];
      acc0 += v.x;
      acc1 += v.y;
    }
  }
  red[rl][cl][0] = acc0;
  red[rl][cl][1] = acc1;
  __syncthreads();
  if (rl == 0 && c < t.C) {
    double s0 = 0.0, s1 = 0.0;
    for (int r = 0; r < 32; ++r) {
      s0 += red[r][cl][0];
      s1 += red[r][cl][1];
    }
    t.dgamma[c] = (float)s0;
    t.dbeta[c] = (float)s1;
  }
}

// 3x3 / stride 2 / pad 1 max pool with the first maximum in (u, v) order.  Thread = (output pixel,
// 4 channels): the 9 window loads (float4) are independent and in flight together; 32-bit indices.
__global__ void maxpool_fwd_kernel(const float* __restrict__ x, int F, int H, int W, int C, int Ho, int Wo,
                                   float* __restrict__ y, uint8_t* __restrict__ arg, __nv_bfloat16* __restrict__ yb) {
  pdl_enter();
  const int C4 = C >> 2, n4 = F * Ho * Wo * C4;
  const int i4 = blockIdx.x * blockDim.x + threadIdx.x;
  if (i4 >= n4) return;
  const int c4 = i4 % C4, pix = i4 / C4;
  const int j = pix % Wo, ii = (pix / Wo) % Ho, f = pix / (Wo * Ho);
  float4 w[9];
#pragma unroll
  for (int t = 0; t < 9; ++t) {
    const int yy = 2 * ii - 1 + t / 3, xx = 2 * j - 1 + t % 3;
    w[t] = (yy >= 0 && yy < H && xx >= 0 && xx < W)
               ? *reinterpret_cast<const float4*>(x + ((f * H + yy) * W + xx) * C + 4 * c4)
               : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
  }
  float best[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
  int ba[4] = {0, 0, 0, 0};
#pragma unroll
  for (int t = 0; t < 9; ++t) {
    const float v[4] = {w[t].x, w[t].y, w[t].z, w[t].w};
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (v[e] > best[e]) {
        best[e] = v[e];
        ba[e] = t;
      }
  }
  const int o = pix * C + 4 * c4;
  *reinterpret_cast<float4*>(y + o) = make_float4(best[0], best[1], best[2], best[3]);
  *reinterpret_cast<uchar4*>(arg + o) = make_uchar4((uint8_t)ba[0], (uint8_t)ba[1], (uint8_t)ba[2], (uint8_t)ba[3]);
  if (yb) {
    __nv_bfloat16 hi[4], lo[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      hi[e] = __float2bfloat16_rn(best[e]);
      lo[e] = __float2bfloat16_rn(best[e] - __bfloat162float(hi[e]));
    }
    const size_t n = (size_t)F * Ho * Wo * C;
    *reinterpret_cast<uint2*>(yb + o) = *reinterpret_cast<const uint2*>(hi);
    *reinterpret_cast<uint2*>(yb + n + o) = *reinterpret_cast<const uint2*>(lo);
  }
}
// dx[f][y][x][c] = sum over windows whose argmax is (y, x) of dy (gather, fixed window order).
// Thread = (input pixel, 4 channels) of one frame (grid.y).
__global__ void maxpool_bwd_kernel(const float* __restrict__ dy, const uint8_t* __restrict__ arg, int F, int H, int W,
                                   int C, int Ho, int Wo, float* __restrict__ dx) {
  pdl_enter();
  // grid (pixels x channel quads of one frame, F): no division by runtime frame sizes for the frame
  const int C4 = C >> 2, f = blockIdx.y;
  const int i4 = blockIdx.x * blockDim.x + threadIdx.x;
  if (i4 >= H * W * C4) return;
  const int c4 = i4 % C4, pix = i4 / C4;
  const int xx = pix % W, yq = pix / W;
  // windows (ii, jj) with 2*ii - 1 + u = y, u in [0, 3): even y one window (u = 1), odd y two
  // (u = 0, 2); the same for x / v.  q = 0..3 enumerates them with (u, v) ascending, so summing in
  // q order is the reference order (windows by (u, v) ascending).
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int u = (yq & 1) ? 2 * (q >> 1) : 1, v = (xx & 1) ? 2 * (q & 1) : 1;
    const int yy = yq + 1 - u, xv = xx + 1 - v;
    const int ii = yy >> 1, jj = xv >> 1;
    const bool dup = (!(yq & 1) && (q >> 1)) || (!(xx & 1) && (q & 1));
    if (dup || yy < 0 || xv < 0 || ii >= Ho || jj >= Wo) continue;
    const int o = ((f * Ho + ii) * Wo + jj) * C + 4 * c4, uv = u * 3 + v;
    const uchar4 a = *reinterpret_cast<const uchar4*>(arg + o);
    const float4 d = *reinterpret_cast<const float4*>(dy + o);
    if (a.x == uv) acc[0] += d.x;
    if (a.y == uv) acc[1] += d.y;
    if (a.z == uv) acc[2] += d.z;
    if (a.w == uv) acc[3] += d.w;
  }
  *reinterpret_cast<float4*>(dx + ((size_t)f * H * W + pix) * C + 4 * c4) = make_float4(acc[0], acc[1], acc[2], acc[3]);
}

// The same for even H = 2 Hp, W = 2 Wp, thread = (2x2 pixel block (2a.., 2b..), 4 channels): the
// block's candidate windows are (a | a+1) x (b | b+1), each (argmax, gradient) pair loaded once for
// the 4 pixels (the per-pixel kernel loads 2.25 pairs per pixel); every pixel adds its windows in
// the same (u, v) order as maxpool_bwd_kernel, so the result is bit-identical.
__global__ void maxpool_bwd2_kernel(const float* __restrict__ dy, const uint8_t* __restrict__ arg, int Hp, int Wp,
                                    int C, float* __restrict__ dx) {
  pdl_enter();
  const int C4 = C >> 2, f = blockIdx.y;
  const int i4 = blockIdx.x * blockDim.x + threadIdx.x;
  if (i4 >= Hp * Wp * C4) return;
  const int c4 = i4 % C4, blk = i4 / C4, b = blk % Wp, a = blk / Wp;
  uchar4 wa[2][2];
  float4 wd[2][2];
#pragma unroll
  for (int da = 0; da < 2; ++da)
#pragma unroll
    for (int db = 0; db < 2; ++db) {
      const bool ok = a + da < Hp && b + db < Wp;
      const size_t o = ok ? (((size_t)f * Hp + a + da) * Wp + b + db) * C + 4 * c4 : 0;
      wa[da][db] = ok ? *reinterpret_cast<const uchar4*>(arg + o) : make_uchar4(255, 255, 255, 255);
      wd[da][db] = ok ? *reinterpret_cast<const float4*>(dy + o) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  auto add = [](float (&acc)[4], const uchar4 a4, const float4 d4, int uv) {
    if (a4.x == uv) acc[0] += d4.x;
    if (a4.y == uv) acc[1] += d4.y;
    if (a4.z == uv) acc[2] += d4.z;
    if (a4.w == uv) acc[3] += d4.w;
  };
  // pixel (2a + r, 2b + s): windows in (u, v) ascending order; uv = u * 3 + v
  float p00[4] = {0.f, 0.f, 0.f, 0.f}, p01[4] = {0.f, 0.f, 0.f, 0.f}, p10[4] = {0.f, 0.f, 0.f, 0.f},
        p11[4] = {0.f, 0.f, 0.f, 0.f};
  add(p00, wa[0][0], wd[0][0], 4);  // (u 1, v 1)
  add(p01, wa[0][1], wd[0][1], 3);  // (1, 0) window b + 1
  add(p01, wa[0][0], wd[0][0], 5);  // (1, 2) window b
  add(p10, wa[1][0], wd[1][0], 1);  // (0, 1) window a + 1
  add(p10, wa[0][0], wd[0][0], 7);  // (2, 1) window a
  add(p11, wa[1][1], wd[1][1], 0);  // (0, 0)
  add(p11, wa[1][0], wd[1][0], 2);  // (0, 2)
  add(p11, wa[0][1], wd[0][1], 6);  // (2, 0)
  add(p11, wa[0][0], wd[0][0], 8);  // (2, 2)
  const int W = 2 * Wp;
  float* o0 = dx + (((size_t)f * 2 * Hp + 2 * a) * W + 2 * b) * C + 4 * c4;
  float* o1 = o0 + (size_t)W * C;
  *reinterpret_cast<float4*>(o0) = make_float4(p00[0], p00[1], p00[2], p00[3]);
  *reinterpret_cast<float4*>(o0 + C) = make_float4(p01[0], p01[1], p01[2], p01[3]);
  *reinterpret_cast<float4*>(o1) = make_float4(p10[0], p10[1], p10[2], p10[3]);
  *reinterpret_cast<float4*>(o1 + C) = make_float4(p11[0], p11[1], p11[2], p11[3]);
}

// NHWC [F][HW][C] <-> flat [F][C*HW] in (c, h, w) order (PyTorch flatten of NCHW)
__global__ void flatten_kernel(const float* __restrict__ in, int F, int HW, int C, float* __restrict__ out,
                               int to_flat) {
  pdl_enter();
  const int per = HW * C;
  const size_t n = (size_t)F * per;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int f = (int)(i / per), q = (int)(i % per);
    const int c = q / HW, hw = q % HW;
    const size_t nhwc = (size_t)f * per + hw * C + c;
    if (to_flat) out[i] = in[nhwc];
    else out[nhwc] = in[i];
  }
}

// y[m][n] = act(y[m][n] + bias[n])   (act: 1 = ReLU)
__global__ void bias_act_kernel(float* __restrict__ y, const float* __restrict__ bias, int M, int N, int relu) {
  pdl_enter();
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
  pdl_enter();
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
  pdl_enter();
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
  pdl_enter();
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

// dgoal[s][c] = sum_j dx[s][512 + j] * Wg[j][c]: the gradient wrt the goal input of goal_fc
__global__ void goal_input_grad_kernel(const float* __restrict__ dx, const float* __restrict__ Wg, int S,
                                       float* __restrict__ dgoal) {
  pdl_enter();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < S * 3; i += gridDim.x * blockDim.x) {
    const int s = i / 3, c = i - s * 3;
    float acc = 0.f;
    for (int j = 0; j < 32; ++j) acc += dx[(size_t)s * kXin + 512 + j] * Wg[j * 3 + c];
    dgoal[i] = acc;
  }
}

__global__ void relu_mask_kernel(const float* __restrict__ dz, const float* __restrict__ z, size_t n,
                                 float* __restrict__ out) {
  pdl_enter();
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    out[i] = z[i] > 0.f ? dz[i] : 0.f;
}


// ------------------------------------------------------------------ squeeze-excitation (SE-ResNeXt, R9)
// One block per frame.  z3 = GN3 output [F][HW][C] (NHWC), sc = shortcut; out = relu(z3 * s + sc) and
// its bf16 hi / lo planes (plane = F*HW*C); s = sigmoid(W2 relu(W1 pool + b1) + b2), pool = mean_hw z3.
// Sums in fixed order (thread per channel over pixels; warp per fc1 unit over channels).
__global__ void __launch_bounds__(256) se_fwd_kernel(const float* __restrict__ z3, const float* __restrict__ sc,
                                                     const float* __restrict__ W1, const float* __restrict__ b1,
                                                     const float* __restrict__ W2, const float* __restrict__ b2, int HW,
                                                     int C, int R, float* __restrict__ out,
                                                     __nv_bfloat16* __restrict__ outb, size_t plane,
                                                     float* __restrict__ s_out, float* __restrict__ pool_out,
                                                     float* __restrict__ a1_out) {
  pdl_enter();
  extern __shared__ float sm[];  // pool[C], s[C], a1[R]
  float *pool = sm, *sv = sm + C, *a1 = sm + 2 * C;
  const int f = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const size_t base = (size_t)f * HW * C;
  for (int c = tid; c < C; c += blockDim.x) {
    float acc = 0.f;
    for (int q = 0; q < HW; ++q) acc += z3[base + (size_t)q * C + c];
    pool[c] = acc / (float)HW;
    pool_out[(size_t)f * C + c] = pool[c];
  }
  __syncthreads();
  for (int j = warp; j < R; j += blockDim.x / 32) {
    float acc = 0.f;
    for (int c = lane; c < C; c += 32) acc += W1[(size_t)j * C + c] * pool[c];
    acc = warp_sum(acc);
    if (lane == 0) {
      a1[j] = acc + b1[j];
      a1_out[(size_t)f * R + j] = a1[j];
    }
  }
  __syncthreads();
  for (int c = tid; c < C; c += blockDim.x) {
    float t = b2[c];
    for (int j = 0; j < R; ++j) t += W2[(size_t)c * R + j] * fmaxf(a1[j], 0.f);
    sv[c] = 1.f / (1.f + expf(-t));
    s_out[(size_t)f * C + c] = sv[c];
  }
  __syncthreads();
  for (size_t i = tid; i < (size_t)HW * C; i += blockDim.x) {
    const int c = (int)(i & (size_t)(C - 1));
    const float v = fmaxf(z3[base + i] * sv[c] + sc[base + i], 0.f);
    out[base + i] = v;
    const __nv_bfloat16 h = __float2bfloat16_rn(v);
    outb[base + i] = h;
    outb[plane + base + i] = __float2bfloat16_rn(v - __bfloat162float(h));
  }
}

// d = dz * [out > 0] (the block output's ReLU); ds = sum_hw d z3; da2 = ds s (1 - s); da1 = (W2^T da2) [a1 > 0];
// dz3 = d s + (W1^T da1) / HW.  Per-frame da1 / da2 feed se_param_grad_kernel.
__global__ void __launch_bounds__(256) se_bwd_kernel(const float* __restrict__ dz, const float* __restrict__ out,
                                                     const float* __restrict__ z3, const float* __restrict__ s_in,
                                                     const float* __restrict__ a1_in, const float* __restrict__ W1,
                                                     const float* __restrict__ W2, int HW, int C, int R,
                                                     float* __restrict__ dz3, float* __restrict__ da1_out,
                                                     float* __restrict__ da2_out) {
  pdl_enter();
  extern __shared__ float sm[];  // da2[C], dpool[C], da1[R]
  float *da2 = sm, *dpool = sm + C, *da1 = sm + 2 * C;
  const int f = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const size_t base = (size_t)f * HW * C;
  for (int c = tid; c < C; c += blockDim.x) {
    float acc = 0.f;
    for (int q = 0; q < HW; ++q) {
      const size_t i = base + (size_t)q * C + c;
      if (out[i] > 0.f) acc += dz[i] * z3[i];
    }
    const float sv = s_in[(size_t)f * C + c];
    da2[c] = acc * sv * (1.f - sv);
    da2_out[(size_t)f * C + c] = da2[c];
  }
  __syncthreads();
  for (int j = warp; j < R; j += blockDim.x / 32) {
    float acc = 0.f;
    for (int c = lane; c < C; c += 32) acc += W2[(size_t)c * R + j] * da2[c];
    acc = warp_sum(acc);
    if (lane == 0) {
      da1[j] = a1_in[(size_t)f * R + j] > 0.f ? acc : 0.f;
      da1_out[(size_t)f * R + j] = da1[j];
    }
  }
  __syncthreads();
  for (int c = tid; c < C; c += blockDim.x) {
    float acc = 0.f;
    for (int j = 0; j < R; ++j) acc += W1[(size_t)j * C + c] * da1[j];
    dpool[c] = acc / (float)HW;
  }
  __syncthreads();
  for (size_t i = tid; i < (size_t)HW * C; i += blockDim.x) {
    const int c = (int)(i & (size_t)(C - 1));
    const float d = out[base + i] > 0.f ? dz[base + i] : 0.f;
    dz3[base + i] = d * s_in[(size_t)f * C + c] + dpool[c];
  }
}

// dW1[j][c] = sum_f da1[f][j] pool[f][c]; db1[j] = sum_f da1[f][j]; dW2[c][j] = sum_f da2[f][c] relu(a1[f][j]);
// db2[c] = sum_f da2[f][c]  (one thread per output, frames in order)
__global__ void se_param_grad_kernel(const float* __restrict__ da1, const float* __restrict__ da2,
                                     const float* __restrict__ pool, const float* __restrict__ a1, int F, int C, int R,
                                     float* __restrict__ dW1, float* __restrict__ db1, float* __restrict__ dW2,
                                     float* __restrict__ db2) {
  pdl_enter();
  const int n1 = R * C, n = 2 * R * C + R + C;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    float acc = 0.f;
    if (i < n1) {
      const int j = i / C, c = i - j * C;
      for (int f = 0; f < F; ++f) acc += da1[(size_t)f * R + j] * pool[(size_t)f * C + c];
      dW1[i] = acc;
    } else if (i < 2 * n1) {
      const int k = i - n1, c = k / R, j = k - c * R;
      for (int f = 0; f < F; ++f) acc += da2[(size_t)f * C + c] * fmaxf(a1[(size_t)f * R + j], 0.f);
      dW2[k] = acc;
    } else if (i < 2 * n1 + R) {
      const int j = i - 2 * n1;
      for (int f = 0; f < F; ++f) acc += da1[(size_t)f * R + j];
      db1[j] = acc;
    } else {
      const int c = i - 2 * n1 - R;
      for (int f = 0; f < F; ++f) acc += da2[(size_t)f * C + c];
      db2[c] = acc;
    }
  }
}

// ------------------------------------------------------------------ network plan
struct ConvGN {
  int Ci, Co, k, s, p, H, W, Ho, Wo;  // GEMM geometry: input H x W x Ci (Ci padded to 8 for the RGB-D stem)
  int Ci_real;                        // channels of the parameter tensor
  int64_t w, gw, gb;                  // parameter offsets (conv weight, GN gamma, GN beta)
  float *x, *y, *z, *stats;           // input (not owned), conv out (pre-GN), GN out, GN stats [F][16][2]
  float* gn_part;                     // this layer's dgamma / dbeta row partials [F*S][Co][2]
  int gn_rows;                        // F*S
  __nv_bfloat16 *xb, *zb;             // input / output as bf16 hi / lo planes (GEMM operands; zb may be null)
  __nv_bfloat16 *wr_b, *wd_b;         // this minibatch's weights as GEMM operands (Wr planes, Wd)
  __nv_bfloat16* dyb;                 // GN-backward output (gradient wrt y, bf16): read by dgrad and, on the
                                      // side stream, by wgrad -- one buffer per layer
  int groups = 1;                     // grouped convolution (SE-ResNeXt's 3x3): computed as the dense
                                      // convolution with block-diagonal weights (R9)
};

struct Plan {
  bool rgbd = false;
  int F = 0, layers = 1, fc_in = 512, feat_hw = 4;
  int H = 512, G4 = 2048;     // LSTM hidden size (512, or 1024: lstm_wide.cu) and its 4 gates
  void* lstm_x = nullptr;     // LSTM-1024 L2 exchange buffers (lstm_wide_exchange_bytes)
  std::vector<ConvGN> convs;  // stem, per block: main-branch convs, [down], compress
  struct Block {
    std::vector<int> main;   // convs of the residual branch (ReLU after all but the last)
    int down;                // shortcut conv (-1: identity)
    float *in, *out;         // block input, block output (after residual + ReLU)
    // squeeze-excitation (SE-ResNeXt, R9): out = relu(z3 * s + shortcut), s = sigmoid(W2 relu(W1 pool(z3)
    // + b1) + b2); per-frame s, pooled z3, fc1 pre-activations and the backward's per-frame fc gradients
    bool se = false;
    __nv_bfloat16* outb = nullptr;  // out as bf16 hi / lo planes (the next convolution's operand)
    float *se_s = nullptr, *se_pool = nullptr, *se_a1 = nullptr, *se_da1 = nullptr, *se_da2 = nullptr;
    int64_t se_w1 = 0, se_b1 = 0, se_w2 = 0, se_b2 = 0;
    int C = 0, R = 0, HW = 0;
  };
  std::vector<Block> blocks;
  float *x0, *pool_out;
  __nv_bfloat16 *x0b, *pool_b;
  uint8_t* pool_arg;
  int pool_hw = 0;
  float *flat, *vis, *xin;
  struct Rnn {
    float *GI, *Hs, *Hin, *Cin, *Cs, *IFGO, *dH, *dG;
  } rnn[2];
  // scratch (reused by every layer)
  __nv_bfloat16* dyb;         // GN-backward output (bf16)
  float *dwt, *part, *gn_part, *dz_a, *dz_b, *dz_c, *dz_se, *dxin, *dflat, *dvis;
  size_t part_n = 0;
  float *part_w = nullptr, *part2 = nullptr;  // side-stream partials (weight gradients)
  size_t part_w_n = 0;
  cudaStream_t side = nullptr;                // backward: weight gradients run here (fork / join)
  int grad_planes = 1;                        // 2: the input-gradient chain carries bf16 hi / lo planes
  double* gn_gpart;           // GroupNorm per-chunk group partials (large frames)
  size_t bytes = 0;
};

int64_t off_of(const ModelLayout& L, const std::string& n) { return layout_offset(L, n.c_str()); }

constexpr int kMaxSplits = 64;

// Deterministic carve of the workspace (base == nullptr: size only)
void make_plan(const ModelLayout& L, bool rgbd, int B, int T_run, void* base, Plan* plan) {
  Plan& P = *plan;
  P = Plan();
  const int F = B * T_run;
  P.F = F;
  P.rgbd = rgbd;
  P.layers = rgbd ? 2 : 1;
  const bool serx = layout_offset(L, "enc.layer1.0.se.fc1.weight") >= 0;  // SE-ResNeXt50/2 (R9)
  P.fc_in = rgbd ? 2048 : 512;
  {
    const int i = [&] {
      for (int k = 0; k < L.n; ++k)
        if (!strcmp(L.t[k].name, "head.weight")) return k;
      return -1;
    }();
    P.H = i >= 0 ? (int)L.t[i].shape[1] : 512;
    P.G4 = 4 * P.H;
  }
  // ResNet50/2 is ~50 layers deep: its input-gradient GEMMs take hi / lo operand planes so that the
  // bf16 rounding does not accumulate along the chain (the earliest layers' gradients stay within
  // north_star's 2e-2); the 20-layer ResNet18/2 chain is within it with single bf16 planes
  P.grad_planes = rgbd ? 2 : 1;
  P.feat_hw = rgbd ? 16 : 4;
  size_t off = 0;
  auto take_bytes = [&](size_t bytes) {
    char* p = base ? reinterpret_cast<char*>(base) + off : nullptr;
    off = align_up(off + bytes, 256);
    return p;
  };
  auto take = [&](size_t n) { return reinterpret_cast<float*>(take_bytes(n * sizeof(float))); };
  auto take_b = [&](size_t n) { return reinterpret_cast<__nv_bfloat16*>(take_bytes(n * sizeof(__nv_bfloat16))); };
  size_t max_act = 0, max_w = 0, max_gn_rows = 0, max_gn_part = 0;
  auto add_conv = [&](const std::string& cname, const std::string& gname, int Ci, int Ci_real, int Co, int k, int s,
                      int p, int H, float* x, __nv_bfloat16* xb, bool planes_out, bool needs_dx, int groups = 1) {
    ConvGN c;
    c.groups = groups;
    c.Ci = Ci;
    c.Ci_real = Ci_real;
    c.Co = Co;
    c.k = k;
    c.s = s;
    c.p = p;
    c.H = H;
    c.W = H;
    c.Ho = (H + 2 * p - k) / s + 1;
    c.Wo = c.Ho;
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
    c.wd_b = (Ci > 1 && needs_dx) ? take_b((size_t)P.grad_planes * nw) : nullptr;
    c.dyb = take_b((size_t)P.grad_planes * act);
    max_act = std::max(max_act, std::max(act, (size_t)F * H * H * Ci));
    max_w = std::max(max_w, nw);
    const size_t S = ((size_t)c.Ho * c.Wo * Co + gn_chunk(Co) - 1) / gn_chunk(Co);
    max_gn_rows = std::max(max_gn_rows, (size_t)F * S);
    max_gn_part = std::max(max_gn_part, (size_t)F * S * Co * 2);
    c.gn_part = take((size_t)F * S * Co * 2);  // per layer: reduced once after the whole backward
    c.gn_rows = (int)(F * S);
    P.convs.push_back(c);
    return (int)P.convs.size() - 1;
  };
  int stem;
  if (!rgbd) {
    P.x0 = take((size_t)F * kImg * kImg);
    P.x0b = nullptr;
    stem = add_conv("enc.stem.conv", "enc.stem.gn", 1, 1, 32, 7, 2, 3, kImg, P.x0, nullptr, false, false);
  } else {
    const int h0 = kImgRgbd / 2;  // after the 2x2 average pool
    P.x0 = take((size_t)F * h0 * h0 * 8);
    P.x0b = take_b((size_t)2 * F * h0 * h0 * 8);
    stem = add_conv("enc.stem.conv", "enc.stem.gn", 8, 4, 32, 7, 2, 3, h0, P.x0, P.x0b, false, false);
  }
  const int hs = P.convs[stem].Ho;
  const int hp = (hs + 2 - 3) / 2 + 1;
  P.pool_hw = hp;
  P.pool_out = take((size_t)F * hp * hp * 32);
  P.pool_b = take_b((size_t)2 * F * hp * hp * 32);
  P.pool_arg = reinterpret_cast<uint8_t*>(take_bytes((size_t)F * hp * hp * 32));
  float* z = P.pool_out;
  __nv_bfloat16* zb = P.pool_b;
  int H = hp, cin = 32;
  const int widths[4] = {32, 64, 128, 256};
  const bool r101 = layout_offset(L, "enc.layer3.22.conv1.weight") >= 0;  // SE-ResNeXt101/2
  const int nblocks[4] = {3, 4, r101 ? 23 : 6, 3};
  for (int li = 0; li < 4; ++li) {
    for (int bi = 0; bi < (rgbd ? nblocks[li] : 2); ++bi) {
      const int s = (bi == 0 && li > 0) ? 2 : 1, w = widths[li], cout = rgbd ? 4 * w : w;
      const std::string pre = "enc.layer" + std::to_string(li + 1) + "." + std::to_string(bi);
      Plan::Block blk;
      blk.in = z;
      int Ho;
      if (!rgbd) {  // BasicBlock: 3x3 (stride) -> 3x3
        const int c1 = add_conv(pre + ".conv1", pre + ".gn1", cin, cin, w, 3, s, 1, H, z, zb, true, true);
        Ho = P.convs[c1].Ho;
        const int c2 = add_conv(pre + ".conv2", pre + ".gn2", w, w, w, 3, 1, 1, Ho, P.convs[c1].z, P.convs[c1].zb,
                                true, true);
        blk.main = {c1, c2};
      } else {  // Bottleneck: 1x1 -> 3x3 (stride) -> 1x1 (x4); SE-ResNeXt: inner width 2w, grouped 3x3, SE
        const int wi = serx ? 2 * w : w;
        const int c1 = add_conv(pre + ".conv1", pre + ".gn1", cin, cin, wi, 1, 1, 0, H, z, zb, true, true);
        const int c2 = add_conv(pre + ".conv2", pre + ".gn2", wi, wi, wi, 3, s, 1, H, P.convs[c1].z, P.convs[c1].zb,
                                true, true, serx ? 16 : 1);
        Ho = P.convs[c2].Ho;
        const int c3 = add_conv(pre + ".conv3", pre + ".gn3", wi, wi, cout, 1, 1, 0, Ho, P.convs[c2].z,
                                P.convs[c2].zb, !serx, true);
        blk.main = {c1, c2, c3};
        if (serx) {
          const size_t act = (size_t)F * Ho * Ho * cout;
          blk.se = true;
          blk.C = cout;
          blk.R = cout / 16;
          blk.HW = Ho * Ho;
          blk.out = take(act);
          blk.outb = take_b(2 * act);
          blk.se_s = take((size_t)F * cout);
          blk.se_pool = take((size_t)F * cout);
          blk.se_a1 = take((size_t)F * blk.R);
          blk.se_da1 = take((size_t)F * blk.R);
          blk.se_da2 = take((size_t)F * cout);
          blk.se_w1 = off_of(L, pre + ".se.fc1.weight");
          blk.se_b1 = off_of(L, pre + ".se.fc1.bias");
          blk.se_w2 = off_of(L, pre + ".se.fc2.weight");
          blk.se_b2 = off_of(L, pre + ".se.fc2.bias");
        }
      }
      blk.down = (s != 1 || cin != cout)
                     ? add_conv(pre + ".down.conv", pre + ".down.gn", cin, cin, cout, 1, s, 0, H, z, zb, false, true)
                     : -1;
      const ConvGN& last = P.convs[blk.main.back()];
      if (!blk.se) {
        blk.out = last.z;  // the last main conv's GN output buffer holds relu(gn + shortcut)
        blk.outb = last.zb;
      }
      P.blocks.push_back(blk);
      z = blk.out;
      zb = blk.outb;
      H = Ho;
      cin = cout;
    }
  }
  add_conv("enc.compress.conv", "enc.compress.gn", cin, cin, 128, 3, 1, 1, H, z, zb, false, true);
  P.flat = take((size_t)F * P.fc_in);
  P.vis = take((size_t)F * 512);
  P.xin = take((size_t)F * kXin);
  for (int l = 0; l < P.layers; ++l) {
    Plan::Rnn& r = P.rnn[l];
    r.GI = take((size_t)F * P.G4);
    r.Hs = take((size_t)F * P.H);
    r.Hin = take((size_t)F * P.H);
    r.Cin = take((size_t)F * P.H);
    r.Cs = take((size_t)F * P.H);
    r.IFGO = take((size_t)F * P.H * 4);
    r.dH = take((size_t)F * P.H);
    r.dG = take((size_t)F * P.G4);
  }
  if (P.H != 512) P.lstm_x = take_bytes(lstm_wide_exchange_bytes());
  P.dyb = take_b(max_act);
  P.dwt = take(max_w);
  P.part_n = std::max({(size_t)kMaxSplits * max_w, (size_t)16 * F * P.G4, (size_t)16 * P.G4 * std::max(kXin, P.H)});
  P.part = take(P.part_n);
  // side-stream scratch: weight-gradient partials (tconv split-K: at most ~2 work items of 128 x 64 per
  // SM; the stem's per-frame partials) and the LSTM / visual-FC weight-gradient GEMMs' partials
  P.part_w_n = std::max((size_t)2 * 160 * 128 * 128, (size_t)F * 32 * 64);
  P.part_w = take(P.part_w_n);
  P.part2 = take((size_t)16 << 20);
  P.gn_part = take(max_gn_part);
  P.gn_gpart = reinterpret_cast<double*>(take_bytes(max_gn_rows * kGroups * 2 * sizeof(double)));
  P.dz_a = take(max_act);
  P.dz_b = take(max_act);
  P.dz_c = take(max_act);
  P.dz_se = take(max_act);
  P.dxin = take((size_t)F * kXin);
  P.dflat = take((size_t)F * P.fc_in);
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
  int Cr;  // channels of the parameter tensor (Ci may be padded)
  int groups = 1;
  int K() const { return k * k * Ci; }
  int M() const { return F * Ho * Wo; }
};
struct ConvScratch {
  __nv_bfloat16 *wr_b, *wd_b;  // weights as bf16 (hi/lo planes) / bf16
  float *dwt, *part;           // weight-gradient GEMM output [(u,v,c)][o], split-K partials
  size_t part_n;               // floats available at part
  int slot = 0;                // tconv tile-counter slot (one per concurrently running stream)
};
// split count the partial buffer can hold for an M x N output (<= cap)
inline int split_cap(const ConvScratch& sc, long long M, long long N, int cap) {
  return (int)std::max(1LL, std::min<long long>(cap, (long long)(sc.part_n / (size_t)(M * N))));
}

bool is_stem(const ConvGeom& g) { return g.Ci == 1; }
// the stem shapes the warp-MMA kernels take (the fp32 SIMT kernels take the rest)
bool stem_mma_ok(const ConvGeom& g) {
  return is_stem(g) && (g.Co == 16 || g.Co == 32) && (g.Ho * g.Wo) % 16 == 0 && (g.k == 3 || g.k == 5 || g.k == 7) &&
         g.s <= 2;
}

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
// gsum (nullable): scratch for the stem's GroupNorm sums [F][16][2]; *gsum_done = whether the
// launched kernel wrote them (the warp-MMA stem does, every other path does not)
ddppo_status conv_fwd(ddppo_ctx* ctx, const ConvGeom& g, const float* x, const __nv_bfloat16* xb, const float* w,
                      const __nv_bfloat16* wr_b, float* y, const ConvScratch& sc, cudaStream_t st,
                      double* gsum = nullptr, bool* gsum_done = nullptr, const FrameSrc* fs = nullptr) {
  if (gsum_done) *gsum_done = false;
  if (is_stem(g)) {
    DDPPO_REQUIRE(ctx, g.Co <= kStemCoMax && g.Co % 8 == 0 && (g.k == 3 || g.k == 5 || g.k == 7) && g.s <= 2,
                  "stem conv: Co in {8,..,32}, k in {3, 5, 7}, stride 1 or 2");
    const size_t smem = (size_t)((g.H + 2 * g.p) * (g.W + 2 * g.p + 16) + g.Co * g.k * g.k) * sizeof(float);
    DDPPO_REQUIRE(ctx, smem <= 48 * 1024, "stem conv: frame too large for shared memory");
    if (stem_mma_ok(g)) {  // warp-MMA stem
      const FrameSrc src = fs ? *fs : FrameSrc{x, nullptr, nullptr, 0, 1};
      const size_t sm2 = (size_t)(g.H + 2 * g.p) * (g.W + 2 * g.p) * sizeof(uint32_t);
#define STEM_FWD(K_, S_, C_)                                                                                  \
  if (g.k == K_ && g.s == S_ && g.Co == C_)                                                                  \
    launch_k(ctx, stem_fwd_mma_kernel<K_, S_, C_>, g.F, kThreads, sm2, st, src, w, g.H, g.W, g.p, g.Ho, g.Wo, y, gsum);
      STEM_FWD(7, 2, 32) STEM_FWD(7, 1, 32) STEM_FWD(5, 2, 32) STEM_FWD(5, 1, 32) STEM_FWD(3, 2, 32)
      STEM_FWD(3, 1, 32) STEM_FWD(7, 2, 16) STEM_FWD(7, 1, 16) STEM_FWD(5, 2, 16) STEM_FWD(5, 1, 16)
      STEM_FWD(3, 2, 16) STEM_FWD(3, 1, 16)
#undef STEM_FWD
      if (gsum_done) *gsum_done = gsum != nullptr;
    } else {
      DDPPO_REQUIRE(ctx, !fs || !fs->obs, "stem conv: observation frames need the warp-MMA stem");
#define STEM_FWD(K_, S_)                                                                                   \
  if (g.k == K_ && g.s == S_)                                                                             \
    launch_k(ctx, stem_fwd_kernel<K_, S_>, g.F, kThreads, smem, st, x, w, g.H, g.W, g.Co, g.p, g.Ho, g.Wo, y);
      STEM_FWD(7, 2) STEM_FWD(7, 1) STEM_FWD(5, 2) STEM_FWD(5, 1) STEM_FWD(3, 2) STEM_FWD(3, 1)
#undef STEM_FWD
    }
    ctx->count(1);
    DDPPO_CUDA_TRY(ctx, cudaGetLastError());
    return DDPPO_OK;
  }
  const int K = g.K(), M = g.M();
  if (!wr_b) {  // weights not prepared by weights_prep_kernel (diagnostic entry)
    DDPPO_REQUIRE(ctx, sc.wr_b && g.Cr == g.Ci, "conv: unprepared weights need scratch");
    launch_k(ctx, weights_bf16_kernel, blocks_for(ctx, (size_t)g.Co * K), kThreads, 0, st, w, g.Co, g.Ci, g.k,
             sc.wr_b, nullptr);
    ctx->count(1);
    DDPPO_CUDA_TRY(ctx, cudaGetLastError());
    wr_b = sc.wr_b;
  }
  if (ctx->conv_engine == DDPPO_CONV_TMA && g.Ci % 32 == 0) {
    int splits = 1;
    ddppo_status r = launch_tconv_fwd(ctx, xb, (int64_t)g.F * g.H * g.W * g.Ci, g.F, g.H, g.W, g.Ci, g.k, g.s, g.p, 0,
                                      wr_b, (int64_t)g.Co * K, g.Co, ctx->fwd_planes, y, g.Co, 0, sc.part,
                                      split_cap(sc, M, g.Co, 16), sc.slot, &splits, st);
    if (r != DDPPO_OK || splits == 1) return r;
    return launch_splitk_reduce(ctx, sc.part, splits, (int64_t)M * g.Co, M, g.Co, y, g.Co, 0, st);
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

// dy (bf16, gradient wrt the conv output) -> dw (PyTorch order)
ddppo_status conv_wgrad(ddppo_ctx* ctx, const ConvGeom& g, const float* x, const __nv_bfloat16* xb,
                        const __nv_bfloat16* dy, float* dw, const ConvScratch& sc, cudaStream_t st,
                        const FrameSrc* fs = nullptr) {
  if (is_stem(g)) {
    DDPPO_REQUIRE(ctx, (g.Ho * g.Wo * g.Co) % 8 == 0, "stem conv: Ho*Wo*Co must be a multiple of 8");
    const size_t hp = (size_t)(g.H + 2 * g.p) * (g.W + 2 * g.p);
    const size_t smem = (((size_t)g.Ho * g.Wo * g.Co / 2 + 3) / 4 * 4 + std::max<size_t>(hp, 128 * 16)) * sizeof(float);
    DDPPO_REQUIRE(ctx, smem <= 200 * 1024, "stem conv: frame too large for shared memory");
    static bool attr_set = false;
    if (!attr_set) {
      DDPPO_CUDA_TRY(ctx, cudaFuncSetAttribute(stem_wgrad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               200 * 1024));
      attr_set = true;
    }
    if (stem_mma_ok(g)) {  // warp-MMA stem
      const FrameSrc src = fs ? *fs : FrameSrc{x, nullptr, nullptr, 0, 1};
      const int NC = (g.k * g.k + 7) / 8 * 8;
      const size_t dyw = std::max<size_t>((size_t)g.Ho * g.Wo * g.Co / 2, (size_t)(kThreads / 32) * g.Co * NC);
      const size_t sm2 = (dyw + hp) * sizeof(uint32_t);
      DDPPO_REQUIRE(ctx, sm2 <= 200 * 1024, "stem conv: frame too large for shared memory");
      static bool attr2 = false;
      if (!attr2) {
        for (const void* fn : {(const void*)stem_wgrad_mma_kernel<7, 32>, (const void*)stem_wgrad_mma_kernel<5, 32>,
                               (const void*)stem_wgrad_mma_kernel<3, 32>, (const void*)stem_wgrad_mma_kernel<7, 16>,
                               (const void*)stem_wgrad_mma_kernel<5, 16>, (const void*)stem_wgrad_mma_kernel<3, 16>})
          DDPPO_CUDA_TRY(ctx, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr2 = true;
      }
#define STEM_WG(K_, C_)                                                                                  \
  if (g.k == K_ && g.Co == C_)                                                                          \
    launch_k(ctx, stem_wgrad_mma_kernel<K_, C_>, g.F, kThreads, sm2, st, src, dy, g.H, g.W, g.s, g.p, g.Ho, g.Wo, \
             sc.part);
      STEM_WG(7, 32) STEM_WG(5, 32) STEM_WG(3, 32) STEM_WG(7, 16) STEM_WG(5, 16) STEM_WG(3, 16)
#undef STEM_WG
    } else {
      DDPPO_REQUIRE(ctx, !fs || !fs->obs, "stem conv: observation frames need the warp-MMA stem");
      launch_k(ctx, stem_wgrad_kernel, g.F, kThreads, smem, st, x, dy, g.H, g.W, g.Co, g.k, g.s, g.p, g.Ho, g.Wo,
               sc.part);
    }
    launch_k(ctx, frame_sum_kernel, g.Co * g.k * g.k, kThreads, 0, st, sc.part, g.F, g.Co * g.k * g.k, dw);
    ctx->count(2);
    DDPPO_CUDA_TRY(ctx, cudaGetLastError());
    return DDPPO_OK;
  }
  const int K = g.K(), M = g.M();
  // wgrad: dWt[(u,v,c)][o] = sum_q x[tap(q; u, v)][c] dy[q][o]  (k runs over the M output pixels)
  if (ctx->conv_engine == DDPPO_CONV_TMA && g.Ci % 32 == 0) {
    int splits = 1;
    return launch_tconv_wgrad(ctx, xb, g.F, g.H, g.W, g.Ci, g.k, g.s, g.p, dy, g.Co, dw, g.Cr, sc.part,
                              split_cap(sc, K, g.Co, kMaxSplits), sc.slot, &splits, st, g.groups);
  } else {
    DDPPO_REQUIRE(ctx, g.groups == 1, "conv: grouped convolutions need the TMA engine");
    // split the pixel range so that ~2 CTAs per SM stream (each >= 4 chunks of 64 pixels)
    const int bn = g.Co <= 32 ? 32 : g.Co <= 64 ? 64 : 128;
    const long long tiles = (long long)((g.Co + bn - 1) / bn) * ((K + 127) / 128);
    const int splits = (int)std::max(1LL, std::min<long long>({(2LL * ctx->sm_count + tiles - 1) / tiles,
                                                               (long long)M / 256, (long long)kMaxSplits}));
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
    gm.wg_out = dw;  // the split sum lands in PyTorch order [o][c][u][v] (no dWt round trip)
    gm.wg_cp = g.Ci;
    gm.wg_cr = g.Cr;
    gm.wg_kk = g.k * g.k;
    return launch_igemm(ctx, gm, st);
  }
}

// dx (+)= input gradient of the convolution (not for the stem)
// res != nullptr: dx = dgrad + (res_mask > 0 ? res : 0) (accumulate_dx must be 0): the TMA engine adds
// it in the conv epilogue, the other paths write the masked residual first and accumulate onto it
ddppo_status conv_dgrad(ddppo_ctx* ctx, const ConvGeom& g, const float* w, const __nv_bfloat16* wd_b,
                        const __nv_bfloat16* dy, float* dx, int accumulate_dx, const ConvScratch& sc, cudaStream_t st,
                        int planes = 1, const float* res = nullptr, const float* res_mask = nullptr) {
  DDPPO_REQUIRE(ctx, !is_stem(g), "stem conv: no input gradient");
  DDPPO_REQUIRE(ctx, planes == 1 || wd_b, "conv: hi / lo input gradients need prepared weights");
  const int64_t dy_plane = planes == 2 ? (int64_t)g.M() * g.Co : 0, wd_plane = planes == 2 ? (int64_t)g.Co * g.K() : 0;
  const int K = g.K();
  // dgrad: dx[p][c] (+)= sum_{(u,v,o)} dy[tap^T(p; u, v)][o] W[o][c][u][v]
  if (!wd_b) {
    DDPPO_REQUIRE(ctx, sc.wd_b && g.Cr == g.Ci, "conv: unprepared weights need scratch");
    launch_k(ctx, weights_bf16_kernel, blocks_for(ctx, (size_t)g.Co * K), kThreads, 0, st, w, g.Co, g.Ci, g.k,
             nullptr, sc.wd_b);
    ctx->count(1);
    DDPPO_CUDA_TRY(ctx, cudaGetLastError());
    wd_b = sc.wd_b;
  }
  const int Kd = g.k * g.k * g.Co;
  if (ctx->conv_engine == DDPPO_CONV_TMA && g.s == 1 && g.Co % 32 == 0) {
    // stride 1: the input gradient is the convolution of dy with the mirrored window
    int splits = 1;
    const int Md = g.F * g.H * g.W;
    ddppo_status r = launch_tconv_fwd(ctx, dy, dy_plane, g.F, g.Ho, g.Wo, g.Co, g.k, 1, g.k - 1 - g.p, 1, wd_b,
                                      wd_plane, g.Ci, planes, dx, g.Ci, accumulate_dx, sc.part,
                                      split_cap(sc, Md, g.Ci, 16), sc.slot, &splits, st, res, res_mask);
    if (r != DDPPO_OK || splits == 1) return r;
    return launch_splitk_reduce(ctx, sc.part, splits, (int64_t)Md * g.Ci, Md, g.Ci, dx, g.Ci, accumulate_dx, st);
  }
  if (res) {  // the other engines: the masked residual first, then accumulate onto it
    const size_t n = (size_t)g.F * g.H * g.W * g.Ci;
    launch_k(ctx, relu_mask_kernel, blocks_for(ctx, n), kThreads, 0, st, res, res_mask, n, dx);
    ctx->count(1);
    DDPPO_CUDA_TRY(ctx, cudaGetLastError());
    accumulate_dx = 1;
  }
  if (ctx->conv_engine == DDPPO_CONV_TMA && g.s == 2 && g.Co % 32 == 0 && g.k <= 3 && g.Ci % 8 == 0 &&
      g.k <= g.p + 2) {
    // stride 2: the four output phases, each a stride-1 tap subset over dy, in one launch
    return launch_tconv_dgrad_s2(ctx, dy, dy_plane, g.F, g.Ho, g.Wo, g.Co, g.H, g.W, g.Ci, g.k, g.p, wd_b, wd_plane,
                                 planes, dx, accumulate_dx, st);
  }
  IGemm gm;
  gm.a = op_pix(dy, g.H, g.W, g.Ho, g.Wo, g.Co, g, 1, dy_plane);
  gm.b = op_dense(IG_DENSE_K, wd_b, Kd, wd_plane);
  gm.planes = planes;
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

// elements per thread of a one-block frame (<= NV)
static int gn_vpt(int n, int nt) { return (n + nt - 1) / nt; }

// z = (relu)(GN(y) (+ residual)); stats [F][16][2] = (mean, rstd); zb (nullable) = z as bf16 planes
ddppo_status gn_fwd(ddppo_ctx* ctx, int F, int HW, int C, const float* y, const float* gamma, const float* beta,
                    const float* residual, int relu, float* stats, float* z, __nv_bfloat16* zb, double* gpart,
                    cudaStream_t st, bool pre_stats = false) {
  ProfScope pg(ctx, DDPPO_K_GN, st, 0);
  const int nt = gn_threads(C);
  DDPPO_REQUIRE(ctx, C >= kGroups && C <= kGnMaxThreads && nt % C == 0, "groupnorm: C a power of two in [16, 1024]");
  const int S = (HW * C + gn_chunk(C) - 1) / gn_chunk(C);
  if (S == 1) {  // one block per frame: statistics and normalisation in one pass over the slab
    const int nv = gn_vpt(HW * C, nt);
#define GN_FWD(NV) \
  launch_k(ctx, gn_fwd_kernel<NV>, F, nt, 0, st, y, gamma, beta, residual, HW, C, relu, (size_t)F * HW * C, stats, z, zb)
    if (nv <= 4) GN_FWD(4);
    else if (nv <= 8) GN_FWD(8);
    else if (nv <= 16) GN_FWD(16);
    else GN_FWD(32);
#undef GN_FWD
    ctx->count(1);
  } else {
    DDPPO_REQUIRE(ctx, gpart != nullptr, "groupnorm: large frames need partial-sum scratch");
    // pre_stats: gpart already holds each frame's total sums (one part per frame: the stem kernel)
#define GN_FWD2(NV)                                                                                   \
  do {                                                                                                \
    if (!pre_stats) launch_k(ctx, gn_stats_part_kernel<NV>, dim3(S, F), nt, 0, st, y, HW, C, gpart);  \
    launch_k(ctx, gn_apply_part_kernel<NV>, dim3(S, F), nt, 0, st, y, gpart, gamma, beta, residual, HW, \
             C, relu, (size_t)F * HW * C, stats, z, zb, pre_stats ? 1 : S);                           \
  } while (0)
    if (nt == 1024) GN_FWD2(8);
    else if (nt == 512) GN_FWD2(16);
    else GN_FWD2(32);
#undef GN_FWD2
    ctx->count(pre_stats ? 1 : 2);
  }
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  return DDPPO_OK;
}

// dz: gradient wrt z; relu_z: z if a ReLU produced it (mask z > 0), else null.  Writes dy (gradient
// wrt y, bf16), dgamma, dbeta.  part [F*S][C][2] and gpart [F*S][16][2] (S > 1) are scratch.
template <typename K>
static ddppo_status gn_smem_attr(ddppo_ctx* ctx, K kernel, size_t bytes) {
  static std::map<const void*, size_t> set;  // per kernel: the largest size opted in so far
  size_t& cur = set[reinterpret_cast<const void*>(kernel)];
  if (bytes > cur) {  // (static + dynamic shared memory above 48 KB needs the opt-in)
    DDPPO_CUDA_TRY(ctx, cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    cur = bytes;
  }
  return DDPPO_OK;
}

// cluster launch of gn_bwd_cluster_kernel (S CTAs per frame); *done = false if clusters of S such CTAs
// cannot be resident (the caller falls back to the two-kernel path)
template <typename K>
static ddppo_status gn_bwd_cluster(ddppo_ctx* ctx, K kern, int S, int F, int nt, size_t smem, const float* dz,
                                   const float* relu_z, const float* y, const float* stats, const float* gamma,
                                   int HW, int C, float* part, __nv_bfloat16* dy, size_t lo, cudaStream_t st,
                                   bool* done) {
  static std::map<std::pair<const void*, int>, bool> ok_cache;
  *done = false;
  ddppo_status s = gn_smem_attr(ctx, kern, smem);
  if (s != DDPPO_OK) return s;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(S, F, 1);
  cfg.blockDim = dim3(nt, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)S;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const auto key = std::make_pair(reinterpret_cast<const void*>(kern), S);
  auto it = ok_cache.find(key);
  if (it == ok_cache.end()) {
    bool ok = true;
    if (S > 8) ok = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess;
    int nclus = 0;
    ok = ok && cudaOccupancyMaxActiveClusters(&nclus, kern, &cfg) == cudaSuccess && nclus > 0;
    cudaGetLastError();
    it = ok_cache.emplace(key, ok).first;
  }
  if (!it->second) return DDPPO_OK;
  DDPPO_CUDA_TRY(ctx, cudaLaunchKernelEx(&cfg, kern, dz, relu_z, y, stats, gamma, HW, C, part, dy, lo));
  ctx->count(1);
  *done = true;
  return DDPPO_OK;
}

ddppo_status gn_bwd(ddppo_ctx* ctx, int F, int HW, int C, const float* dz, const float* relu_z, const float* y,
                    const float* stats, const float* gamma, __nv_bfloat16* dy, float* dgamma, float* dbeta,
                    float* part, double* gpart, cudaStream_t st, bool reduce_params = true, size_t lo = 0) {
  ProfScope pg(ctx, DDPPO_K_GN, st, 0);
  ddppo_status s = DDPPO_OK;
  const int nt = gn_threads(C);
  DDPPO_REQUIRE(ctx, C >= kGroups && C <= kGnMaxThreads && nt % C == 0, "groupnorm: C a power of two in [16, 1024]");
  const int S = (HW * C + gn_chunk(C) - 1) / gn_chunk(C);
  if (S == 1) {
    const int nv = gn_vpt(HW * C, nt);
#define GN_BWD(NV)                                                                                    \
  do {                                                                                                \
    s = gn_smem_attr(ctx, gn_bwd_kernel<NV>, gn_bwd_smem(NV, nt));                                    \
    if (s != DDPPO_OK) return s;                                                                      \
    launch_k(ctx, gn_bwd_kernel<NV>, F, nt, gn_bwd_smem(NV, nt), st, dz, relu_z, y, stats, gamma, HW, \
             C, dy, part, lo);                                                                        \
  } while (0)
    if (nv <= 4) GN_BWD(4);
    else if (nv <= 8) GN_BWD(8);
    else if (nv <= 16) GN_BWD(16);
    else GN_BWD(32);
#undef GN_BWD
    ctx->count(1);
  } else {
    DDPPO_REQUIRE(ctx, gpart != nullptr, "groupnorm: large frames need partial-sum scratch");
#define GN_BWD2(NV)                                                                                   \
  do {                                                                                                \
    s = gn_smem_attr(ctx, gn_bwd_part_kernel<NV>, gn_bwd_smem(NV, nt));                               \
    if (s != DDPPO_OK) return s;                                                                      \
    s = gn_smem_attr(ctx, gn_bwd_apply_kernel<NV>, gn_bwd_smem(NV, nt));                              \
    if (s != DDPPO_OK) return s;                                                                      \
    launch_k(ctx, gn_bwd_part_kernel<NV>, dim3(S, F), nt, gn_bwd_smem(NV, nt), st, dz, relu_z, y,     \
             stats, gamma, HW, C, gpart, part);                                                       \
    launch_k(ctx, gn_bwd_apply_kernel<NV>, dim3(S, F), nt, gn_bwd_smem(NV, nt), st, dz, relu_z, y,    \
             stats, gamma, gpart, HW, C, dy, lo);                                                     \
  } while (0)
    bool done = false;
    if (S <= 16) {  // one pass: the frame's chunks as a thread-block cluster
#define GN_BWDC(NV) s = gn_bwd_cluster(ctx, gn_bwd_cluster_kernel<NV>, S, F, nt, gn_bwd_smem(NV, nt), dz, relu_z, y, \
                                      stats, gamma, HW, C, part, dy, lo, st, &done)
      if (nt == 1024) GN_BWDC(8);
      else if (nt == 512) GN_BWDC(16);
      else GN_BWDC(32);
#undef GN_BWDC
      if (s != DDPPO_OK) return s;
    }
    if (!done) {
      if (nt == 1024) GN_BWD2(8);
      else if (nt == 512) GN_BWD2(16);
      else GN_BWD2(32);
      ctx->count(2);
    }
#undef GN_BWD2
  }
  if (reduce_params) {  // else the caller reduces `part` later (gn_param_reduce_all)
    launch_k(ctx, gn_param_reduce_kernel, C, kThreads, 0, st, part, F * S, C, dgamma, dbeta);
    ctx->count(1);
  }
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  return DDPPO_OK;
}

ConvGeom geom_of(const Plan& P, const ConvGN& c) {
  return ConvGeom{P.F, c.H, c.W, c.Ci, c.Co, c.k, c.s, c.p, c.Ho, c.Wo, c.Ci_real, c.groups};
}
ConvScratch scratch_of(const Plan& P) { return ConvScratch{nullptr, nullptr, P.dwt, P.part, P.part_n}; }  // weights prepared

// conv (+GN (+residual) (+ReLU)) forward
ddppo_status conv_gn_fwd(ddppo_ctx* ctx, const float* prm, Plan& P, ConvGN& c, const float* residual, int relu,
                         cudaStream_t st, const FrameSrc* fs = nullptr) {
  bool pre = false;  // (the stem writes its GroupNorm sums itself)
  ddppo_status s =
      conv_fwd(ctx, geom_of(P, c), c.x, c.xb, prm + c.w, c.wr_b, c.y, scratch_of(P), st, P.gn_gpart, &pre, fs);
  if (s != DDPPO_OK) return s;
  return gn_fwd(ctx, P.F, c.Ho * c.Wo, c.Co, c.y, prm + c.gw, prm + c.gb, residual, relu, c.stats, c.z, c.zb,
                P.gn_gpart, st, pre);
}

// backward of conv+GN: dz = gradient wrt the GN(+residual)(+ReLU) output; relu_z = that output if a
// ReLU followed (its > 0 mask), else null.  Writes dW, dgamma, dbeta into grad; dx (+)= into dx.
// The weight gradient only feeds a8, so with a side stream it leaves the critical path: it is
// forked after the GN backward (its own dy buffer and partials) and joined once after the backward.
ddppo_status conv_gn_bwd(ddppo_ctx* ctx, const float* prm, float* grad, Plan& P, ConvGN& c, const float* dz,
                         const float* relu_z, float* dx, int accumulate_dx, cudaStream_t st, const float* res = nullptr,
                         const float* res_mask = nullptr, const FrameSrc* fs = nullptr) {
  const size_t lo = P.grad_planes == 2 ? (size_t)P.F * c.Ho * c.Wo * c.Co : 0;
  ddppo_status s = gn_bwd(ctx, P.F, c.Ho * c.Wo, c.Co, dz, relu_z, c.y, c.stats, prm + c.gw, c.dyb, grad + c.gw,
                          grad + c.gb, c.gn_part, P.gn_gpart, st, /*reduce_params=*/false, lo);
  if (s != DDPPO_OK) return s;
  const ConvGeom g = geom_of(P, c);
  if (P.side) {
    DDPPO_CUDA_TRY(ctx, fork_to(ctx, st, P.side));
    ConvScratch ws = {nullptr, nullptr, P.dwt, P.part_w, P.part_w_n, 1};
    s = conv_wgrad(ctx, g, c.x, c.xb, c.dyb, grad + c.w, ws, P.side, fs);
  } else {
    s = conv_wgrad(ctx, g, c.x, c.xb, c.dyb, grad + c.w, scratch_of(P), st, fs);
  }
  if (s != DDPPO_OK || dx == nullptr) return s;
  return conv_dgrad(ctx, g, prm + c.w, c.wd_b, c.dyb, dx, accumulate_dx, scratch_of(P), st, P.grad_planes, res,
                    res_mask);
}

// gemm_tc with split-K chosen so that small-M / long-K GEMMs still fill the GPU (partials in P.part)
ddppo_status gemm_split(ddppo_ctx* ctx, GemmTC g, const Plan& P, cudaStream_t st, float* part = nullptr) {
  const int bn = g.N <= 32 ? 32 : (g.N <= 64 || g.prec == 3) ? 64 : 128;
  const long long tiles = (long long)((g.N + bn - 1) / bn) * ((g.M + 127) / 128);
  const int chunks = (g.K + 63) / 64;
  // split-K toward one wave of CTAs, >= 2 K chunks per split (measured r2: 2x the SM count or
  // >= 4 chunks per split are 0.4-1.1 % slower per Depth step; no split 6 % slower)
  const int splits =
      (int)std::max(1LL, std::min<long long>({((long long)ctx->sm_count + tiles - 1) / tiles, chunks / 2, 16}));
  if (splits > 1) {
    g.splits = splits;
    g.partial = part ? part : P.part;
  }
  return launch_gemm_tc(ctx, g, st);
}

// parameter names of LSTM layer l ("rnn.weight_ih" for the 1-layer Depth agent, "..._l<l>" for RGB-D)
std::string rnn_name(const Plan& P, const char* base, int l) {
  return P.layers == 1 ? std::string(base) : std::string(base) + "_l" + std::to_string(l);
}

LstmPtrs lstm_ptrs(const ModelLayout& L, const float* prm, const ddppo_batch& b, Plan& P, int l) {
  const Plan::Rnn& r = P.rnn[l];
  LstmPtrs q;
  q.Whh = prm + off_of(L, rnn_name(P, "rnn.weight_hh", l));
  q.bih = prm + off_of(L, rnn_name(P, "rnn.bias_ih", l));
  q.bhh = prm + off_of(L, rnn_name(P, "rnn.bias_hh", l));
  q.GI = r.GI;
  q.mask = b.mask;
  q.h0 = b.h0 + (size_t)l * P.H;
  q.c0 = b.c0 + (size_t)l * P.H;
  q.sld = P.layers * P.H;
  q.H = P.H;
  if (P.lstm_x) {
    q.hx = P.lstm_x;
    q.xcnt = reinterpret_cast<unsigned*>(reinterpret_cast<char*>(P.lstm_x) + lstm_wide_exchange_bytes() - 256);
    q.xpart = reinterpret_cast<float*>(reinterpret_cast<char*>(P.lstm_x) + lstm_wide_part_offset());
  }
  q.env_idx = b.env_idx;
  q.B = b.B;
  q.T_run = b.T_run;
  q.ld = b.ld;
  q.Hs = r.Hs;
  q.Hin = r.Hin;
  q.Cin = r.Cin;
  q.Cs = r.Cs;
  q.IFGO = reinterpret_cast<float4*>(r.IFGO);
  q.dH = r.dH;
  q.dG = r.dG;
  return q;
}

bool is_rgbd(const ModelLayout& L) { return layout_offset(L, "rnn.weight_ih_l0") >= 0; }

}  // namespace

// h_t / c_t of LSTM layer l for every sample [B*T_run][hidden] in a forward's workspace (act path)
void depth_state_out(const ModelLayout& L, void* ws, int B, int T_run, int l, const float** Hs, const float** Cs) {
  Plan P;
  make_plan(L, is_rgbd(L), B, T_run, ws, &P);
  *Hs = P.rnn[l].Hs;
  *Cs = P.rnn[l].Cs;
}

size_t depth_workspace(int arch, int hidden, int max_B, int T) {
  ddppo_model_desc d = {};
  d.arch = arch;
  d.hidden = hidden;
  d.num_actions = 4;
  ModelLayout L;
  build_layout(&d, &L);
  Plan P;
  make_plan(L, arch_rgbd(arch), max_B, T, nullptr, &P);
  return P.bytes;
}

namespace {
// encoder -> visual FC -> LSTM input -> (per LSTM layer: input GEMM, recurrence)
ddppo_status depth_fwd_net(ddppo_ctx* ctx, const ModelLayout& L, const float* prm, const ddppo_batch& b, Plan& P,
                           cudaStream_t st) {
  const int F = P.F;
  cudaStream_t prep_st = st;
  {
    WeightPrep prep;
    prep.n = 0;
    prep.off[0] = 0;
    prep.offd[0] = 0;
    for (size_t i = 0; i < P.convs.size(); ++i) {
      const ConvGN& c = P.convs[i];
      if (c.Ci == 1) continue;  // the Depth stem splits its fp32 weights into bf16 planes itself
      DDPPO_REQUIRE(ctx, prep.n < kMaxConvs, "too many convolutions for one weight-prep launch");
      prep.it[prep.n] = WeightPrep::Item{prm + c.w, c.wr_b, c.wd_b, c.Co, c.Ci_real, c.Ci, c.k, P.grad_planes, c.groups};
      prep.off[prep.n + 1] = prep.off[prep.n] + c.Co;
      prep.offd[prep.n + 1] = prep.offd[prep.n] + (c.wd_b ? c.Ci_real : 0);
      ++prep.n;
    }
    // the operand prep (the conv kernels' bf16 weight planes: the role of a bf16 parameter shadow)
    // runs on the side stream beside the input prologue and (Depth) the stem + max-pool; joined
    // before the first TMA convolution
    if (ctx->conv_engine == DDPPO_CONV_TMA) {
      cudaStream_t sb = nullptr;
      ddppo_status r = ctx_side_streams(ctx, &P.side, &sb);
      if (r != DDPPO_OK) return r;
      DDPPO_CUDA_TRY(ctx, fork_to(ctx, st, P.side));
      prep_st = P.side;
    }
    launch_k(ctx, weights_prep_kernel, prep.off[prep.n] + prep.offd[prep.n], 256, 0, prep_st, prep);
    ctx->count(1);
  }
  auto join_prep = [&]() -> cudaError_t {
    if (prep_st == st) return cudaSuccess;
    prep_st = st;
    return fork_to(ctx, P.side, st);
  };
  const FrameSrc fs{P.x0, reinterpret_cast<const __nv_bfloat16*>(b.obs), b.env_idx, b.T, b.T_run};
  const bool direct = !P.rgbd && stem_mma_ok(geom_of(P, P.convs[0]));  // the stem reads the observations
  if (!P.rgbd && !direct) {
    launch_k(ctx, gather_obs_kernel, blocks_for(ctx, (size_t)F * kImg * kImg / 8), kThreads, 0, st,
             reinterpret_cast<const __nv_bfloat16*>(b.obs), b.env_idx, b.T, b.T_run, F, P.x0);
    ctx->count(1);
  } else if (P.rgbd) {
    DDPPO_REQUIRE(ctx, kImgRgbd % 4 == 0, "rgbd: input width must be a multiple of 4");
    launch_k(ctx, rgbd_prologue_kernel, (F * (kImgRgbd / 2) * (kImgRgbd / 4) + kThreads - 1) / kThreads, kThreads, 0,
             st, b.obs_rgb, reinterpret_cast<const __nv_bfloat16*>(b.obs), b.env_idx, b.T, b.T_run, F, kImgRgbd,
             P.x0, P.x0b);
    ctx->count(1);
  }
  if (P.convs[0].Ci != 1) DDPPO_CUDA_TRY(ctx, join_prep());  // RGB-D: the stem is a TMA convolution
  ddppo_status s = conv_gn_fwd(ctx, prm, P, P.convs[0], nullptr, 1, st, direct ? &fs : nullptr);
  if (s != DDPPO_OK) return s;
  {
    ConvGN& c = P.convs[0];
    const int hp = P.pool_hw;
    launch_k(ctx, maxpool_fwd_kernel, (F * hp * hp * 8 + kThreads - 1) / kThreads, kThreads, 0, st, 
        c.z, F, c.Ho, c.Wo, 32, hp, hp, P.pool_out, P.pool_arg, P.pool_b);
    ctx->count(1);
  }
  DDPPO_CUDA_TRY(ctx, join_prep());
  for (auto& blk : P.blocks) {
    const float* sc = blk.in;
    if (blk.down >= 0) {
      if ((s = conv_gn_fwd(ctx, prm, P, P.convs[blk.down], nullptr, 0, st)) != DDPPO_OK) return s;
      sc = P.convs[blk.down].z;
    }
    for (size_t j = 0; j < blk.main.size(); ++j) {
      const bool last = j + 1 == blk.main.size();
      // SE blocks: the last GN output (z3) is excited before the residual addition + ReLU
      const bool fuse_res = last && !blk.se;
      if ((s = conv_gn_fwd(ctx, prm, P, P.convs[blk.main[j]], fuse_res ? sc : nullptr, last && blk.se ? 0 : 1, st)) !=
          DDPPO_OK)
        return s;
    }
    if (blk.se) {
      const ConvGN& c3 = P.convs[blk.main.back()];
      const size_t smem = (size_t)(2 * blk.C + blk.R) * sizeof(float);
      launch_k(ctx, se_fwd_kernel, F, 256, smem, st, c3.z, sc, prm + blk.se_w1, prm + blk.se_b1, prm + blk.se_w2,
               prm + blk.se_b2,
                                          blk.HW, blk.C, blk.R, blk.out, blk.outb, (size_t)F * blk.HW * blk.C,
                                          blk.se_s, blk.se_pool, blk.se_a1);
      ctx->count(1);
      DDPPO_CUDA_TRY(ctx, cudaGetLastError());
    }
  }
  ConvGN& comp = P.convs.back();
  if ((s = conv_gn_fwd(ctx, prm, P, comp, nullptr, 1, st)) != DDPPO_OK) return s;
  launch_k(ctx, flatten_kernel, blocks_for(ctx, (size_t)F * P.fc_in), kThreads, 0, st, comp.z, F, P.feat_hw, 128,
           P.flat, 1);
  ctx->count(1);
  // visual FC + ReLU
  if ((s = gemm_split(ctx, GemmTC{P.flat, P.fc_in, 1, prm + off_of(L, "visual_fc.weight"), P.fc_in, 1, P.vis, 512, F,
                                  512, P.fc_in, 1, nullptr, kPrecFwd},
                      P, st)) != DDPPO_OK)
    return s;
  launch_k(ctx, bias_act_kernel, blocks_for(ctx, (size_t)F * 512), kThreads, 0, st, P.vis, prm + off_of(L,
           "visual_fc.bias"), F,
                                                                         512, 1);
  ctx->count(1);
  launch_k(ctx, lstm_input_kernel, blocks_for(ctx, (size_t)F * kXin), kThreads, 0, st, 
      P.vis, b.goal, b.prev_action, b.env_idx, prm + off_of(L, "goal_fc.weight"), prm + off_of(L, "goal_fc.bias"),
      prm + off_of(L, "act_embed.weight"), b.T, b.ld, b.T_run, F, P.xin);
  ctx->count(1);
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  for (int l = 0; l < P.layers; ++l) {
    // GI = x W_ih^T (biases are added inside the recurrence); layer l > 0 reads layer l-1's h
    const float* xl = l == 0 ? P.xin : P.rnn[l - 1].Hs;
    const int nin = l == 0 ? kXin : P.H;
    if ((s = gemm_split(ctx, GemmTC{xl, nin, 1, prm + off_of(L, rnn_name(P, "rnn.weight_ih", l)), nin, 1, P.rnn[l].GI,
                                    P.G4, F, P.G4, nin, 1, nullptr, kPrecFwd},
                        P, st)) != DDPPO_OK)
      return s;
    if ((s = launch_lstm_fwd(ctx, lstm_ptrs(L, prm, b, P, l), st)) != DDPPO_OK) return s;
  }
  return DDPPO_OK;
}
}  // namespace

ddppo_status depth_fwd(ddppo_ctx* ctx, const ModelLayout& L, const float* prm, const ddppo_batch& b, float* logits,
                       float* values, void* ws, cudaStream_t st) {
  DDPPO_REQUIRE(ctx, b.obs && b.c0, "visual agent: batch needs obs and c0");
  DDPPO_REQUIRE(ctx, !is_rgbd(L) || b.obs_rgb, "RGB-D agent: batch needs obs_rgb");
  DDPPO_REQUIRE(ctx, ((uintptr_t)b.obs & 15) == 0 && ((uintptr_t)b.obs_rgb & 3) == 0,
                "visual agent: obs must be 16-byte aligned, obs_rgb 4-byte aligned");
  DDPPO_REQUIRE(ctx, b.B >= 1 && b.B <= 8 && b.T_run <= 1024, "visual agent: minibatch must hold 1..8 envs, T <= 1024");
  Plan P;
  make_plan(L, is_rgbd(L), b.B, b.T_run, ws, &P);
  {
    ProfScope ps(ctx, DDPPO_K_NET_FWD, st, 0);
    ddppo_status s = depth_fwd_net(ctx, L, prm, b, P, st);
    if (s != DDPPO_OK) return s;
  }
  ProfScope ps(ctx, DDPPO_K_HEAD, st, 0);
  return launch_head_fwd(ctx, prm + off_of(L, "head.weight"), prm + off_of(L, "head.bias"), P.rnn[P.layers - 1].Hs,
                         P.F, P.H, logits, values, st);
}

ddppo_status depth_bwd(ddppo_ctx* ctx, const ModelLayout& L, const float* prm, const ddppo_batch& b,
                       const float* dlogits, const float* dvalues, float* grad, void* ws, cudaStream_t st) {
  Plan P;
  make_plan(L, is_rgbd(L), b.B, b.T_run, ws, &P);
  const int F = P.F;
  ddppo_status s;
  {
    ProfScope ps(ctx, DDPPO_K_HEAD, st, 0);
    s = launch_head_bwd(ctx, prm + off_of(L, "head.weight"), P.rnn[P.layers - 1].Hs, dlogits, dvalues, F, P.H,
                        P.rnn[P.layers - 1].dH, grad + off_of(L, "head.weight"), grad + off_of(L, "head.bias"), st);
    if (s != DDPPO_OK) return s;
  }
  ProfScope ps(ctx, DDPPO_K_NET_BWD, st, 0);
  // weight gradients (LSTM, visual FC, convolutions) only feed a8: they run on a side stream beside
  // the chain of input gradients, joined once at the end
  cudaStream_t wst = st;
  if (ctx->conv_engine == DDPPO_CONV_TMA) {
    cudaStream_t sb = nullptr;
    if ((s = ctx_side_streams(ctx, &P.side, &sb)) != DDPPO_OK) return s;
    wst = P.side;
  }
  for (int l = P.layers - 1; l >= 0; --l) {
    Plan::Rnn& r = P.rnn[l];
    if ((s = launch_lstm_bwd(ctx, lstm_ptrs(L, prm, b, P, l), st)) != DDPPO_OK) return s;
    // weight gradients and db (b_ih and b_hh receive the same gradient)
    const float* xl = l == 0 ? P.xin : P.rnn[l - 1].Hs;
    const int nin = l == 0 ? kXin : P.H;
    const int kG4 = P.G4, kH = P.H;
    const float* Wih = prm + off_of(L, rnn_name(P, "rnn.weight_ih", l));
    if (wst != st) DDPPO_CUDA_TRY(ctx, fork_to(ctx, st, wst));
    if ((s = gemm_split(ctx, GemmTC{r.dG, 1, kG4, xl, 1, nin, grad + off_of(L, rnn_name(P, "rnn.weight_ih", l)), nin,
                                    kG4, nin, F},
                        P, wst, P.part2)) != DDPPO_OK)
      return s;
    if ((s = gemm_split(ctx, GemmTC{r.dG, 1, kG4, r.Hin, 1, kH, grad + off_of(L, rnn_name(P, "rnn.weight_hh", l)), kH,
                                    kG4, kH, F},
                        P, wst, P.part2)) != DDPPO_OK)
      return s;
    if ((s = launch_colsum(ctx, r.dG, kG4, F, kG4, grad + off_of(L, rnn_name(P, "rnn.bias_ih", l)), wst)) != DDPPO_OK)
      return s;
    if ((s = launch_colsum(ctx, r.dG, kG4, F, kG4, grad + off_of(L, rnn_name(P, "rnn.bias_hh", l)), wst)) != DDPPO_OK)
      return s;
    // input gradient: into the layer below's dH, or dx = dG W_ih [F][576] for layer 0
    float* dxl = l == 0 ? P.dxin : P.rnn[l - 1].dH;
    if ((s = gemm_split(ctx, GemmTC{r.dG, kG4, 1, Wih, 1, nin, dxl, nin, F, nin, kG4}, P, st)) != DDPPO_OK) return s;
  }
  launch_k(ctx, goal_emb_grads_kernel, 64, kThreads, 0, st, P.dxin, b.goal, b.prev_action, b.env_idx, b.T, b.ld,
           b.T_run, F,
                                                 grad + off_of(L, "goal_fc.weight"), grad + off_of(L, "goal_fc.bias"),
                                                 grad + off_of(L, "act_embed.weight"));
  ctx->count(1);
  if (b.dgoal) {  // the planner's gradient through the (frozen) controller
    launch_k(ctx, goal_input_grad_kernel, blocks_for(ctx, (size_t)F * 3), kThreads, 0, st, 
        P.dxin, prm + off_of(L, "goal_fc.weight"), F, b.dgoal);
    ctx->count(1);
  }
  launch_k(ctx, vis_mask_kernel, blocks_for(ctx, (size_t)F * 512), kThreads, 0, st, P.dxin, P.vis, F, P.dvis);
  ctx->count(1);
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  // visual FC: dW = dVpre^T flat, db = colsum(dVpre) (side stream), dflat = dVpre W
  if (wst != st) DDPPO_CUDA_TRY(ctx, fork_to(ctx, st, wst));
  if ((s = gemm_split(ctx, GemmTC{P.dvis, 1, 512, P.flat, 1, P.fc_in, grad + off_of(L, "visual_fc.weight"), P.fc_in,
                                  512, P.fc_in, F},
                      P, wst, P.part2)) != DDPPO_OK)
    return s;
  if ((s = launch_colsum(ctx, P.dvis, 512, F, 512, grad + off_of(L, "visual_fc.bias"), wst)) != DDPPO_OK) return s;
  if (b.flags & DDPPO_BATCH_FREEZE_ENCODER) {
    // frozen encoder (NEXT-4): no encoder backward; its gradient entries are 0 (they lead the layout)
    DDPPO_CUDA_TRY(ctx, cudaMemsetAsync(grad, 0, (size_t)encoder_end(L) * sizeof(float), st));
    if (wst != st) DDPPO_CUDA_TRY(ctx, fork_to(ctx, wst, st));
    return DDPPO_OK;
  }
  if ((s = gemm_split(ctx, GemmTC{P.dvis, 512, 1, prm + off_of(L, "visual_fc.weight"), 1, P.fc_in, P.dflat, P.fc_in,
                                  F, P.fc_in, 512},
                      P, st)) != DDPPO_OK)
    return s;
  // encoder: dz = gradient wrt the current block output; three rotating activation buffers
  ConvGN& comp = P.convs.back();
  float* dz = P.dz_a;
  float* da = P.dz_b;
  float* dn = P.dz_c;
  launch_k(ctx, flatten_kernel, blocks_for(ctx, (size_t)F * P.fc_in), kThreads, 0, st, P.dflat, F, P.feat_hw, 128, da,
           0);
  ctx->count(1);
  if ((s = conv_gn_bwd(ctx, prm, grad, P, comp, da, comp.z, dz, 0, st)) != DDPPO_OK) return s;
  for (int bi = (int)P.blocks.size() - 1; bi >= 0; --bi) {
    const Plan::Block& blk = P.blocks[bi];
    ConvGN& last = P.convs[blk.main.back()];
    // out = relu(gn_last(conv_last(...)) (* SE) + shortcut(in)); the ReLU mask of the sum is `out`
    // identity shortcut of a two-conv block: the first conv's input-gradient epilogue adds the masked
    // shortcut gradient (dz stays intact until then); otherwise it is written first and accumulated onto
    // (bottlenecks: the middle conv's gradient goes to dz_se, free outside SE blocks, so dz survives;
    // in SE blocks the chain starts from dz_se and never touches dz)
    const bool fuse_res = blk.down < 0;
    if (blk.down >= 0) {
      if ((s = conv_gn_bwd(ctx, prm, grad, P, P.convs[blk.down], dz, blk.out, dn, 0, st)) != DDPPO_OK) return s;
    } else if (!fuse_res) {
      const size_t n = (size_t)F * last.Ho * last.Wo * last.Co;
      launch_k(ctx, relu_mask_kernel, blocks_for(ctx, n), kThreads, 0, st, dz, blk.out, n, dn);
      ctx->count(1);
    }
    // main branch, last conv first: its upstream mask is the block output (or, after the SE module, none),
    // the others' their own ReLU
    float* g_in = dz;    // gradient wrt the current conv's output
    float* g_out = da;   // gradient wrt its input
    if (blk.se) {
      const size_t smem = (size_t)(2 * blk.C + blk.R) * sizeof(float);
      launch_k(ctx, se_bwd_kernel, F, 256, smem, st, dz, blk.out, last.z, blk.se_s, blk.se_a1, prm + blk.se_w1,
               prm + blk.se_w2,
                                          blk.HW, blk.C, blk.R, P.dz_se, blk.se_da1, blk.se_da2);
      ctx->count(1);
      DDPPO_CUDA_TRY(ctx, cudaGetLastError());
      cudaStream_t pst = st;
      if (P.side) {  // the SE parameters' gradient only feeds a8: side stream
        DDPPO_CUDA_TRY(ctx, fork_to(ctx, st, P.side));
        pst = P.side;
      }
      const int n = 2 * blk.R * blk.C + blk.R + blk.C;
      launch_k(ctx, se_param_grad_kernel, blocks_for(ctx, (size_t)n), kThreads, 0, pst, 
          blk.se_da1, blk.se_da2, blk.se_pool, blk.se_a1, F, blk.C, blk.R, grad + blk.se_w1, grad + blk.se_b1,
          grad + blk.se_w2, grad + blk.se_b2);
      ctx->count(1);
      DDPPO_CUDA_TRY(ctx, cudaGetLastError());
      g_in = P.dz_se;
    }
    for (int j = (int)blk.main.size() - 1; j >= 0; --j) {
      ConvGN& c = P.convs[blk.main[j]];
      const bool first = j == 0;
      float* target = first ? dn : g_out;
      const float* relu_z = (j + 1 == (int)blk.main.size()) ? (blk.se ? nullptr : blk.out) : c.z;
      if (first && fuse_res)
        s = conv_gn_bwd(ctx, prm, grad, P, c, g_in, relu_z, target, 0, st, dz, blk.out);
      else
        s = conv_gn_bwd(ctx, prm, grad, P, c, g_in, relu_z, target, first ? 1 : 0, st);
      if (s != DDPPO_OK) return s;
      if (!first) {
        std::swap(g_in, g_out);  // g_in <- this conv's input gradient; g_out <- a free buffer
        if (g_out == dn) g_out = (g_in == dz) ? da : dz;
        if (fuse_res && g_out == dz) g_out = (g_in == P.dz_se) ? da : P.dz_se;  // dz: the first conv's residual
      }
    }
    std::swap(dz, dn);  // dn (the block input's gradient) becomes the next dz
  }
  // max-pool, then the stem (no input gradient).  (Gathering the pool's gradient inside the stem's
  // GroupNorm backward instead -- no dense gradient in HBM -- measured 3 us slower per minibatch:
  // the cluster kernel's 2 CTAs / SM cannot hide the gather's L2 latency.)
  ConvGN& stem = P.convs[0];
  if (stem.Ho == 2 * P.pool_hw && stem.Wo == 2 * P.pool_hw)
    launch_k(ctx, maxpool_bwd2_kernel, dim3((P.pool_hw * P.pool_hw * 8 + kThreads - 1) / kThreads, F), kThreads, 0, st,
             dz, P.pool_arg, P.pool_hw, P.pool_hw, 32, da);
  else
    launch_k(ctx, maxpool_bwd_kernel, dim3((stem.Ho * stem.Wo * 8 + kThreads - 1) / kThreads, F), kThreads, 0, st, dz,
             P.pool_arg, F, stem.Ho, stem.Wo, 32, P.pool_hw, P.pool_hw, da);
  ctx->count(1);
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  const FrameSrc fs{P.x0, reinterpret_cast<const __nv_bfloat16*>(b.obs), b.env_idx, b.T, b.T_run};
  const bool direct = !P.rgbd && stem_mma_ok(geom_of(P, stem));  // (as in the forward)
  if ((s = conv_gn_bwd(ctx, prm, grad, P, stem, da, stem.z, nullptr, 0, st, nullptr, nullptr, direct ? &fs : nullptr)) !=
      DDPPO_OK)
    return s;
  // all layers' dgamma / dbeta from their row partials, one launch
  GnParamAll a;
  a.n = 0;
  a.ch_off[0] = 0;
  for (const ConvGN& c : P.convs) {
    DDPPO_REQUIRE(ctx, a.n < kMaxConvsGn, "too many GroupNorm layers for one reduction launch");
    a.it[a.n] = GnParamAll::Item{c.gn_part, grad + c.gw, grad + c.gb, c.gn_rows, c.Co};
    a.ch_off[a.n + 1] = a.ch_off[a.n] + (c.Co + 31) / 32;  // blocks of 32 channels
    ++a.n;
  }
  launch_k(ctx, gn_param_reduce_all_kernel, a.ch_off[a.n], kGnRedThreads, 0, st, a);
  ctx->count(1);
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  if (wst != st) DDPPO_CUDA_TRY(ctx, fork_to(ctx, wst, st));  // join: every weight gradient is final
  return DDPPO_OK;
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
  ConvGeom g{F, H, W, Ci, Co, k, s, p, Ho, Wo, Ci};
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
  sc.part_n = nf - ok;
  cudaStream_t st = as_stream(stream);
  ProfScope ps(ctx, DDPPO_K_OTHER, st, 0);
  launch_k(ctx, to_planes_kernel, blocks_for(ctx, nx), kThreads, 0, st, x, nx, xb);
  ctx->count(1);
  if (y) {
    ddppo_status r = conv_fwd(ctx, g, x, xb, w, nullptr, y, sc, st);
    if (r != DDPPO_OK) return r;
  }
  if (dy) {
    launch_k(ctx, to_bf16_kernel, blocks_for(ctx, ny), kThreads, 0, st, dy, ny, dyb);
    ctx->count(1);
    ddppo_status r = conv_wgrad(ctx, g, x, xb, dyb, dw, sc, st);
    if (r != DDPPO_OK || Ci == 1 || dx == nullptr) return r;
    return conv_dgrad(ctx, g, w, nullptr, dyb, dx, 0, sc, st);
  }
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  return DDPPO_OK;
}

namespace {
__global__ void bf16_to_f32_kernel(const __nv_bfloat16* __restrict__ x, size_t n, float* __restrict__ y) {
  pdl_enter();
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
  const int S = (HW * C + gn_chunk(C) - 1) / gn_chunk(C);
  float* part = scratch;                                                                 // [F*S][C][2]
  double* gpart = reinterpret_cast<double*>(scratch + align_up((size_t)F * S * C * 2, 2));  // [F*S][16][2]
  __nv_bfloat16* dyb = reinterpret_cast<__nv_bfloat16*>(gpart + (size_t)F * S * kGroups * 2);
  ddppo_status r = gn_fwd(ctx, F, HW, C, y, gamma, beta, residual, relu, stats, z, nullptr, gpart, st);
  if (r != DDPPO_OK || !dz) return r;
  r = gn_bwd(ctx, F, HW, C, dz, relu ? z : nullptr, y, stats, gamma, dyb, dgamma, dbeta, part, gpart, st);
  if (r != DDPPO_OK) return r;
  launch_k(ctx, bf16_to_f32_kernel, blocks_for(ctx, (size_t)F * HW * C), kThreads, 0, st, dyb, (size_t)F * HW * C, dy);
  ctx->count(1);
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  return DDPPO_OK;
}

extern "C" ddppo_status ddppo_debug_maxpool(ddppo_ctx* ctx, const float* x, int F, int H, int W, int C, float* y,
                                            uint8_t* arg, const float* dy, float* dx, void* stream) {
  if (!ctx) return DDPPO_ERR_CONFIG;
  DDPPO_REQUIRE(ctx, F >= 1 && H >= 2 && W >= 2 && C >= 4 && C % 4 == 0, "maxpool: bad geometry (C % 4 == 0)");
  DDPPO_REQUIRE(ctx, (size_t)F * H * W * C < (1u << 31), "maxpool: tensor too large");
  const int Ho = (H + 2 - 3) / 2 + 1, Wo = (W + 2 - 3) / 2 + 1;
  cudaStream_t st = as_stream(stream);
  ProfScope ps(ctx, DDPPO_K_OTHER, st, 0);
  launch_k(ctx, maxpool_fwd_kernel, (F * Ho * Wo * (C / 4) + kThreads - 1) / kThreads, kThreads, 0, st, x, F, H, W, C,
           Ho, Wo, y, arg,
                                                                                     nullptr);
  ctx->count(1);
  if (dy) {  // the Depth step's dispatch: the 2x2-block kernel for even maps
    if (H == 2 * Ho && W == 2 * Wo)
      launch_k(ctx, maxpool_bwd2_kernel, dim3((Ho * Wo * (C / 4) + kThreads - 1) / kThreads, F), kThreads, 0, st, dy,
               arg, Ho, Wo, C, dx);
    else
      launch_k(ctx, maxpool_bwd_kernel, dim3((H * W * (C / 4) + kThreads - 1) / kThreads, F), kThreads, 0, st, dy, arg,
               F, H, W, C, Ho, Wo, dx);
    ctx->count(1);
  }
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  return DDPPO_OK;
}

namespace {
__global__ void positive_mask_kernel(const float* __restrict__ z, size_t n, uint8_t* __restrict__ out) {
  pdl_enter();
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    out[i] = z[i] > 0.f ? 1 : 0;
}
}  // namespace

// The forward's discrete decisions (every ReLU mask and the max-pool argmax), from the workspace of
// the last ddppo_policy_fwd on `batch`, in the order documented in include/ddppo.h.
extern "C" ddppo_status ddppo_debug_depth_decisions(ddppo_ctx* ctx, const ddppo_model_desc* host_desc,
                                                    const ddppo_batch* host_batch, void* ws, uint8_t* out, int64_t cap,
                                                    int64_t* host_n, void* stream) {
  if (!ctx || !host_batch || !host_desc) return DDPPO_ERR_CONFIG;
  ModelLayout L;
  DDPPO_REQUIRE(ctx, build_layout(host_desc, &L) == DDPPO_OK &&
                         arch_visual(host_desc->arch),
                "depth decisions: visual agents only");
  Plan P;
  make_plan(L, host_desc->arch != DDPPO_ARCH_DEPTH_R18_LSTM, host_batch->B, host_batch->T_run, ws, &P);
  const int F = P.F;
  std::vector<std::pair<const float*, size_t>> masks;  // (tensor, size); the pool argmax is copied after the first
  auto add = [&](const ConvGN& c) { masks.push_back({c.z, (size_t)F * c.Ho * c.Wo * c.Co}); };
  add(P.convs[0]);
  const size_t pool_n = (size_t)F * P.pool_hw * P.pool_hw * 32;
  for (const auto& blk : P.blocks) {
    for (size_t j = 0; j + 1 < blk.main.size(); ++j) add(P.convs[blk.main[j]]);  // the branch's inner ReLUs
    const ConvGN& last = P.convs[blk.main.back()];
    masks.push_back({blk.out, (size_t)F * last.Ho * last.Wo * last.Co});  // the block output's ReLU
  }
  add(P.convs.back());
  masks.push_back({P.vis, (size_t)F * 512});
  int64_t total = (int64_t)pool_n;
  for (auto& m : masks) total += (int64_t)m.second;
  if (host_n) *host_n = total;
  if (!out) return DDPPO_OK;
  DDPPO_REQUIRE(ctx, cap >= total, "depth decisions: buffer too small");
  cudaStream_t st = as_stream(stream);
  size_t off = 0;
  for (size_t i = 0; i < masks.size(); ++i) {
    launch_k(ctx, positive_mask_kernel, blocks_for(ctx, masks[i].second), kThreads, 0, st, masks[i].first,
             masks[i].second,
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
