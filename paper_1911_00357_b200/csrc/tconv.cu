// TMA-fed, warp-specialised, persistent tcgen05 implicit-GEMM convolution (a5 / a7 for the visual
// agents' encoders, P:L212 / P:L582-584; BASELINE.json north_star: "Encoder ... GEMMs use
// tcgen05/TMEM tiles fed by TMA").
//
//   FPROP  y[q][o]        = sum_{(u,v,c)} x[q @ (u,v)][c] Wr[o][(u,v,c)]        q = output pixel
//   DGRAD  dx[q][c]       = sum_{(u,v,o)} dy[q @ (k-1-u,k-1-v)][o] Wd[c][(u,v,o)]  (stride-1 convs)
//   WGRAD  dWt[(u,v,c)][o] = sum_q x[q @ (u,v)][c] dy[q][o]
//
// The im2col matrix never exists: the A operand of FPROP / DGRAD (pixels x channels, K-major) and
// of WGRAD (channels x pixels, MN-major) is loaded by the TMA unit in im2col mode
// (cp.async.bulk.tensor.4d.im2col) straight from the NHWC bf16 activation: a box of 128
// consecutive output pixels (walking W, then H, then frames) x CS channels of one filter tap, the
// tap given as the instruction's im2col offsets, padding and ragged tails zero-filled by the TMA
// unit.  Weights (FPROP / DGRAD B) and dy (WGRAD B) are plain 2-D tiled TMA boxes.  Swizzle
// 64 B (CS = 32) or 128 B (CS = 64) on both sides, matching the UMMA descriptors.
//
// CTA = 6 warps, persistent over a static list of (tile, split) work items:
//   warp 0     TMA producer (one elected lane): stage ring of STAGES {A, B} boxes, full/empty mbarriers
//   warp 1     MMA issuer: tcgen05.mma.kind::f16 (M = 128, N = BN, K = 16) into one of two TMEM
//              accumulators, tcgen05.commit -> empty[stage] (slot reuse) and -> tmem_full[acc]
//   warps 2-5  epilogue: tcgen05.ld (each warp its TMEM lane quarter), fp32 rows to global (or a
//              split-K partial), then tmem_empty[acc] -- so tile i's epilogue overlaps tile i+1's
//              main loop.
// Precision: NPL = 1 (bf16 operands) or 2 (x = hi + lo bf16 planes, products lo*hi + hi*lo +
// hi*hi, ~16-bit mantissas; the Depth forward decides ReLU / max-pool masks with it).
#include <cuda.h>
#include <string.h>

#include <algorithm>

#include "common.cuh"

namespace {

constexpr int kBM = 128;         // output rows per tile (TMEM lanes)
constexpr int kPix = 128;        // pixels per im2col box (FPROP rows / WGRAD k-chunk)
constexpr int kThreadsTC = 192;  // producer warp, MMA warp, 4 epilogue warps
enum { TC_FWD = 0, TC_WGRAD = 1 };

__device__ __forceinline__ uint32_t s_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra W_%=;\n}\n" ::"r"(s_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mb_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s_u32(b)) : "memory");
}
__device__ __forceinline__ void tma_im2col(uint32_t dst, const CUtensorMap* map, uint64_t* bar, int c, int w, int h,
                                           int n, uint16_t ow, uint16_t oh) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
      "[%2], {%7, %8};" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(s_u32(bar)), "r"(c), "r"(w), "r"(h), "r"(n), "h"(ow), "h"(oh)
      : "memory");
}
__device__ __forceinline__ void tma_2d(uint32_t dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(s_u32(bar)), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ bool elect_one() {
  uint32_t p = 0;
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\nselp.u32 %0, 1, 0, e;\n}\n"
      : "=r"(p));
  return p != 0;
}
// UMMA shared-memory descriptor (sm100): start, LBO, SBO (bytes), layout 2 = SW128, 4 = SW64
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)layout << 61);
}
template <int BYTES_ROW>
__host__ __device__ constexpr uint32_t swz_layout() { return BYTES_ROW == 128 ? 2u : 4u; }
__device__ __forceinline__ void mma_f16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_commit1(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s_u32(bar))
               : "memory");
}

struct TcArgs {
  int M, N;               // output rows / columns
  int n_k, kper;          // k-iterations (FPROP/DGRAD: taps x channel slices; WGRAD: pixel chunks), per split
  int tiles_m, tiles_n, n_work;
  int Ho, Wo, s, p, k;    // im2col traversal geometry (output pixel grid of the box walk)
  int F;                  // frames (WGRAD: the reduction runs over F * Ho * Wo pixels)
  int C, nsl;             // channels of the im2col'd tensor, C / CS
  // FPROP / DGRAD tap lists: phase q (nphase > 1: the 4 output phases of a stride-2 input gradient)
  // runs ntap[q] taps; tap i multiplies weight column block uv[q][i] (of k*k) with the im2col box at
  // offset (oh, ow)[q][i]; phase q's output rows land on pixels (2i + rh[q], 2j + rw[q]) of the
  // OH x OW output (scatter), else on row q of the grid
  int nphase, scatter, OH, OW;
  int8_t ntap[4], rh[4], rw[4];
  int8_t uv[4][9], oh[4][9], ow[4][9];
  float* out;             // result: [M][ldc] rows (FPROP / DGRAD), or the weight gradient (wg)
  long long ldc;
  int accumulate;         // out (+)= (FPROP / DGRAD)
  int splits;             // > 1: partial tiles in part[z][M][N]; the last split of a tile sums them
  float* part;
  int* cnt;               // per-tile arrival counters (zero; reset by the last arrival)
  int wg, Cr;             // WGRAD: write out[o][c < Cr][tap] (PyTorch order; rows are (tap, c < C))
  int groups;             // WGRAD of a grouped conv: keep the block-diagonal entries, out[o][c % (C/g)][tap]
  int trace;              // debug build (DDPPO_TCONV_TRACE): this launch's slot in the phase trace
  // FPROP / DGRAD: out = result + (res_mask > 0 ? res : 0) (a residual block's ReLU-masked shortcut
  // gradient added in the epilogue; res == nullptr: off)
  const float *res, *res_mask;
};

// Debug-build phase trace (compiled out of the product library): %globaltimer stamps per CTA --
// 0 entry, 1 prologue done, 2 past griddepcontrol.wait, 3 producer issued its last TMA, 4 first
// accumulator ready (epilogue warp 2), 5 epilogue done, 6 exit.
#ifdef DDPPO_TCONV_TRACE
constexpr int kTcTraceLaunches = 1024, kTcTraceCtas = 160;
__device__ unsigned long long g_tc_trace[kTcTraceLaunches][kTcTraceCtas][8];
long long g_tc_meta[kTcTraceLaunches][16];
int g_tc_next = 0;
#define TC_STAMP(cond, k)                                                                          \
  if ((cond) && a.trace < kTcTraceLaunches && blockIdx.x < kTcTraceCtas) {                         \
    unsigned long long t_;                                                                         \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                         \
    g_tc_trace[a.trace][blockIdx.x][k] = t_;                                                       \
  }
#else
#define TC_STAMP(cond, k)
#endif

// first output pixel q -> im2col box coordinates (W, H, N) of its receptive field's corner
__device__ __forceinline__ void pix_coords(const TcArgs& a, int q, int& w, int& h, int& n) {
  const int hw = a.Ho * a.Wo;
  n = q / hw;
  const int r = q - n * hw;
  const int oh = r / a.Wo;
  h = oh * a.s - a.p;
  w = (r - oh * a.Wo) * a.s - a.p;
}

// 8 consecutive output columns of one row: rows of out (FPROP / DGRAD, optionally accumulated), or
// the weight gradient in PyTorch order out[o][c][tap] for row = tap * C + c (c < Cr)
__device__ __forceinline__ void store_final(const TcArgs& a, int row, int col, const float (&v)[8]) {
  if (!a.wg) {
    float4* o = reinterpret_cast<float4*>(a.out + (long long)row * a.ldc + col);
    float4 v0 = make_float4(v[0], v[1], v[2], v[3]), v1 = make_float4(v[4], v[5], v[6], v[7]);
    if (a.res) {
      const long long o8 = (long long)row * a.ldc + col;
      const float4 r0 = *reinterpret_cast<const float4*>(a.res + o8), r1 = *reinterpret_cast<const float4*>(a.res + o8 + 4);
      const float4 m0 = *reinterpret_cast<const float4*>(a.res_mask + o8),
                   m1 = *reinterpret_cast<const float4*>(a.res_mask + o8 + 4);
      v0.x += m0.x > 0.f ? r0.x : 0.f; v0.y += m0.y > 0.f ? r0.y : 0.f;
      v0.z += m0.z > 0.f ? r0.z : 0.f; v0.w += m0.w > 0.f ? r0.w : 0.f;
      v1.x += m1.x > 0.f ? r1.x : 0.f; v1.y += m1.y > 0.f ? r1.y : 0.f;
      v1.z += m1.z > 0.f ? r1.z : 0.f; v1.w += m1.w > 0.f ? r1.w : 0.f;
    } else if (a.accumulate) {
      const float4 p0 = o[0], p1 = o[1];
      v0.x += p0.x; v0.y += p0.y; v0.z += p0.z; v0.w += p0.w;
      v1.x += p1.x; v1.y += p1.y; v1.z += p1.z; v1.w += p1.w;
    }
    o[0] = v0;
    o[1] = v1;
  } else {
    const int kk = a.k * a.k, tap = row / a.C, c = row - tap * a.C;
    if (c >= a.Cr) return;
    if (a.groups > 1) {
      const int cgi = a.C / a.groups, cgo = a.N / a.groups;
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (c / cgi == (col + e) / cgo) a.out[((long long)(col + e) * cgi + c % cgi) * kk + tap] = v[e];
      return;
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) a.out[((long long)(col + e) * a.Cr + c) * kk + tap] = v[e];
  }
}

template <int CS, int BN, int NPL, int MODE, int STAGES>
struct TcCfg {
  static constexpr int kRowB = CS * 2;                                        // A (FPROP) / K-row bytes
  static constexpr uint32_t kABox = kPix * CS * 2;                            // one im2col box
  static constexpr uint32_t kA = MODE == TC_FWD ? kABox : kBM * kPix * 2;     // A tile (WGRAD: 128/CS boxes)
  static constexpr uint32_t kB = MODE == TC_FWD ? BN * CS * 2 : kPix * BN * 2;
  static constexpr uint32_t kStage = NPL * (kA + kB);
  static constexpr int kTmemCols = 2 * BN <= 32 ? 32 : 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128 : 256;
  static constexpr size_t kSmem = (size_t)STAGES * kStage + 1024;
};

template <int CS, int BN, int NPL, int MODE, int STAGES>
__global__ void __launch_bounds__(kThreadsTC, 1)
tconv_kernel(const __grid_constant__ CUtensorMap mA0, const __grid_constant__ CUtensorMap mA1,
             const __grid_constant__ CUtensorMap mB0, const __grid_constant__ CUtensorMap mB1, const TcArgs a) {
  using Cfg = TcCfg<CS, BN, NPL, MODE, STAGES>;
  TC_STAMP(threadIdx.x == 0, 0);
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024 - (s_u32(smem_raw) & 1023)) & 1023);
  __shared__ uint64_t full[STAGES], empty[STAGES], tfull[2], tempty[2];
  __shared__ uint32_t tmem_slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mb_init(&full[s], 1);
      mb_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mb_init(&tfull[i], 1);
      mb_init(&tempty[i], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mA0)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mB0)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s_u32(&tmem_slot)),
                 "n"(Cfg::kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;
  const int tiles = a.tiles_m * a.tiles_n * max(1, a.nphase);
  TC_STAMP(threadIdx.x == 0, 1);
  // PDL: barriers, TMEM and the tensor-map prefetch above overlap the predecessor's tail; nothing it
  // writes is read before this point
  pdl_enter();
  TC_STAMP(threadIdx.x == 0, 2);

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (elect_one()) {
      int stage = 0;
      uint32_t ph = 0;
      for (int wi = blockIdx.x; wi < a.n_work; wi += gridDim.x) {
        const int z = wi / tiles, t = wi - z * tiles;
        const int q = t / (a.tiles_m * a.tiles_n), tq = t - q * a.tiles_m * a.tiles_n;
        const int m0 = (tq % a.tiles_m) * kBM, n0 = (tq / a.tiles_m) * BN;
        const int nk = MODE == TC_FWD ? a.ntap[q] * a.nsl : a.n_k;
        const int k0 = z * a.kper, k1 = min(nk, k0 + a.kper);
        int w = 0, h = 0, n = 0;
        if (MODE == TC_FWD) pix_coords(a, m0, w, h, n);
        for (int it = k0; it < k1; ++it) {
          mb_wait(&empty[stage], ph ^ 1u);
          mb_expect_tx(&full[stage], Cfg::kStage);
          const uint32_t sA = s_u32(smem + stage * Cfg::kStage), sB = sA + NPL * Cfg::kA;
          if constexpr (MODE == TC_FWD) {
            const int tap = it / a.nsl, sl = it - tap * a.nsl;
            const int col = a.uv[q][tap] * a.C + sl * CS;
            const uint16_t ow = (uint16_t)a.ow[q][tap], oh = (uint16_t)a.oh[q][tap];
            tma_im2col(sA, &mA0, &full[stage], sl * CS, w, h, n, ow, oh);
            tma_2d(sB, &mB0, &full[stage], col, n0);
            if constexpr (NPL == 2) {
              tma_im2col(sA + Cfg::kA, &mA1, &full[stage], sl * CS, w, h, n, ow, oh);
              tma_2d(sB + Cfg::kB, &mB1, &full[stage], col, n0);
            }
          } else {
            // k-chunk = pixels [it*128, +128); A = 128/CS boxes of (tap, channel slice) rows of this M-block
            pix_coords(a, it * kPix, w, h, n);
            const int taps = a.k * a.k;
#pragma unroll
            for (int b = 0; b < kBM / CS; ++b) {
              const int row0 = m0 + b * CS;
              int tap = row0 / a.C;
              const int c0 = row0 - tap * a.C;
              tap = min(tap, taps - 1);  // rows past the last tap: any valid box (masked in the epilogue)
              const int u = tap / a.k, v = tap - u * a.k;
              tma_im2col(sA + b * Cfg::kABox, &mA0, &full[stage], c0, w, h, n, (uint16_t)v, (uint16_t)u);
            }
            tma_2d(sB, &mB0, &full[stage], n0, it * kPix);
          }
          if (++stage == STAGES) {
            stage = 0;
            ph ^= 1u;
          }
        }
      }
      TC_STAMP(true, 3);
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(MODE == TC_WGRAD) << 15) |
                               ((uint32_t)(MODE == TC_WGRAD) << 16) | ((uint32_t)(BN >> 3) << 17) |
                               ((uint32_t)(kBM >> 4) << 24);
    int stage = 0, acc = 0;
    uint32_t ph = 0, aph = 0;
    for (int wi = blockIdx.x; wi < a.n_work; wi += gridDim.x) {
      const int z = wi / tiles, t = wi - z * tiles;
      const int q = t / (a.tiles_m * a.tiles_n);
      const int nk = MODE == TC_FWD ? a.ntap[q] * a.nsl : a.n_k;
      const int k0 = z * a.kper, k1 = min(nk, k0 + a.kper);
      mb_wait(&tempty[acc], aph ^ 1u);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t d = tmem + (uint32_t)(acc * BN);
      for (int it = k0; it < k1; ++it) {
        mb_wait(&full[stage], ph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (elect_one()) {
          const uint32_t sA = s_u32(smem + stage * Cfg::kStage), sB = sA + NPL * Cfg::kA;
          if constexpr (MODE == TC_FWD) {
            constexpr uint32_t L = swz_layout<CS * 2>(), SBO = 8 * CS * 2;
#pragma unroll
            for (int kk = 0; kk < CS / 16; ++kk) {
#pragma unroll
              for (int t = 0; t < (NPL == 2 ? 3 : 1); ++t) {  // NPL == 2: lo*hi, hi*lo, hi*hi
                const uint32_t ao = (NPL == 2 && t == 0) ? Cfg::kA : 0u, bo = (NPL == 2 && t == 1) ? Cfg::kB : 0u;
                const uint64_t ad = sdesc(sA + ao + kk * 32, 16, SBO, L), bd = sdesc(sB + bo + kk * 32, 16, SBO, L);
                mma_f16(d, ad, bd, idesc, (it > k0 || kk > 0 || t > 0) ? 1u : 0u);
              }
            }
          } else {
            constexpr uint32_t LA = swz_layout<CS * 2>(), LB = swz_layout<BN * 2>();
#pragma unroll
            for (int kk = 0; kk < kPix / 16; ++kk) {
              const uint64_t ad = sdesc(sA + kk * 16 * CS * 2, Cfg::kABox, 8 * CS * 2, LA);
              const uint64_t bd = sdesc(sB + kk * 16 * BN * 2, Cfg::kB, 8 * BN * 2, LB);
              mma_f16(d, ad, bd, idesc, (it > k0 || kk > 0) ? 1u : 0u);
            }
          }
          mma_commit1(&empty[stage]);  // frees the slot once these MMAs have read it
        }
        __syncwarp();
        if (++stage == STAGES) {
          stage = 0;
          ph ^= 1u;
        }
      }
      if (elect_one()) mma_commit1(&tfull[acc]);
      __syncwarp();
      if (++acc == 2) {
        acc = 0;
        aph ^= 1u;
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (TMEM -> global)
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int et = threadIdx.x - 64;  // 0..127
    int acc = 0;
    uint32_t aph = 0;
    for (int wi = blockIdx.x; wi < a.n_work; wi += gridDim.x) {
      const int z = wi / tiles, t = wi - z * tiles;
      const int ph = t / (a.tiles_m * a.tiles_n), tq = t - ph * a.tiles_m * a.tiles_n;
      const int m0 = (tq % a.tiles_m) * kBM, n0 = (tq / a.tiles_m) * BN;
      int row = m0 + q * 32 + lane;
      bool rok = row < a.M;
      if (a.scatter && rok) {  // phase grid position -> output pixel (2i + rh, 2j + rw)
        const int hw = a.Ho * a.Wo, f = row / hw, r = row - f * hw, i = r / a.Wo, j = r - i * a.Wo;
        const int y = 2 * i + a.rh[ph], x = 2 * j + a.rw[ph];
        rok = y < a.OH && x < a.OW;
        row = (f * a.OH + y) * a.OW + x;
      }
      mb_wait(&tfull[acc], aph);
      TC_STAMP(et == 0 && wi == (int)blockIdx.x, 4);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      float* prow = a.splits > 1 ? a.part + ((long long)z * a.M + row) * a.N + n0 : nullptr;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 8) {
        uint32_t r[8];
        const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + c0);
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                     : "r"(ta));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (rok && n0 + c0 < a.N) {
          float v[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) v[e] = __uint_as_float(r[e]);
          if (prow) {  // this split's partial tile
            reinterpret_cast<float4*>(prow + c0)[0] = make_float4(v[0], v[1], v[2], v[3]);
            reinterpret_cast<float4*>(prow + c0)[1] = make_float4(v[4], v[5], v[6], v[7]);
          } else {
            store_final(a, row, n0 + c0, v);
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mb_arrive(&tempty[acc]);  // the accumulator is free for the MMA warp's next tile
      if (++acc == 2) {
        acc = 0;
        aph ^= 1u;
      }
      if (a.splits > 1) {
        // distributed split-K fixup: every work item is resident (n_work <= grid, one item per CTA),
        // so the S splits of a tile wait for one another, then split z adds rows
        // [z*128/S, (z+1)*128/S) of the S partial tiles in split order (deterministic) and writes them
        int* cnt = a.cnt + 2 * t;
        __threadfence();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (et == 0) {
          atomicAdd(cnt, 1);
          while (ld_acquire_gpu(cnt) < a.splits) {
          }
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        const int r0 = z * kBM / a.splits, r1 = (z + 1) * kBM / a.splits;
        const int cpr = BN / 8;  // 8-column chunks per row
        for (int i = et; i < (r1 - r0) * cpr; i += 128) {
          const int rr = m0 + r0 + i / cpr, c0 = (i % cpr) * 8;
          if (rr >= a.M || n0 + c0 >= a.N) continue;
          float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
          const float* pr = a.part + (long long)rr * a.N + n0 + c0;
          for (int zz = 0; zz < a.splits; ++zz) {
            const float4 p0 = __ldcg(reinterpret_cast<const float4*>(pr + (long long)zz * a.M * a.N));
            const float4 p1 = __ldcg(reinterpret_cast<const float4*>(pr + (long long)zz * a.M * a.N) + 1);
            v[0] += p0.x; v[1] += p0.y; v[2] += p0.z; v[3] += p0.w;
            v[4] += p1.x; v[5] += p1.y; v[6] += p1.z; v[7] += p1.w;
          }
          store_final(a, rr, n0 + c0, v);
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        // the last split to finish resets the tile's counters for the next launch
        if (et == 0 && atomicAdd(cnt + 1, 1) == a.splits - 1) {
          cnt[0] = 0;
          cnt[1] = 0;
        }
      }
    }
  }
  TC_STAMP(threadIdx.x == 64, 5);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(Cfg::kTmemCols) : "memory");
  TC_STAMP(threadIdx.x == 0, 6);
}

// ---------------------------------------------------------------- host: tensor maps
typedef CUresult (*EncIm2colFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t, const cuuint32_t*,
                                CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                CUtensorMapFloatOOBfill);
typedef CUresult (*EncTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                               const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                               CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <typename F>
ddppo_status driver_fn(ddppo_ctx* ctx, const char* name, F* out) {
  if (*out) return DDPPO_OK;
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  DDPPO_CUDA_TRY(ctx, cudaGetDriverEntryPoint(name, &f, cudaEnableDefault, &q));
  DDPPO_REQUIRE(ctx, f != nullptr && q == cudaDriverEntryPointSuccess, "tconv: driver entry point unavailable");
  *out = reinterpret_cast<F>(f);
  return DDPPO_OK;
}

CUtensorMapSwizzle swz_for(int row_bytes) {
  return row_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : row_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                                         : CU_TENSOR_MAP_SWIZZLE_32B;
}

// im2col view of x[F][H][W][C] (bf16) for a k x k / stride s / pad p window: boxes of 128 output
// pixels x cs channels
ddppo_status map_im2col(ddppo_ctx* ctx, CUtensorMap* m, const __nv_bfloat16* x, int F, int H, int W, int C, int k,
                        int s, int p, int cs, bool corners = false, int lo_c = 0, int up_c = 0) {
  static EncIm2colFn enc = nullptr;
  ddppo_status st = driver_fn(ctx, "cuTensorMapEncodeIm2col", &enc);
  if (st != DDPPO_OK) return st;
  const cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)F};
  const cuuint64_t strides[3] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2};
  // traversal box: the k x k / pad p window, or explicit corners (the stride-2 input gradient's phases)
  const int lower[2] = {corners ? lo_c : -p, corners ? lo_c : -p};
  const int upper[2] = {corners ? up_c : p - (k - 1), corners ? up_c : p - (k - 1)};
  const cuuint32_t estr[4] = {1, (cuuint32_t)s, (cuuint32_t)s, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<__nv_bfloat16*>(x), dims, strides, lower, upper,
                   (cuuint32_t)cs, (cuuint32_t)kPix, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz_for(cs * 2),
                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  DDPPO_REQUIRE(ctx, r == CUDA_SUCCESS, "tconv: cuTensorMapEncodeIm2col rejected the geometry");
  return DDPPO_OK;
}
// 2-D tiles of a row-major [rows][cols] bf16 matrix: boxes of box_rows x box_cols
ddppo_status map_2d(ddppo_ctx* ctx, CUtensorMap* m, const __nv_bfloat16* x, int64_t rows, int64_t cols, int box_cols,
                    int box_rows) {
  static EncTiledFn enc = nullptr;
  ddppo_status st = driver_fn(ctx, "cuTensorMapEncodeTiled", &enc);
  if (st != DDPPO_OK) return st;
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  const cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<__nv_bfloat16*>(x), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, swz_for(box_cols * 2), CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  DDPPO_REQUIRE(ctx, r == CUDA_SUCCESS, "tconv: cuTensorMapEncodeTiled rejected the matrix");
  return DDPPO_OK;
}

template <int CS, int BN, int NPL, int MODE>
ddppo_status run(ddppo_ctx* ctx, const CUtensorMap (&maps)[4], TcArgs a, int min_iters, int max_splits, int slot,
                 cudaStream_t st) {
  constexpr uint32_t kStage = TcCfg<CS, BN, NPL, MODE, 1>::kStage;
  constexpr int STAGES = (int)std::min<uint32_t>(8u, (200u * 1024u) / kStage);
  static_assert(STAGES >= 2, "stage too large");
  using Cfg = TcCfg<CS, BN, NPL, MODE, STAGES>;
  auto kern = tconv_kernel<CS, BN, NPL, MODE, STAGES>;
  static bool attr = false;
  if (!attr) {
    DDPPO_CUDA_TRY(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::kSmem));
    attr = true;
  }
  const int per_sm = std::max(1, (int)((227u * 1024u) / (Cfg::kSmem + 2048)));
  // slot 1 = the side stream (weight gradients beside the critical path): at most a quarter of the SMs
  // (measured: 1/2 -1 %, 1/6 -1.4 %, 1/8 -4 %)
  static const int side_div = getenv("DDPPO_TCONV_SIDEDIV") ? atoi(getenv("DDPPO_TCONV_SIDEDIV")) : 4;  // A/B knob
  // (measured: leaving the side stream's SMs free for critical-path grids while it runs -- the
  // phase trace shows their last CTAs starting up to 15 us late -- is 0.3 % / 1.3 % slower on Depth /
  // RGB-D: the fuller grids win)
  const int cap = slot == 0 ? ctx->sm_count * std::min(per_sm, 2) : std::max(1, ctx->sm_count / side_div);
  // split-K over the k-iterations: ~one work item per resident CTA, each >= min_iters iterations; the
  // split tiles' fixup needs every work item resident at once (n_work <= grid)
  const int tiles = a.tiles_m * a.tiles_n * std::max(1, (int)a.nphase);
  int splits = 1;
  static const int min_it_f = getenv("DDPPO_TCONV_MINIT_F") ? atoi(getenv("DDPPO_TCONV_MINIT_F")) : 0;
  static const int min_it_w = getenv("DDPPO_TCONV_MINIT_W") ? atoi(getenv("DDPPO_TCONV_MINIT_W")) : 0;
  if (MODE == TC_FWD && min_it_f > 0) min_iters = min_it_f;  // A/B knobs
  if (MODE == TC_WGRAD && min_it_w > 0) min_iters = min_it_w;
  if (max_splits > 1 && tiles < cap && a.nphase <= 1)
    splits = std::max(1, std::min({cap / tiles, a.n_k / std::max(1, min_iters), max_splits}));
  DDPPO_REQUIRE(ctx, a.n_k >= 1, "tconv: empty reduction");
  a.kper = (a.n_k + splits - 1) / splits;
  splits = (a.n_k + a.kper - 1) / a.kper;
  a.splits = splits;
  a.n_work = tiles * splits;
  DDPPO_REQUIRE(ctx, splits == 1 || (2 * tiles <= kMaxTileCounters / 2 && a.part), "tconv: split-K needs scratch");
  const int grid = std::max(1, std::min(a.n_work, cap));
  ProfScope ps(ctx, DDPPO_K_CONV, st, 1);
  if (ctx->prof) {
    double taps = 0;
    for (int q = 0; q < std::max(1, (int)a.nphase); ++q) taps += a.ntap[q];
    ctx->flops[DDPPO_K_CONV] += 2.0 * a.M * a.N * (MODE == TC_FWD ? taps * a.C : (double)a.Ho * a.Wo * a.F);
    // shared-memory traffic: every k-iteration of every tile (splits partition the iterations) has
    // the TMA write its stage and the MMAs read A (128 x 16) and B (BN x 16) bf16 per K = 16 step, once
    // per product (bf16x3: 3)
    const double iters = (double)a.tiles_m * a.tiles_n * (MODE == TC_FWD ? taps * a.nsl : (double)a.n_k);
    const double k16 = MODE == TC_FWD ? CS / 16 : kPix / 16, prods = NPL == 2 ? 3 : 1;
    ctx->smem_bytes[DDPPO_K_CONV] += iters * (Cfg::kStage + k16 * prods * (kBM * 16 * 2 + BN * 16 * 2));
  }
#ifdef DDPPO_TCONV_TRACE
  {
    const int next = g_tc_next++;
    a.trace = next;
    if (next < kTcTraceLaunches) {
      long long* m = g_tc_meta[next];
      m[0] = MODE; m[1] = CS; m[2] = BN; m[3] = NPL; m[4] = a.M; m[5] = a.N; m[6] = a.n_k; m[7] = a.kper;
      m[8] = a.n_work; m[9] = grid; m[10] = slot; m[11] = splits;
    }
  }
#else
  a.trace = 0;
#endif
  launch_k(ctx, kern, grid, kThreadsTC, Cfg::kSmem, st, maps[0], maps[1], maps[2], maps[3], a);
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  return DDPPO_OK;
}

}  // namespace

#ifdef DDPPO_TCONV_TRACE
extern "C" int ddppo_debug_tconv_trace(unsigned long long* host, long long* meta, int n) {
  memcpy(meta, g_tc_meta, sizeof(long long) * 16 * (size_t)std::min(n, kTcTraceLaunches));
  return (int)cudaMemcpyFromSymbol(host, g_tc_trace, sizeof(unsigned long long) * kTcTraceCtas * 8 *
                                                         (size_t)std::min(n, kTcTraceLaunches));
}
#endif

// N tile of FPROP / DGRAD (tiles_m = 128-row M tiles)
// (measured: RGB-D +0.9 %, Depth unchanged -- none of its layers has 148 128-wide tiles; 128 for
// every N >= 128: Depth -3 %, RGB-D +1.7 %)
static int bn_for(const ddppo_ctx* ctx, int N, int tiles_m) {
  if (N <= 32) return 32;
  if (N <= 64) return 64;
  if (!ctx->tconv_bn64) return 128;
  return (long long)tiles_m * ((N + 127) / 128) >= ctx->sm_count ? 128 : 64;
}

// FPROP (flip = 0) or stride-1 DGRAD (flip = 1) over x[F][H][W][C]:
//   out[q][o] (+)= sum_{tap, c} x[q @ tap][c] w[o][tap*C + c],  q over the F x Ho x Wo output grid.
// w: [N][k*k*C] bf16 (plane stride wplane elements when planes == 2; x likewise xplane).
// With `partial` (>= splits*M*N floats) and a long k loop the work is split over K; each tile's last
// split adds the partial tiles in split order and writes out (*splits_out = 1: nothing left to do).
ddppo_status launch_tconv_fwd(ddppo_ctx* ctx, const __nv_bfloat16* x, int64_t xplane, int F, int H, int W, int C,
                              int k, int s, int p, int flip, const __nv_bfloat16* w, int64_t wplane, int N, int planes,
                              float* out, int64_t ldc, int accumulate, float* partial, int max_splits, int slot,
                              int* splits_out, cudaStream_t st, const float* res, const float* res_mask) {
  DDPPO_REQUIRE(ctx, C % 32 == 0 && N % 8 == 0 && ldc % 4 == 0, "tconv: C % 32 == 0, N % 8 == 0 required");
  DDPPO_REQUIRE(ctx, !res || (res_mask && !accumulate && ((uintptr_t)res & 15) == 0 && ((uintptr_t)res_mask & 15) == 0),
                "tconv: the masked residual needs 16-byte aligned res / res_mask and no accumulation");
  DDPPO_REQUIRE(ctx, !flip || s == 1, "tconv: transposed taps only for stride-1 convolutions");
  DDPPO_REQUIRE(ctx, k <= 3, "tconv: kernels up to 3x3 (tap lists)");
  DDPPO_REQUIRE(ctx, ((uintptr_t)x & 15) == 0 && ((uintptr_t)w & 15) == 0 && ((uintptr_t)out & 15) == 0,
                "tconv: 16-byte aligned operands required");
  const int Ho = (H + 2 * p - k) / s + 1, Wo = (W + 2 * p - k) / s + 1;
  const int cs = C % 64 == 0 ? 64 : 32;
  // N tile: 64 columns for the small-M deep layers (twice the tiles: less split-K, deeper rings);
  // 128 once 128-wide tiles alone fill a wave of the SMs (each A box then feeds twice the columns:
  // half the im2col re-reads) -- measured, DESIGN.md §7
  const int bn = bn_for(ctx, N, (F * Ho * Wo + kBM - 1) / kBM);
  TcArgs a = {};
  a.M = F * Ho * Wo;
  a.N = N;
  a.Ho = Ho;
  a.Wo = Wo;
  a.s = s;
  a.p = p;
  a.k = k;
  a.C = C;
  a.nsl = C / cs;
  a.nphase = 1;
  a.ntap[0] = (int8_t)(k * k);
  for (int u = 0; u < k; ++u)
    for (int v = 0; v < k; ++v) {
      a.uv[0][u * k + v] = (int8_t)(u * k + v);
      a.oh[0][u * k + v] = (int8_t)(flip ? k - 1 - u : u);
      a.ow[0][u * k + v] = (int8_t)(flip ? k - 1 - v : v);
    }
  a.n_k = k * k * a.nsl;
  a.tiles_m = (a.M + kBM - 1) / kBM;
  a.tiles_n = (N + bn - 1) / bn;
  if (!partial) max_splits = 1;
  a.out = out;
  a.ldc = ldc;
  a.part = partial;
  a.cnt = ctx->d_tile_cnt + (size_t)slot * (kMaxTileCounters / 2);
  a.accumulate = accumulate;
  a.res = res;
  a.res_mask = res_mask;
  if (splits_out) *splits_out = 1;  // the split sum happens inside the kernel
  CUtensorMap maps[4];
  memset(maps, 0, sizeof(maps));
  const int K = k * k * C;
  // im2col geometry of the box walk: FPROP walks x with the conv's own window; DGRAD walks dy with
  // the mirrored window (pad k-1-p), producing the input-resolution grid
  ddppo_status r = map_im2col(ctx, &maps[0], x, F, H, W, C, k, s, p, cs);
  if (r == DDPPO_OK && planes == 2) r = map_im2col(ctx, &maps[1], x + xplane, F, H, W, C, k, s, p, cs);
  if (r == DDPPO_OK) r = map_2d(ctx, &maps[2], w, N, K, cs, bn);
  if (r == DDPPO_OK && planes == 2) r = map_2d(ctx, &maps[3], w + wplane, N, K, cs, bn);
  if (r != DDPPO_OK) return r;
#define TC_CASE(CS_, BN_, NPL_) \
  if (cs == CS_ && bn == BN_ && planes == NPL_) return run<CS_, BN_, NPL_, TC_FWD>(ctx, maps, a, 4, max_splits, slot, st);
  TC_CASE(32, 32, 1) TC_CASE(32, 64, 1) TC_CASE(32, 128, 1) TC_CASE(64, 32, 1) TC_CASE(64, 64, 1)
  TC_CASE(64, 128, 1) TC_CASE(32, 32, 2) TC_CASE(32, 64, 2) TC_CASE(32, 128, 2) TC_CASE(64, 32, 2)
  TC_CASE(64, 64, 2) TC_CASE(64, 128, 2)
#undef TC_CASE
  DDPPO_REQUIRE(ctx, false, "tconv: no instantiation for this shape");
  return DDPPO_ERR_CONFIG;
}

// WGRAD: dw[o][c][u][v] (PyTorch order, c < Cr) = sum over the output pixels q of
//   x[q @ (u, v)][c] * dy[q][o]   (x [F][H][W][C] bf16, dy [F*Ho*Wo][N] bf16); split over pixels
// with partial tiles in `partial`, summed in split order by each tile's last split.
ddppo_status launch_tconv_wgrad(ddppo_ctx* ctx, const __nv_bfloat16* x, int F, int H, int W, int C, int k, int s,
                                int p, const __nv_bfloat16* dy, int N, float* dw, int Cr, float* partial, int max_splits,
                                int slot, int* splits_out, cudaStream_t st, int groups) {
  DDPPO_REQUIRE(ctx, C % 32 == 0 && N % 8 == 0, "tconv wgrad: C % 32 == 0, N % 8 == 0 required");
  DDPPO_REQUIRE(ctx, ((uintptr_t)x & 15) == 0 && ((uintptr_t)dy & 15) == 0 && ((uintptr_t)partial & 15) == 0,
                "tconv wgrad: 16-byte aligned operands required");
  const int Ho = (H + 2 * p - k) / s + 1, Wo = (W + 2 * p - k) / s + 1;
  const int cs = C % 64 == 0 ? 64 : 32;
  const int bn = N <= 32 ? 32 : 64;
  TcArgs a = {};
  a.M = k * k * C;
  a.N = N;
  a.Ho = Ho;
  a.Wo = Wo;
  a.s = s;
  a.p = p;
  a.k = k;
  a.C = C;
  a.nsl = C / cs;
  const int pix = F * Ho * Wo;
  a.F = F;
  a.n_k = (pix + kPix - 1) / kPix;
  a.tiles_m = (a.M + kBM - 1) / kBM;
  a.tiles_n = (N + bn - 1) / bn;
  a.out = dw;
  a.part = partial;
  a.cnt = ctx->d_tile_cnt + (size_t)slot * (kMaxTileCounters / 2);
  a.wg = 1;
  a.Cr = Cr;
  a.groups = groups;
  DDPPO_REQUIRE(ctx, groups >= 1 && C % groups == 0 && N % groups == 0, "tconv wgrad: bad group count");
  if (splits_out) *splits_out = 1;
  CUtensorMap maps[4];
  memset(maps, 0, sizeof(maps));
  ddppo_status r = map_im2col(ctx, &maps[0], x, F, H, W, C, k, s, p, cs);
  if (r == DDPPO_OK) r = map_2d(ctx, &maps[2], dy, pix, N, bn, kPix);
  if (r != DDPPO_OK) return r;
  if (cs == 32 && bn == 32) return run<32, 32, 1, TC_WGRAD>(ctx, maps, a, 32, max_splits, slot, st);
  if (cs == 32 && bn == 64) return run<32, 64, 1, TC_WGRAD>(ctx, maps, a, 32, max_splits, slot, st);
  if (cs == 64 && bn == 32) return run<64, 32, 1, TC_WGRAD>(ctx, maps, a, 32, max_splits, slot, st);
  return run<64, 64, 1, TC_WGRAD>(ctx, maps, a, 32, max_splits, slot, st);
}

// Input gradient of a stride-2 convolution (k <= 3) as one launch over its 4 output phases: dx pixel
// (2i + rh, 2j + rw) receives sum over the taps u, v with (rh + p - u), (rw + p - v) even of
// dy[i + (rh + p - u) / 2][j + (rw + p - v) / 2] Wd[c][(u, v, o)] -- a stride-1 tap subset per phase
// over dy's grid, the epilogue scattering each phase's rows onto its pixels.  dy [F][Ho][Wo][Co] bf16
// (hi / lo planes when planes == 2), Wd [Ci][k*k*Co]; dx [F][H][W][Ci] fp32 (+)=.
ddppo_status launch_tconv_dgrad_s2(ddppo_ctx* ctx, const __nv_bfloat16* dy, int64_t dy_plane, int F, int Ho, int Wo,
                                   int Co, int H, int W, int Ci, int k, int p, const __nv_bfloat16* wd,
                                   int64_t wd_plane, int planes, float* dx, int accumulate, cudaStream_t st) {
  DDPPO_REQUIRE(ctx, Co % 32 == 0 && Ci % 8 == 0 && k <= 3, "tconv dgrad s2: Co % 32 == 0, Ci % 8 == 0, k <= 3");
  DDPPO_REQUIRE(ctx, ((uintptr_t)dy & 15) == 0 && ((uintptr_t)wd & 15) == 0 && ((uintptr_t)dx & 15) == 0,
                "tconv dgrad s2: 16-byte aligned operands required");
  const int cs = Co % 64 == 0 ? 64 : 32;
  const int bn = bn_for(ctx, Ci, (F * Ho * Wo + kBM - 1) / kBM);
  TcArgs a = {};
  a.M = F * Ho * Wo;
  a.N = Ci;
  a.Ho = Ho;
  a.Wo = Wo;
  a.s = 1;
  a.p = 0;
  a.k = k;
  a.C = Co;
  a.nsl = Co / cs;
  a.nphase = 4;
  a.scatter = 1;
  a.OH = H;
  a.OW = W;
  bool empty_phase = false;
  for (int rh = 0; rh < 2; ++rh)
    for (int rw = 0; rw < 2; ++rw) {
      const int q = rh * 2 + rw;
      a.rh[q] = (int8_t)rh;
      a.rw[q] = (int8_t)rw;
      int n = 0;
      for (int u = 0; u < k; ++u)
        for (int v = 0; v < k; ++v) {
          if ((rh + p - u) % 2 || (rw + p - v) % 2) continue;
          const int oh = (rh + p - u) / 2, ow = (rw + p - v) / 2;
          DDPPO_REQUIRE(ctx, rh + p - u >= 0 && rw + p - v >= 0, "tconv dgrad s2: negative phase offset");
          a.uv[q][n] = (int8_t)(u * k + v);
          a.oh[q][n] = (int8_t)oh;
          a.ow[q][n] = (int8_t)ow;
          ++n;
        }
      a.ntap[q] = (int8_t)n;
      empty_phase = empty_phase || n == 0;
    }
  // phases without taps (a 1x1 stride-2 conv touches only the even pixels) must read 0: zero dx once
  if (empty_phase && !accumulate) {
    DDPPO_CUDA_TRY(ctx, cudaMemsetAsync(dx, 0, (size_t)F * H * W * Ci * sizeof(float), st));
    accumulate = 1;
  }
  // skip empty phases: pack the non-empty ones first (the epilogue reads rh / rw per phase)
  int np = 0;
  for (int q = 0; q < 4; ++q)
    if (a.ntap[q] > 0) {
      if (np != q) {
        a.ntap[np] = a.ntap[q];
        a.rh[np] = a.rh[q];
        a.rw[np] = a.rw[q];
        for (int i = 0; i < 9; ++i) {
          a.uv[np][i] = a.uv[q][i];
          a.oh[np][i] = a.oh[q][i];
          a.ow[np][i] = a.ow[q][i];
        }
      }
      ++np;
    }
  a.nphase = np;
  for (int q = 0; q < np; ++q) a.n_k = std::max(a.n_k, a.ntap[q] * a.nsl);  // (one split: kper = the longest)
  a.tiles_m = (a.M + kBM - 1) / kBM;
  a.tiles_n = (Ci + bn - 1) / bn;
  a.out = dx;
  a.ldc = Ci;
  a.accumulate = accumulate;
  a.cnt = ctx->d_tile_cnt;
  CUtensorMap maps[4];
  memset(maps, 0, sizeof(maps));
  const int K = k * k * Co;
  ddppo_status r = map_im2col(ctx, &maps[0], dy, F, Ho, Wo, Co, 1, 1, 0, cs, true, 0, 0);
  if (r == DDPPO_OK && planes == 2) r = map_im2col(ctx, &maps[1], dy + dy_plane, F, Ho, Wo, Co, 1, 1, 0, cs, true, 0, 0);
  if (r == DDPPO_OK) r = map_2d(ctx, &maps[2], wd, Ci, K, cs, bn);
  if (r == DDPPO_OK && planes == 2) r = map_2d(ctx, &maps[3], wd + wd_plane, Ci, K, cs, bn);
  if (r != DDPPO_OK) return r;
#define TC_CASE(CS_, BN_, NPL_) \
  if (cs == CS_ && bn == BN_ && planes == NPL_) return run<CS_, BN_, NPL_, TC_FWD>(ctx, maps, a, 1, 1, 0, st);
  TC_CASE(32, 32, 1) TC_CASE(32, 64, 1) TC_CASE(32, 128, 1) TC_CASE(64, 32, 1) TC_CASE(64, 64, 1)
  TC_CASE(64, 128, 1) TC_CASE(32, 32, 2) TC_CASE(32, 64, 2) TC_CASE(32, 128, 2) TC_CASE(64, 32, 2)
  TC_CASE(64, 64, 2) TC_CASE(64, 128, 2)
#undef TC_CASE
  DDPPO_REQUIRE(ctx, false, "tconv dgrad s2: no instantiation for this shape");
  return DDPPO_ERR_CONFIG;
}
