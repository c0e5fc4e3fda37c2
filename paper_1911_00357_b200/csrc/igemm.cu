// Implicit-GEMM tcgen05 kernel for the Depth encoder's convolutions (a5 / a7, configs[2]).
//
//   C[m][n] (+)= sum_k A(m, k) B(n, k)       fp32 accumulation in TMEM, fp32 C
//
// Operands are bf16 in HBM (activations / gradients / reordered weights are produced in that
// form by the kernels before), so every 16-byte piece of a tile is copied HBM -> shared memory by
// cp.async straight into its place in the UMMA canonical SWIZZLE_NONE layout: no fp32 staging,
// no conversion pass, zero-fill for padding / out-of-range.  Per operand one of four sources:
//   DENSE_K   X[r*ld + k]        (K-major: 8 consecutive k in 16 B)
//   DENSE_MN  X[k*ld + r]        (MN-major: 8 consecutive rows in 16 B)
//   PIX_K     conv gather, rows = pixels, k = (u, v, c)   (K-major; 8 channels in 16 B)
//   TAP_MN    conv gather, rows = (u, v, c), k = pixels   (MN-major; 8 channels in 16 B)
// Precision: NPL = 1 plane (bf16 operands) or 2 planes (x = hi + lo, both bf16; the product is
// hi*hi + hi*lo + lo*hi: ~16-bit-mantissa operands, used by the forward).
// Tile 128 x BN x 64, STAGES-deep cp.async ring; one thread issues the MMAs of a stage after a
// CTA barrier and commits them to the stage's mbarrier, which gates the stage's reuse.
#include <cuda_bf16.h>

#include <algorithm>

#include "common.cuh"

namespace {

constexpr int kBM = 128, kBK = 64, kThreads = 512;

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra W_%=;\n}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)layout << 61);
}
// Shared-memory tile layouts (tile = ROWS x 64 k of bf16, base 1024-byte aligned):
//  K-major, SWIZZLE_128B: row r is 128 contiguous bytes at r*128, its 16-byte chunk j (k 8j..8j+7)
//    stored at chunk j ^ (r & 7); descriptor LBO 16 (unused), SBO 1024 (8-row groups), k-step
//    advance +32 B on the start address.
//  MN-major, SWIZZLE_128B (ROWS >= 64): atom = 8 k-rows x 128 B (64 MN elements); chunk j of k-row
//    kr at j ^ kr; atom (MN block mb, k group kg) at mb*8192 + kg*1024 -> LBO 8192, SBO 1024,
//    k-step (16) advance +2048 B.
//  MN-major, no swizzle (ROWS < 64): 8 k x 16 B core matrices, k groups 128 B apart (LBO), 8-row
//    groups 1024 B apart (SBO), k-step advance +256 B.
constexpr uint32_t kSwz128 = 2, kSwzNone = 0;
template <int ROWS, bool MN>
__device__ __forceinline__ uint64_t tile_desc(uint32_t base, int kk) {
  if constexpr (!MN) return make_desc(base + kk * 32, 16, 1024, kSwz128);
  else if constexpr (ROWS >= 64) return make_desc(base + kk * 2048, 8192, 1024, kSwz128);
  else return make_desc(base + kk * 256, 128, 1024, kSwzNone);
}
// kind::f16, bf16 x bf16 -> f32, M = 128, N = n; a_mn / b_mn: operand is MN-major
__device__ __forceinline__ uint32_t make_idesc(int n, int a_mn, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(n >> 3) << 17) | ((uint32_t)(kBM >> 4) << 24);
}
// byte offset of the 16-byte piece holding (row, k) in an unswizzled MN-major [rows x 64] tile
__device__ __forceinline__ uint32_t off_mn(int row, int k) { return (row >> 3) * 1024 + (k >> 3) * 128 + (k & 7) * 16; }

// fast pixel / tap decomposition (power-of-two shifts when the host found them, else division)
__device__ __forceinline__ int3 ig_pixel(const IGather& g, int q) {
  int f, i, j;
  if (g.pw_log2 >= 0 && g.php_log2 >= 0) {
    f = q >> g.php_log2;
    const int rem = q & ((1 << g.php_log2) - 1);
    i = rem >> g.pw_log2;
    j = rem & ((1 << g.pw_log2) - 1);
  } else {
    const int php = g.PH * g.PW;
    f = q / php;
    const int rem = q - f * php;
    i = rem / g.PW;
    j = rem - i * g.PW;
  }
  return make_int3(f * g.SH, i, j);
}
__device__ __forceinline__ int3 ig_tap(const IGather& g, int kk) {
  int uv, c;
  if (g.sc_log2 >= 0) {
    uv = kk >> g.sc_log2;
    c = kk & ((1 << g.sc_log2) - 1);
  } else {
    uv = kk / g.SC;
    c = kk - uv * g.SC;
  }
  const int u = uv / g.k;
  return make_int3(u, uv - u * g.k, c);
}
template <bool TRANSPOSED>
__device__ __forceinline__ const __nv_bfloat16* ig_src(const IGather& g, int fSH, int i, int j, int u, int v, int c) {
  int y, xx;
  if (!TRANSPOSED) {
    y = i * g.s - g.p + u;
    xx = j * g.s - g.p + v;
  } else {
    const int ty = i + g.p - u, tx = j + g.p - v;
    if (ty < 0 || tx < 0) return nullptr;
    if (g.s == 1) {
      y = ty;
      xx = tx;
    } else {
      if (ty % g.s || tx % g.s) return nullptr;
      y = ty / g.s;
      xx = tx / g.s;
    }
  }
  if (y < 0 || y >= g.SH || xx < 0 || xx >= g.SW) return nullptr;
  return g.x + (((long long)(fSH + y) * g.SW + xx) * g.SC + c);
}

struct OpDev {
  int kind;          // IG_DENSE_K, IG_DENSE_MN, IG_PIX_K, IG_TAP_MN
  const __nv_bfloat16* x;
  long long ld;      // dense: leading dimension (elements)
  long long plane;   // elements between the hi and lo planes (NPL == 2)
  IGather g;         // gathers
  int rows;          // valid rows (M or N)
};

// one operand tile (ROWS x 64, NPL planes) of k-chunk [k0, k0+64) (global k = kg0 + k): cp.async.
// Piece p of the tile -> thread p % 128.  Consecutive threads take consecutive 16-byte pieces of
// one 128-byte core matrix (conflict-free shared-memory writes), and each warp covers 4
// neighbouring pieces along the contiguous HBM direction (full 32-byte sectors).
constexpr int IG_PIX_KT = 100;  // internal: PIX_K over transposed taps (input gradient)
template <int KIND>
__host__ __device__ constexpr bool kind_mn() { return KIND == IG_DENSE_MN || KIND == IG_TAP_MN; }

template <int ROWS, int NPL, int KIND>
__device__ __forceinline__ void load_tile(const OpDev& op, unsigned char* dst, uint32_t plane_bytes, int r0, int k0,
                                          int K, int kg0, const int4* rt) {
  const int tid = threadIdx.x;
  if constexpr (!kind_mn<KIND>()) {
    // K-major piece = 8 k of one row: p -> row p >> 3, chunk j = p & 7 (8 consecutive threads =
    // one row's 128 contiguous HBM bytes; the swizzle spreads them over all banks)
    const int kgp = tid & 7, k = k0 + 8 * kgp;
    const bool kok = k < K;
    int3 tap = make_int3(0, 0, 0);
    if (KIND != IG_DENSE_K && kok) tap = ig_tap(op.g, kg0 + k);
#pragma unroll
    for (int p = tid; p < ROWS * 8; p += kThreads) {
      const int row = p >> 3;
      const int r = r0 + row;
      const __nv_bfloat16* src = nullptr;
      if (kok) {
        if constexpr (KIND == IG_DENSE_K) {
          if (r < op.rows) src = op.x + (long long)r * op.ld + (kg0 + k);
        } else {
          const int4 pr = rt[row];
          if (pr.w) src = ig_src<KIND == IG_PIX_KT>(op.g, pr.x, pr.y, pr.z, tap.x, tap.y, tap.z);
        }
      }
      const uint32_t d = smem_addr(dst + row * 128 + ((kgp ^ (row & 7)) << 4));
#pragma unroll
      for (int pl = 0; pl < NPL; ++pl)
        cp_async16(d + pl * plane_bytes, src ? (const void*)(src + pl * op.plane) : (const void*)op.x, src ? 16u : 0u);
    }
  } else {
    if constexpr (ROWS >= 64) {
      // MN-major SWIZZLE_128B: p -> chunk j = p & 7 (8 rows), MN block mb, k: 8 consecutive threads
      // = 64 contiguous MN elements (128 HBM bytes) of one k
      constexpr int MB = ROWS / 64;
      const int j = tid & 7, mb = (tid >> 3) % MB;
      const int rgi = mb * 8 + j;  // 8-row group index
      const int r = r0 + 8 * rgi;
      int4 tr = make_int4(0, 0, 0, 0);
      if constexpr (KIND == IG_TAP_MN) tr = rt[8 * rgi];
#pragma unroll
      for (int p = tid; p < MB * 8 * kBK; p += kThreads) {
        const int kk = (p >> 3) / MB;
        const int k = k0 + kk;
        const __nv_bfloat16* src = nullptr;
        if (k < K) {
          if constexpr (KIND == IG_DENSE_MN) {
            if (r < op.rows) src = op.x + (long long)(kg0 + k) * op.ld + r;
          } else if (tr.w) {
            const int3 px = ig_pixel(op.g, kg0 + k);
            src = ig_src<false>(op.g, px.x, px.y, px.z, tr.x, tr.y, tr.z);
          }
        }
        const int kr = kk & 7;
        const uint32_t d = smem_addr(dst + mb * 8192 + (kk >> 3) * 1024 + kr * 128 + ((j ^ kr) << 4));
#pragma unroll
        for (int pl = 0; pl < NPL; ++pl)
          cp_async16(d + pl * plane_bytes, src ? (const void*)(src + pl * op.plane) : (const void*)op.x,
                     src ? 16u : 0u);
      }
    } else {
      // MN-major, no swizzle: p -> k (p >> 3) / RG * 8 + (p & 7), rowgroup (p >> 3) % RG
      constexpr int RG = ROWS / 8;
      const int rg = (tid >> 3) % RG;
      const int r = r0 + 8 * rg;
      int4 tr = make_int4(0, 0, 0, 0);
      if constexpr (KIND == IG_TAP_MN) tr = rt[8 * rg];
#pragma unroll
      for (int p = tid; p < RG * kBK; p += kThreads) {
        const int kk = ((p >> 3) / RG) * 8 + (p & 7);
        const int k = k0 + kk;
        const __nv_bfloat16* src = nullptr;
        if (k < K) {
          if constexpr (KIND == IG_DENSE_MN) {
            if (r < op.rows) src = op.x + (long long)(kg0 + k) * op.ld + r;
          } else if (tr.w) {
            const int3 px = ig_pixel(op.g, kg0 + k);
            src = ig_src<false>(op.g, px.x, px.y, px.z, tr.x, tr.y, tr.z);
          }
        }
        const uint32_t d = smem_addr(dst + off_mn(8 * rg, kk));
#pragma unroll
        for (int pl = 0; pl < NPL; ++pl)
          cp_async16(d + pl * plane_bytes, src ? (const void*)(src + pl * op.plane) : (const void*)op.x,
                     src ? 16u : 0u);
      }
    }
  }
}

template <int ROWS, int KIND>
__device__ __forceinline__ void fill_table(const OpDev& op, int r0, int4* rt) {
  for (int row = threadIdx.x; row < ROWS; row += kThreads) {
    const int r = r0 + row;
    const int ok = r < op.rows;
    if constexpr (KIND == IG_PIX_K || KIND == IG_PIX_KT) {
      const int3 px = ig_pixel(op.g, ok ? r : 0);
      rt[row] = make_int4(px.x, px.y, px.z, ok);
    } else if constexpr (KIND == IG_TAP_MN) {
      const int3 t = ig_tap(op.g, ok ? r : 0);
      rt[row] = make_int4(t.x, t.y, t.z, ok);
    }
  }
}

template <int BN, int NPL, int STAGES, int KA, int KB>
__global__ void __launch_bounds__(kThreads, 1)
igemm_kernel(const OpDev opA, const OpDev opB, float* __restrict__ C, long long ldc, int M, int N, int K, int kper,
             long long cz_stride, int accumulate) {
  constexpr uint32_t kAPlane = kBM * kBK * 2, kBPlane = BN * kBK * 2;
  constexpr uint32_t kStage = NPL * (kAPlane + kBPlane);
  constexpr int kTmemCols = BN < 32 ? 32 : BN;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // swizzled tiles need 1024-byte aligned bases (the launch adds 1 KB of slack)
  unsigned char* smem = smem_raw + ((1024 - (smem_addr(smem_raw) & 1023)) & 1023);
  __shared__ uint64_t mma_bar[STAGES];
  __shared__ uint32_t tmem_slot;
  __shared__ int4 rtA[kBM], rtB[BN];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.y * kBM, n0 = blockIdx.x * BN;
  const int kg0 = blockIdx.z * kper;
  K = min(kper, K - kg0);
  C += (long long)blockIdx.z * cz_stride;
  const int n_chunks = (K + kBK - 1) / kBK;

  fill_table<kBM, KA>(opA, m0, rtA);
  fill_table<BN, KB>(opB, n0, rtB);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&tmem_slot)),
                 "n"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&mma_bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;
  const uint32_t idesc = make_idesc(BN, kind_mn<KA>(), kind_mn<KB>());

  auto stage_ptr = [&](int s) { return smem + s * kStage; };
  // prologue: chunks 0 .. STAGES-2
#pragma unroll 1
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < n_chunks) {
      load_tile<kBM, NPL, KA>(opA, stage_ptr(s), kAPlane, m0, s * kBK, K, kg0, rtA);
      load_tile<BN, NPL, KB>(opB, stage_ptr(s) + NPL * kAPlane, kBPlane, n0, s * kBK, K, kg0, rtB);
    }
    cp_async_commit();
  }
  uint32_t phase_bits = 0;  // bit s: parity to wait for on mma_bar[s]
  for (int ch = 0; ch < n_chunks; ++ch) {
    const int s = ch % STAGES;
    cp_async_wait<STAGES - 2>();  // chunk ch has landed (this thread's copies)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();               // ... and every thread's
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t a0 = smem_addr(stage_ptr(s)), b0 = a0 + NPL * kAPlane;
#pragma unroll
      for (int kk = 0; kk < kBK / 16; ++kk) {
#pragma unroll
        for (int t = 0; t < (NPL == 2 ? 3 : 1); ++t) {
          // NPL == 2: lo*hi, hi*lo, then hi*hi
          const uint32_t ao = (NPL == 2 && t == 0) ? kAPlane : 0u, bo = (NPL == 2 && t == 1) ? kBPlane : 0u;
          const uint64_t ad = tile_desc<kBM, kind_mn<KA>()>(a0 + ao, kk), bd = tile_desc<BN, kind_mn<KB>()>(b0 + bo, kk);
          const uint32_t acc = (ch > 0 || kk > 0 || t > 0) ? 1u : 0u;
          asm volatile(
              "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
              "l"(ad), "l"(bd), "r"(idesc), "r"(acc)
              : "memory");
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_addr(&mma_bar[s]))
                   : "memory");
    }
    // refill the stage consumed one iteration ago (its MMAs must have finished reading it)
    const int nxt = ch + STAGES - 1;
    if (nxt < n_chunks) {
      const int sn = nxt % STAGES;
      if (ch >= 1) {
        mbar_wait(&mma_bar[sn], (phase_bits >> sn) & 1u);
        phase_bits ^= 1u << sn;
      }
      load_tile<kBM, NPL, KA>(opA, stage_ptr(sn), kAPlane, m0, nxt * kBK, K, kg0, rtA);
      load_tile<BN, NPL, KB>(opB, stage_ptr(sn) + NPL * kAPlane, kBPlane, n0, nxt * kBK, K, kg0, rtB);
    }
    cp_async_commit();
  }
  cp_async_wait<0>();
  // the last commit covers every MMA issued before it
  if (n_chunks > 0) {
    const int sl = (n_chunks - 1) % STAGES;
    // every stage holds at most one commit not yet waited for (those of the last STAGES chunks), so
    // the stage's current parity is the last chunk's commit, which covers all earlier MMAs
    mbar_wait(&mma_bar[sl], (phase_bits >> sl) & 1u);
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // epilogue (TMEM lanes = rows): 32 x 8 blocks transposed through shared memory for row-contiguous stores
  float* tr = reinterpret_cast<float*>(smem) + warp * (32 * 9);
  // warp w reads TMEM lane quarter w % 4 (rows) and column slice w / 4 of BN / (warps / 4) columns
  const int row0 = m0 + (warp & 3) * 32;
  constexpr int kSlice = BN / (kThreads / 128);
  static_assert(kSlice >= 8 && kSlice % 8 == 0, "epilogue column slice");
#pragma unroll 1
  for (int c0 = (warp >> 2) * kSlice; c0 < (warp >> 2) * kSlice + kSlice; c0 += 8) {
    uint32_t r[8];
    const uint32_t taddr = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int e = 0; e < 8; ++e) tr[lane * 9 + e] = __uint_as_float(r[e]);
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int rr = (lane >> 3) + 4 * i, cc = lane & 7;
      const int row = row0 + rr, col = n0 + c0 + cc;
      if (row < M && col < N) {
        float* cp = C + (long long)row * ldc + col;
        *cp = accumulate ? *cp + tr[rr * 9 + cc] : tr[rr * 9 + cc];
      }
    }
    __syncwarp();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols) : "memory");

}

// C (+)= sum over the splits (fixed order) of the partial tiles
__global__ void ig_splitk_reduce_kernel(const float* __restrict__ P, int splits, long long zs, int M, int N,
                                        float* __restrict__ C, long long ldc, int accumulate) {
  const long long n = (long long)M * N;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long m = i / N, c = i - m * N;
    float s = 0.f;
    for (int z = 0; z < splits; ++z) s += __ldcg(P + z * zs + i);
    float* cp = C + m * ldc + c;
    *cp = accumulate ? *cp + s : s;
  }
}

// weight gradient: dW[o][c][uv] = sum over the splits (fixed order) of P[z][(uv*Cp + c)*N + o], c < Cr
// (walks P in order: coalesced split reads, one scattered store per element)
__global__ void ig_splitk_reduce_wgrad_kernel(const float* __restrict__ P, int splits, long long zs, int N, int Cp,
                                              int Cr, int kk, float* __restrict__ dw) {
  const int n = kk * Cp * N;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int m = i / N, o = i - m * N, uv = m / Cp, c = m - uv * Cp;
    if (c >= Cr) continue;
    float s = 0.f;
    for (int z = 0; z < splits; ++z) s += __ldcg(P + z * zs + i);
    dw[(o * Cr + c) * kk + uv] = s;
  }
}

int log2_exact(int v) {
  if (v <= 0 || (v & (v - 1))) return -1;
  int l = 0;
  while ((1 << l) < v) ++l;
  return l;
}

OpDev to_dev(const IgOperand& o, int rows) {
  OpDev d;
  d.kind = o.kind;
  d.x = o.x;
  d.ld = o.ld;
  d.plane = o.plane;
  d.g = o.g;
  d.g.x = o.x;
  d.g.pw_log2 = log2_exact(o.g.PW);
  d.g.php_log2 = log2_exact(o.g.PH * o.g.PW);
  d.g.sc_log2 = log2_exact(o.g.SC);
  d.rows = rows;
  return d;
}

template <int BN, int NPL, int STAGES, int KA, int KB>
ddppo_status launch_ig(ddppo_ctx* ctx, const IGemm& g, cudaStream_t st) {
  constexpr size_t smem = (size_t)STAGES * NPL * (kBM + BN) * kBK * 2 + 1024;
  auto kern = igemm_kernel<BN, NPL, STAGES, KA, KB>;
  static bool attr_set = false;
  if (!attr_set) {
    DDPPO_CUDA_TRY(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr_set = true;
  }
  int splits = g.splits > 1 && g.partial ? g.splits : 1;
  if (splits == 1 && g.partial && g.auto_split) {
    // few output tiles and a long k loop: split k so that ~2 CTAs per SM stream in parallel
    const long long tiles = (long long)((g.N + BN - 1) / BN) * ((g.M + kBM - 1) / kBM);
    const int chunks = (g.K + kBK - 1) / kBK;
    splits = (int)std::max(1LL, std::min<long long>({(2LL * ctx->sm_count + tiles - 1) / tiles, chunks / 4, 16}));
  }
  int kper = (g.K + splits - 1) / splits;
  kper = (kper + kBK - 1) / kBK * kBK;
  const int nz = (g.K + kper - 1) / kper;
  const OpDev a = to_dev(g.a, g.M), b = to_dev(g.b, g.N);
  dim3 grid((g.N + BN - 1) / BN, (g.M + kBM - 1) / kBM, nz);
  if (g.wg_out) {
    // weight gradient: partial tiles (plain stores), then the split sum in PyTorch weight order
    DDPPO_REQUIRE(ctx, g.partial && !g.accumulate && g.M == g.wg_kk * g.wg_cp, "igemm: bad weight-gradient epilogue");
    const long long zs = (long long)g.M * g.N;
    ctx->count(2);
    kern<<<grid, kThreads, smem, st>>>(a, b, g.partial, g.N, g.M, g.N, g.K, kper, zs, 0);
    DDPPO_CUDA_TRY(ctx, cudaGetLastError());
    const int n = g.M * g.N;
    ig_splitk_reduce_wgrad_kernel<<<grid_for(n, 256, ctx->sm_count * 8), 256, 0, st>>>(
        g.partial, nz, zs, g.N, g.wg_cp, g.wg_cr, g.wg_kk, g.wg_out);
    DDPPO_CUDA_TRY(ctx, cudaGetLastError());
    return DDPPO_OK;
  }
  ctx->count(nz == 1 ? 1 : 2);
  if (nz == 1) {
    kern<<<grid, kThreads, smem, st>>>(a, b, g.C, g.ldc, g.M, g.N, g.K, kper, 0, g.accumulate);
  } else {
    // partial tiles (plain stores), then one parallel pass sums them in split order
    const long long zs = (long long)g.M * g.N;
    kern<<<grid, kThreads, smem, st>>>(a, b, g.partial, g.N, g.M, g.N, g.K, kper, zs, 0);
    DDPPO_CUDA_TRY(ctx, cudaGetLastError());
    ig_splitk_reduce_kernel<<<grid_for((int)std::min<long long>(zs, 1 << 30), 256, ctx->sm_count * 8), 256, 0, st>>>(
        g.partial, nz, zs, g.M, g.N, g.C, g.ldc, g.accumulate);
  }
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  return DDPPO_OK;
}

}  // namespace

ddppo_status launch_splitk_reduce(ddppo_ctx* ctx, const float* part, int splits, int64_t zs, int M, int N, float* C,
                                  int64_t ldc, int accumulate, cudaStream_t st) {
  ig_splitk_reduce_kernel<<<grid_for((int)std::min<int64_t>(zs, 1 << 30), 256, ctx->sm_count * 8), 256, 0, st>>>(
      part, splits, zs, M, N, C, ldc, accumulate);
  ctx->count(1);
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  return DDPPO_OK;
}

ddppo_status launch_splitk_reduce_wgrad(ddppo_ctx* ctx, const float* part, int splits, int64_t zs, int N, int Cp, int Cr,
                                        int kk, float* dw, cudaStream_t st) {
  const int n = kk * Cp * N;
  ig_splitk_reduce_wgrad_kernel<<<grid_for(n, 256, ctx->sm_count * 8), 256, 0, st>>>(part, splits, zs, N, Cp, Cr, kk,
                                                                                     dw);
  ctx->count(1);
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  return DDPPO_OK;
}

ddppo_status launch_igemm(ddppo_ctx* ctx, const IGemm& g, cudaStream_t st) {
  DDPPO_REQUIRE(ctx, g.M >= 1 && g.N >= 1 && g.K >= 1, "igemm: empty shape");
  const bool a_k = g.a.kind == IG_DENSE_K || g.a.kind == IG_PIX_K, b_k = g.b.kind == IG_DENSE_K || g.b.kind == IG_PIX_K;
  DDPPO_REQUIRE(ctx, !(a_k || b_k) || g.K % 8 == 0, "igemm: K-major operands need K % 8 == 0");
  DDPPO_REQUIRE(ctx, g.planes == 1 || g.planes == 2, "igemm: planes must be 1 or 2");
  for (const IgOperand* o : {&g.a, &g.b}) {
    DDPPO_REQUIRE(ctx, o->x && ((uintptr_t)o->x & 15) == 0, "igemm: operands must be 16-byte aligned");
    if (o->kind == IG_DENSE_K || o->kind == IG_DENSE_MN)
      DDPPO_REQUIRE(ctx, o->ld % 8 == 0, "igemm: dense leading dimension must be a multiple of 8");
    else
      DDPPO_REQUIRE(ctx, o->g.SC % 8 == 0, "igemm: gathered tensors need a multiple of 8 channels");
    if (g.planes == 2) DDPPO_REQUIRE(ctx, o->plane % 8 == 0, "igemm: plane offset must be a multiple of 8");
  }
  if (g.a.kind == IG_DENSE_MN || g.a.kind == IG_TAP_MN) DDPPO_REQUIRE(ctx, g.M % 8 == 0, "igemm: MN-major A needs M % 8 == 0");
  if (g.b.kind == IG_DENSE_MN || g.b.kind == IG_TAP_MN) DDPPO_REQUIRE(ctx, g.N % 8 == 0, "igemm: MN-major B needs N % 8 == 0");
  // instantiated operand combinations: forward (gather x dense weights, 2 planes), input gradient
  // (transposed gather x dense weights), weight gradient (tap gather x dense MN-major dy)
  const int ka = (g.a.kind == IG_PIX_K && g.a.g.transposed) ? IG_PIX_KT : g.a.kind;
  if (ka == IG_PIX_K && g.b.kind == IG_DENSE_K && g.planes == 2) {
    if (g.N <= 32) return launch_ig<32, 2, 4, IG_PIX_K, IG_DENSE_K>(ctx, g, st);
    return launch_ig<64, 2, 4, IG_PIX_K, IG_DENSE_K>(ctx, g, st);
  }
  if (ka == IG_PIX_KT && g.b.kind == IG_DENSE_K && g.planes == 2) {
    if (g.N <= 32) return launch_ig<32, 2, 4, IG_PIX_KT, IG_DENSE_K>(ctx, g, st);
    return launch_ig<64, 2, 4, IG_PIX_KT, IG_DENSE_K>(ctx, g, st);
  }
  if (ka == IG_PIX_KT && g.b.kind == IG_DENSE_K && g.planes == 1) {
    if (g.N <= 32) return launch_ig<32, 1, 4, IG_PIX_KT, IG_DENSE_K>(ctx, g, st);
    if (g.N <= 64) return launch_ig<64, 1, 4, IG_PIX_KT, IG_DENSE_K>(ctx, g, st);
    return launch_ig<128, 1, 4, IG_PIX_KT, IG_DENSE_K>(ctx, g, st);
  }
  if (ka == IG_TAP_MN && g.b.kind == IG_DENSE_MN && g.planes == 1) {
    if (g.N <= 32) return launch_ig<32, 1, 4, IG_TAP_MN, IG_DENSE_MN>(ctx, g, st);
    if (g.N <= 64) return launch_ig<64, 1, 4, IG_TAP_MN, IG_DENSE_MN>(ctx, g, st);
    return launch_ig<128, 1, 4, IG_TAP_MN, IG_DENSE_MN>(ctx, g, st);
  }
  DDPPO_REQUIRE(ctx, false, "igemm: operand combination not instantiated");
  return DDPPO_ERR_CONFIG;
}
