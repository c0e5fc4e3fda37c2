// tcgen05 (5th-gen tensor core) GEMM over fp32 operands for the dense contractions off the
// recurrences' dependency chains: the GRU / LSTM weight gradients (dW_hh = dG_h^T H_in, ...),
// input gradients (dX = dG W_ih), the LSTM input projections and the visual FC (steps a5 / a7).
//
//   C[m][n] = sum_k A(m, k) * B(n, k)      A(m,k) = A[m*sam + k*sak], B(n,k) = B[n*sbn + k*sbk]
//
// fp32 operands are rounded to bf16 while they are staged into shared memory in the UMMA
// canonical K-major SWIZZLE_NONE layout (8-row x 16-byte core matrices; LBO = 128 B between the
// two K halves of an MMA, SBO = 1024 B between 8-row groups), so any source strides (K- or
// M/N-contiguous) are accepted without a separate transpose pass.  One CTA = one 128 x BN output
// tile; the fp32 accumulator lives in TMEM (BN columns); one elected thread issues
// tcgen05.mma.cta_group::1.kind::f16 (M=128, N=BN, K=16) and tcgen05.commit signals an mbarrier
// per smem stage (2 stages: the next K chunk is staged while the tensor core runs); the epilogue
// reads TMEM with tcgen05.ld.32x32b.  The sum over k runs in one fixed order (deterministic).
// Options: prec = 3 stages each operand as two bf16 tiles (x = hi + lo) and accumulates
// lo*hi + hi*lo + hi*hi (~fp32 products, the visual agents' forward); splits > 1 splits k over
// grid.z into partial tiles summed afterwards in split order.
#include <cuda_bf16.h>

#include <algorithm>

#include "common.cuh"

namespace {

constexpr int kBM = 128, kBK = 64, kThreads = 512;

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version = 1 (sm100)
  // base_offset = 0, lbo_mode = 0, layout_type (bits 61..63) = 0 : SWIZZLE_NONE
  return d;
}

// kind::f16 instruction descriptor: D f32, A/B bf16, both K-major, M = 128, N = n
__device__ __forceinline__ uint32_t make_idesc(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(kBM >> 4) << 24);
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

// offset (bytes) of element (row, k) of a [rows x 64] bf16 tile in the canonical K-major layout
__device__ __forceinline__ uint32_t tile_off(int row, int kchunk) {
  return (uint32_t)((row >> 3) * 1024 + kchunk * 128 + (row & 7) * 16);
}

// bf16 hi part of 2 floats, and the bf16 rounding of the residual (split mode: x = hi + lo to ~16
// mantissa bits; the product is formed as hi*hi + hi*lo + lo*hi on the tensor core)
__device__ __forceinline__ uint32_t pk_hi(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ uint32_t pk_lo(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  __nv_bfloat162 l = __floats2bfloat162_rn(a - __low2float(h), b - __high2float(h));
  return *reinterpret_cast<uint32_t*>(&l);
}
template <bool SPLIT>
__device__ __forceinline__ void store4(unsigned char* dst, unsigned char* dlo, uint32_t off, float4 v) {
  *reinterpret_cast<uint2*>(dst + off) = make_uint2(pk_hi(v.x, v.y), pk_hi(v.z, v.w));
  if (SPLIT) *reinterpret_cast<uint2*>(dlo + off) = make_uint2(pk_lo(v.x, v.y), pk_lo(v.z, v.w));
}
template <bool SPLIT>
__device__ __forceinline__ void store8(unsigned char* dst, unsigned char* dlo, uint32_t off, const float (&v)[8]) {
  *reinterpret_cast<uint4*>(dst + off) =
      make_uint4(pk_hi(v[0], v[1]), pk_hi(v[2], v[3]), pk_hi(v[4], v[5]), pk_hi(v[6], v[7]));
  if (SPLIT)
    *reinterpret_cast<uint4*>(dlo + off) =
        make_uint4(pk_lo(v[0], v[1]), pk_lo(v[2], v[3]), pk_lo(v[4], v[5]), pk_lo(v[6], v[7]));
}

// Stage rows [r0, r0+ROWS) x k [k0, k0+64) of X(r, k) = X[r*sr + k*sk] (fp32) into a bf16 tile in
// the canonical layout.  K-contiguous sources (sk == 1) use coalesced float4 loads along k;
// otherwise thread t walks row t (consecutive threads -> consecutive rows: coalesced when sr == 1).
template <int ROWS, bool SPLIT>
__device__ __forceinline__ void stage_tile(unsigned char* dst, unsigned char* dlo, const float* __restrict__ X, long long sr,
                                           long long sk, int r0, int R, int k0, int K) {
  const int tid = threadIdx.x;
  if (sk == 1 && (sr & 3) == 0 && ((uintptr_t)X & 15) == 0) {
#pragma unroll 4
    for (int i = tid; i < ROWS * (kBK / 4); i += kThreads) {
      const int row = i / (kBK / 4), c4 = i % (kBK / 4), r = r0 + row, k = k0 + 4 * c4;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (r < R) {
        const float* src = X + (long long)r * sr + k;
        if (k + 3 < K) {
          v = *reinterpret_cast<const float4*>(src);
        } else {
          if (k < K) v.x = src[0];
          if (k + 1 < K) v.y = src[1];
          if (k + 2 < K) v.z = src[2];
        }
      }
      store4<SPLIT>(dst, dlo, tile_off(row, (4 * c4) >> 3) + ((4 * c4) & 7) * 2, v);
    }
    return;
  }
  for (int row = tid; row < ROWS; row += kThreads) {
    const int r = r0 + row;
#pragma unroll
    for (int kc = 0; kc < kBK / 8; ++kc) {
      float v[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int k = k0 + kc * 8 + e;
        v[e] = (r < R && k < K) ? X[(long long)r * sr + (long long)k * sk] : 0.f;
      }
      store8<SPLIT>(dst, dlo, tile_off(row, kc), v);
    }
  }
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Operand staging modes (host-selected): 0 = rows contiguous in HBM (X[r + k*sk]), raw fp32 tile
// [64 k][ROWS]; 1 = k contiguous (X[r*sr + k]), raw tile [ROWS][68]; 2 = anything else (direct
// loads, no raw tile).  Modes 0/1 copy HBM -> smem with 16-byte cp.async (no registers, many
// copies in flight), then the CTA converts the raw fp32 tile to the bf16 canonical tile.
constexpr int kRawPad = 68;

template <int ROWS>
__device__ __forceinline__ void issue_raw(int mode, float* raw, const float* __restrict__ X, long long sr, long long sk,
                                          int r0, int R, int k0, int K) {
  const int tid = threadIdx.x;
  if (mode == 0) {
    for (int i = tid; i < kBK * (ROWS / 4); i += kThreads) {
      const int kk = i / (ROWS / 4), j = i % (ROWS / 4), r = r0 + 4 * j, k = k0 + kk;
      const bool ok = (r < R) && (k < K);  // R % 4 == 0 guaranteed by the host
      const float* src = ok ? X + r + (long long)k * sk : X;
      cp_async16(smem_addr(raw + kk * ROWS + 4 * j), src, ok ? 16u : 0u);
    }
  } else if (mode == 1) {
    for (int i = tid; i < ROWS * (kBK / 4); i += kThreads) {
      const int row = i / (kBK / 4), j = i % (kBK / 4), r = r0 + row, k = k0 + 4 * j;
      const bool ok = (r < R) && (k < K);  // K % 4 == 0 guaranteed by the host
      const float* src = ok ? X + (long long)r * sr + k : X;
      cp_async16(smem_addr(raw + row * kRawPad + 4 * j), src, ok ? 16u : 0u);
    }

  }
}


template <int ROWS, bool SPLIT>
__device__ __forceinline__ void convert_tile(int mode, unsigned char* dst, unsigned char* dlo, const float* raw,
                                             const float* __restrict__ X, long long sr, long long sk, int r0, int R,
                                             int k0, int K) {
  if (mode == 2) {
    stage_tile<ROWS, SPLIT>(dst, dlo, X, sr, sk, r0, R, k0, K);
    return;
  }
  // (row, 8-wide k piece) pairs over all threads; consecutive threads take consecutive rows
  for (int pidx = threadIdx.x; pidx < ROWS * (kBK / 8); pidx += kThreads) {
    const int row = pidx % ROWS, kc = pidx / ROWS;
    {
      float v[8];
      if (mode == 0) {
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] = raw[(kc * 8 + e) * ROWS + row];
      } else {
        const float4 a = *reinterpret_cast<const float4*>(raw + row * kRawPad + kc * 8);
        const float4 b = *reinterpret_cast<const float4*>(raw + row * kRawPad + kc * 8 + 4);
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
      }
      store8<SPLIT>(dst, dlo, tile_off(row, kc), v);
    }
  }
}


template <int ROWS>
__host__ __device__ constexpr uint32_t raw_bytes() {
  return (uint32_t)(ROWS * kRawPad * 4 > kBK * ROWS * 4 ? ROWS * kRawPad * 4 : kBK * ROWS * 4);
}

template <int BN, bool SPLIT>
__global__ void __launch_bounds__(kThreads, 1)
gemm_bf16_tc_kernel(const float* __restrict__ A, long long sam, long long sak, const float* __restrict__ B,
                    long long sbn, long long sbk, float* __restrict__ C, long long ldc, int M, int N, int K, int kper,
                    long long cz_stride, int amode, int bmode, int accumulate) {
  pdl_enter();
  constexpr int kTmemCols = BN < 32 ? 32 : BN;
  constexpr uint32_t kABytes = kBM * kBK * 2, kBBytes = BN * kBK * 2;
  constexpr uint32_t kRawA = raw_bytes<kBM>(), kRawB = raw_bytes<BN>();
  constexpr int kParts = SPLIT ? 2 : 1;  // bf16 tiles per operand and stage (hi [, lo])
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* sA[2] = {smem, smem + kParts * kABytes};
  unsigned char* sB[2] = {smem + 2 * kParts * kABytes, smem + 2 * kParts * kABytes + kParts * kBBytes};
  unsigned char* rbase = smem + 2 * kParts * (kABytes + kBBytes);
  float* rA[2] = {reinterpret_cast<float*>(rbase), reinterpret_cast<float*>(rbase + kRawA)};
  float* rB[2] = {reinterpret_cast<float*>(rbase + 2 * kRawA), reinterpret_cast<float*>(rbase + 2 * kRawA + kRawB)};
  __shared__ uint64_t mma_bar[2];
  __shared__ uint32_t tmem_base_slot;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.y * kBM, n0 = blockIdx.x * BN;
  // split-K: CTA z of grid.z covers k in [z*kper, z*kper + kper) and writes its own partial C
  {
    const long long kbeg = (long long)blockIdx.z * kper;
    A += kbeg * sak;
    B += kbeg * sbk;
    K = (int)min((long long)kper, (long long)K - kbeg);
    C += (long long)blockIdx.z * cz_stride;
  }
  const int n_chunks = (K + kBK - 1) / kBK;

  // start streaming the first two K chunks while TMEM / barriers are set up
  issue_raw<kBM>(amode, rA[0], A, sam, sak, m0, M, 0, K);
  issue_raw<BN>(bmode, rB[0], B, sbn, sbk, n0, N, 0, K);
  cp_async_commit();
  if (n_chunks > 1) {
    issue_raw<kBM>(amode, rA[1], A, sam, sak, m0, M, kBK, K);
    issue_raw<BN>(bmode, rB[1], B, sbn, sbk, n0, N, kBK, K);
  }
  cp_async_commit();

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&tmem_base_slot)),
                 "n"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    mbar_init(&mma_bar[0], 1);
    mbar_init(&mma_bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base_slot;
  const uint32_t idesc = make_idesc(BN);

  uint32_t phase[2] = {0u, 0u};
  for (int ch = 0; ch < n_chunks; ++ch) {
    const int st = ch & 1;
    const int k0 = ch * kBK;
    cp_async_wait<1>();  // chunk ch has landed (chunk ch+1 may still be in flight)
    __syncthreads();
    if (ch >= 2) {  // the MMAs that read this bf16 stage two chunks ago must be done
      mbar_wait(&mma_bar[st], phase[st]);
      phase[st] ^= 1u;
    }
    convert_tile<kBM, SPLIT>(amode, sA[st], sA[st] + kABytes, rA[st], A, sam, sak, m0, M, k0, K);
    convert_tile<BN, SPLIT>(bmode, sB[st], sB[st] + kBBytes, rB[st], B, sbn, sbk, n0, N, k0, K);
    // generic-proxy smem writes -> visible to the tensor core (async proxy)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    // the raw stage is free again: stream chunk ch+2 into it
    if (ch + 2 < n_chunks) {
      issue_raw<kBM>(amode, rA[st], A, sam, sak, m0, M, k0 + 2 * kBK, K);
      issue_raw<BN>(bmode, rB[st], B, sbn, sbk, n0, N, k0 + 2 * kBK, K);
    }
    cp_async_commit();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t a_base = smem_addr(sA[st]), b_base = smem_addr(sB[st]);
      // split mode: the small cross terms lo*hi and hi*lo first, then hi*hi
      constexpr int kTerms = SPLIT ? 3 : 1;
#pragma unroll
      for (int kk = 0; kk < kBK / 16; ++kk) {
#pragma unroll
        for (int term = 0; term < kTerms; ++term) {
          const uint32_t ao = (SPLIT && term == 0) ? kABytes : 0u, bo = (SPLIT && term == 1) ? kBBytes : 0u;
          const uint64_t ad = make_desc(a_base + ao + kk * 256, 128, 1024);
          const uint64_t bd = make_desc(b_base + bo + kk * 256, 128, 1024);
          const uint32_t acc = (ch > 0 || kk > 0 || term > 0) ? 1u : 0u;
          asm volatile(
              "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
              "l"(ad), "l"(bd), "r"(idesc), "r"(acc)
              : "memory");
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_addr(&mma_bar[st]))
                   : "memory");
    }
  }
  cp_async_wait<0>();
  // wait for the last commit of each stage still outstanding
  {
    const int last = n_chunks - 1;
    const int st = last & 1;
    mbar_wait(&mma_bar[st], phase[st]);
    if (n_chunks >= 2) mbar_wait(&mma_bar[st ^ 1], phase[st ^ 1]);
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // epilogue: warp w owns TMEM lanes (rows) 32(w%4)..+31 and column half w/4; 32x8 blocks are
  // transposed through shared memory (the A stage buffer, free now) so that every store
  // instruction writes contiguous columns of one row.
  float* tr = reinterpret_cast<float*>(sA[0]) + warp * (32 * 9);
  const int row0 = m0 + (warp & 3) * 32;
  constexpr int kHalf = BN / (kThreads / 128);  // columns per warp
  static_assert(kHalf >= 8 && kHalf % 8 == 0, "epilogue column slice");
#pragma unroll 1
  for (int c0 = (warp >> 2) * kHalf; c0 < (warp >> 2) * kHalf + kHalf; c0 += 8) {
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
    // lane -> (row offset lane/8 + 4*i, column lane%8): 4 rows x 8 columns per instruction
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

__global__ void splitk_reduce_kernel(const float* __restrict__ P, int splits, long long zs, int M, int N,
                                     float* __restrict__ C, long long ldc, int accumulate) {
  pdl_enter();
  const long long n = (long long)M * N;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long m = i / N, c = i % N;
    float s = 0.f;
    for (int z = 0; z < splits; ++z) s += P[z * zs + m * N + c];  // fixed split order
    C[m * ldc + c] = accumulate ? C[m * ldc + c] + s : s;
  }
}

template <int BN, bool SPLIT>
ddppo_status launch_bn(ddppo_ctx* ctx, const GemmTC& g, cudaStream_t st) {
  auto mode_of = [](const float* X, int64_t sr, int64_t sk, int R, int K) {
    const bool al = ((uintptr_t)X & 15) == 0;
    if (al && sr == 1 && sk % 4 == 0 && R % 4 == 0) return 0;
    if (al && sk == 1 && sr % 4 == 0 && K % 4 == 0) return 1;
    return 2;
  };
  const int am = mode_of(g.A, g.sam, g.sak, g.M, g.K), bm = mode_of(g.B, g.sbn, g.sbk, g.N, g.K);
  const size_t parts = SPLIT ? 2 : 1;
  const size_t smem = 2 * parts * ((size_t)kBM * kBK * 2 + (size_t)BN * kBK * 2) + 2 * (size_t)raw_bytes<kBM>() +
                      2 * (size_t)raw_bytes<BN>();
  auto kern = gemm_bf16_tc_kernel<BN, SPLIT>;
  static bool attr_set = false;  // per device function (BN); smem size is a compile-time constant
  if (!attr_set) {
    DDPPO_CUDA_TRY(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr_set = true;
  }
  const int splits = g.splits > 1 && g.partial ? g.splits : 1;
  int kper = (g.K + splits - 1) / splits;
  kper = (kper + kBK - 1) / kBK * kBK;
  const int nz = (g.K + kper - 1) / kper;
  dim3 grid((g.N + BN - 1) / BN, (g.M + kBM - 1) / kBM, nz);
  ctx->count(nz == 1 ? 1 : 2);
  if (nz == 1) {
    launch_k(ctx, kern, grid, kThreads, smem, st, g.A, g.sam, g.sak, g.B, g.sbn, g.sbk, g.C, g.ldc, g.M, g.N, g.K,
             kper, 0, am, bm,
                                       g.accumulate);
  } else {
    const long long zs = (long long)g.M * g.N;
    launch_k(ctx, kern, grid, kThreads, smem, st, g.A, g.sam, g.sak, g.B, g.sbn, g.sbk, g.partial, g.N, g.M, g.N, g.K,
             kper, zs, am,
                                       bm, 0);
    DDPPO_CUDA_TRY(ctx, cudaGetLastError());
    launch_k(ctx, splitk_reduce_kernel, grid_for((int)std::min<long long>(zs, 1 << 30), 256, ctx->sm_count * 8), 256, 0,
             st, g.partial, nz, zs, g.M, g.N, g.C, g.ldc, g.accumulate);
  }
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  return DDPPO_OK;
}

}  // namespace

ddppo_status launch_gemm_tc(ddppo_ctx* ctx, const GemmTC& g, cudaStream_t st) {
  DDPPO_REQUIRE(ctx, g.M >= 1 && g.N >= 1 && g.K >= 1, "gemm: empty shape");
  DDPPO_REQUIRE(ctx, g.prec == 1 || g.prec == 3, "gemm: prec must be 1 (bf16) or 3 (bf16x3)");
  if (g.prec == 3) {  // two bf16 tiles per operand: BN <= 64 keeps the stages inside 227 KB
    if (g.N <= 32) return launch_bn<32, true>(ctx, g, st);
    return launch_bn<64, true>(ctx, g, st);
  }
  if (g.N <= 32) return launch_bn<32, false>(ctx, g, st);
  if (g.N <= 64) return launch_bn<64, false>(ctx, g, st);
  return launch_bn<128, false>(ctx, g, st);
}

extern "C" ddppo_status ddppo_debug_gemm_bf16(ddppo_ctx* ctx, const float* A, int64_t sam, int64_t sak,
                                              const float* B, int64_t sbn, int64_t sbk, float* C, int64_t ldc, int M,
                                              int N, int K, int splits, float* partial, int prec, void* stream) {
  if (!ctx) return DDPPO_ERR_CONFIG;
  GemmTC g{A, sam, sak, B, sbn, sbk, C, ldc, M, N, K, splits, partial, prec};
  ProfScope ps(ctx, DDPPO_K_OTHER, as_stream(stream), 0);
  return launch_gemm_tc(ctx, g, as_stream(stream));
}
