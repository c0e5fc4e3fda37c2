// LSTM-1024 recurrences (NEXT-3: "a 2-layer LSTM with either a 512-dimensional or 1024-dimensional
// hidden dimension"; the best agent of Table 2, SE-ResNeXt101 + 1024-d LSTM).
// PyTorch gate order i, f, g, o; state and cell multiplied by mask_t (reading Z21), as lstm.cu.
//
// Why a different distribution from lstm.cu.  W_hh of a 1024-unit layer is 4096 x 1024 (8 MB in
// fp16): a 16-CTA cluster holds at most 16 x (256 KB TMEM + 227 KB smem) = 7.7 MB, so the weights
// cannot stay on chip inside one cluster.  Here 32 CTAs (one per SM, launched together; each owns
// 32 hidden units = 128 gate rows) keep their rows resident -- K [0, 768) in TMEM as the A operand
// (384 columns), K [768, 1024) in shared memory (64 KB, canonical K-major, A from a descriptor) --
// and exchange h_t through L2 instead of DSMEM:
//  * forward: each MMA warp publishes its 8 units of h_t (fp16, one 16-byte row per env) into the
//    exchange tile hx[t%2] (the canonical [8 x 1024] B-operand layout) and bumps the counter of
//    its CTA's group (8 CTAs = 256 units = one K quarter) with a release reduction; MMA warp w
//    waits (acquire) for group w only, copies that 4 KB K quarter into its B tile and issues its 16
//    tcgen05.mma (M=128, N=8, K=16) into its own TMEM accumulator -- the tensor pipe runs while
//    other quarters are still in flight; the cells are finished in-warp as in lstm.cu.
//  * backward: W_hh^T restricted to the CTA's 128 gate rows, 8 tiles of 128 units (bf16): tiles
//    0..5 in TMEM, 6..7 in shared memory; per step the partial W_hh^T dG of all 1024 units is
//    written to the owners' slots of a reduce-scatter buffer and each owner sums its 32 sources in
//    CTA order (deterministic).
// Counters are zeroed (cudaMemsetAsync) before every launch; every wait is bounded by %globaltimer
// (a timeout sets ERR_BIT_COMM, reported by ddppo_check, instead of hanging the device).
#include "common.cuh"
#include "tc_util.cuh"

using namespace tcu;

namespace {

constexpr int kH = 1024, kG4 = 4 * kH, kNCta = 32, kUPC = 32, kRows = 128, kBMax = 8;
constexpr int kThreads = 256, kMmaWarps = 4, kGroupCtas = kNCta / kMmaWarps /*8*/;
constexpr int kKTmem = 768;                             // K columns of W held in TMEM (fwd)
constexpr uint32_t kHTile = (kH / 8) * 128;             // [8 x 1024] fp16 B tile: 16 KB
constexpr uint32_t kQuarter = kHTile / kMmaWarps;       // one group's 256 K columns: 4 KB
constexpr uint32_t kASmemSBO = ((kH - kKTmem) / 8) * 128;  // A smem part [128 rows][256 K]: 4096 B / 8 rows
constexpr uint64_t kTimeoutNs = 2000000000ull;

constexpr uint32_t kIdescF16_N8 = (1u << 4) | ((8u >> 3) << 17) | ((128u >> 4) << 24);
constexpr uint32_t kIdescBF16_N8 = (1u << 4) | (1u << 7) | (1u << 10) | ((8u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ uint32_t tile_off(int r, int k, uint32_t sbo) {  // canonical K-major, no swizzle
  return (uint32_t)((r >> 3) * sbo + (k >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2);
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_gpu(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// LL ("low latency") exchange words: 8 bytes = 4 bytes of payload + a 4-byte flag (the step + 1), one
// naturally aligned 8-byte store, so a reader that sees the flag sees the payload: no release fence,
// no counter, one L2 round trip per step.  Buffers are zeroed before every launch (flags start at 1).
__device__ __forceinline__ void st_ll2(void* p, uint32_t d0, uint32_t d1, uint32_t flag) {  // two words
  asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(d0), "r"(flag), "r"(d1), "r"(flag)
               : "memory");
}
__device__ __forceinline__ void st_ll1(void* p, uint32_t d0, uint32_t flag) {
  asm volatile("st.volatile.global.v2.u32 [%0], {%1, %2};" ::"l"(p), "r"(d0), "r"(flag) : "memory");
}
// poll a 16-byte pair of words until both carry `flag`; false after the timeout (sets ERR_BIT_COMM)
__device__ __forceinline__ bool ld_ll2(const void* p, uint32_t flag, uint32_t& d0, uint32_t& d1, int* err) {
  uint32_t a, f0, b, f1;
  asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(a), "=r"(f0), "=r"(b), "=r"(f1) : "l"(p) : "memory");
  if (f0 != flag || f1 != flag) {
    const uint64_t t0 = globaltimer();
    for (int i = 0;; ++i) {
      asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(a), "=r"(f0), "=r"(b), "=r"(f1) : "l"(p) : "memory");
      if (f0 == flag && f1 == flag) break;
      if ((i & 255) == 255 && globaltimer() - t0 > kTimeoutNs) {
        atomicOr(err, ERR_BIT_COMM);
        return false;
      }
    }
  }
  d0 = a;
  d1 = b;
  return true;
}
__device__ __forceinline__ bool ld_ll1(const void* p, uint32_t flag, uint32_t& d0, int* err) {
  uint32_t a, f0;
  asm volatile("ld.volatile.global.v2.u32 {%0, %1}, [%2];" : "=r"(a), "=r"(f0) : "l"(p) : "memory");
  if (f0 != flag) {
    const uint64_t t0 = globaltimer();
    for (int i = 0;; ++i) {
      asm volatile("ld.volatile.global.v2.u32 {%0, %1}, [%2];" : "=r"(a), "=r"(f0) : "l"(p) : "memory");
      if (f0 == flag) break;
      if ((i & 255) == 255 && globaltimer() - t0 > kTimeoutNs) {
        atomicOr(err, ERR_BIT_COMM);
        return false;
      }
    }
  }
  d0 = a;
  return true;
}
constexpr size_t kHxWords = 2 * kBMax * (kH / 2);  // fwd: [parity][env row][unit pair]

// lane 0 polls with acquire loads, the warp barrier then orders the other lanes' reads after it;
// false on timeout (warp-uniform)
__device__ __forceinline__ bool wait_count(const unsigned* cnt, unsigned target, int* err) {
  int ok = 1;
  if ((threadIdx.x & 31) == 0 && ld_acquire_gpu(cnt) < target) {
    const uint64_t t0 = globaltimer();
    for (int i = 0;; ++i) {
      if (ld_acquire_gpu(cnt) >= target) break;
      if ((i & 255) == 255 && globaltimer() - t0 > kTimeoutNs) {
        atomicOr(err, ERR_BIT_COMM);
        ok = 0;
        break;
      }
    }
  }
  return __shfl_sync(0xffffffffu, ok, 0) != 0;
}

// ------------------------------------------------------------------ forward
struct FwdSmem {
  unsigned char a_s[kRows / 8 * kASmemSBO];  // W rows, K [768, 1024), fp16 (64 KB)
  unsigned char h_tile[2][kHTile];           // h_{t-1} fp16 [8 env rows][1024], by step parity
  unsigned char stage[kMmaWarps][128];       // per MMA warp: new h of its 8 units [env][8] fp16
  uint64_t mma_bar;
  uint32_t tmem_slot;
};

__global__ void __launch_bounds__(kThreads, 1) lstm1024_fwd_kernel(LstmPtrs p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  FwdSmem& sm = *reinterpret_cast<FwdSmem*>(smem_raw);
  float* smask = reinterpret_cast<float*>(smem_raw + sizeof(FwdSmem));  // [B][T_run]
  const int c = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int B = p.B, T_run = p.T_run, S = B * T_run;

  {
    uint4* zz = reinterpret_cast<uint4*>(sm.h_tile);
    for (int i = tid; i < (int)(sizeof(sm.h_tile) / 16); i += blockDim.x) zz[i] = make_uint4(0u, 0u, 0u, 0u);
  }
  for (int i = tid; i < S; i += blockDim.x) {
    const int b = i / T_run, t = i - b * T_run;
    smask[i] = p.mask[(size_t)p.env_idx[b] * p.ld + t];
  }
  if (tid == 0) {
    mbar_init(&sm.mma_bar, kMmaWarps);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc<512>(&sm.tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_slot;
  // A operand: row r = 32(w%4) + lane holds gate lane/8 of unit 8(w%4) + lane%8.  Warps w < 4 write
  // TMEM columns [0, 192), warps w >= 4 columns [192, 384) and the smem part (K >= 768).
  {
    const int row = 32 * (warp & 3) + lane;  // M index = TMEM lane
    const int grow = (lane >> 3) * kH + c * kUPC + 8 * (warp & 3) + (lane & 7);
    const float* wh = p.Whh + (size_t)grow * kH;
    const int col_lo = (warp < 4) ? 0 : kKTmem / 4;
#pragma unroll 1
    for (int col0 = col_lo; col0 < col_lo + kKTmem / 4; col0 += 32) {
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
    if (warp >= 4) {
#pragma unroll 1
      for (int k0 = kKTmem; k0 < kH; k0 += 8) {
        const float4 x0 = *reinterpret_cast<const float4*>(wh + k0), x1 = *reinterpret_cast<const float4*>(wh + k0 + 4);
        *reinterpret_cast<uint4*>(sm.a_s + tile_off(row, k0 - kKTmem, kASmemSBO)) =
            make_uint4(pack_f16(x0.x, x0.y), pack_f16(x0.z, x0.w), pack_f16(x1.x, x1.y), pack_f16(x1.z, x1.w));
      }
    }
    tmem_wait_st();
  }
  for (int i = tid; i < B * kH; i += blockDim.x) {
    const int b = i / kH, k = i % kH;
    const float h = smask[b * T_run] * p.h0[(size_t)p.env_idx[b] * p.sld + k];
    *reinterpret_cast<__half*>(sm.h_tile[0] + tile_off(b, k, kHTile)) = __float2half(h);
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  if (warp < kMmaWarps) {
    const int w = warp, u8 = lane & 7, u = 8 * w + u8, gunit = c * kUPC + u;
    float bias[4];
#pragma unroll
    for (int g = 0; g < 4; ++g) bias[g] = p.bih[g * kH + gunit] + p.bhh[g * kH + gunit];
    float hown[2] = {0.f, 0.f}, cown[2] = {0.f, 0.f}, gi[2][4];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int b = (lane >> 3) + 4 * j;
#pragma unroll
      for (int g = 0; g < 4; ++g) gi[j][g] = 0.f;
      if (b < B) {
        const int n = p.env_idx[b];
        hown[j] = smask[b * T_run] * p.h0[(size_t)n * p.sld + gunit];
        cown[j] = smask[b * T_run] * p.c0[(size_t)n * p.sld + gunit];
        const float* g0 = p.GI + (size_t)(b * T_run) * kG4 + gunit;
#pragma unroll
        for (int g = 0; g < 4; ++g) gi[j][g] = g0[g * kH];
      }
    }
    const uint32_t a_s_base = smem_u32(sm.a_s), h_base0 = smem_u32(sm.h_tile[0]);
    const uint32_t d_acc = tmem + kKTmem / 2 + 8u * (uint32_t)w;
    bool ok = true;
    for (int t = 0; t < T_run; ++t) {
      const int cur = t & 1;
      if (t > 0) {
        // h_{t-1} of group w (units [256w, +256)), LL words of step t-1 (flag t): 4 units per 16 bytes;
        // every load of the lane in flight at once, re-read until all flags match
        const uint2* hx = reinterpret_cast<const uint2*>(p.hx) + (size_t)((t - 1) & 1) * kBMax * (kH / 2);
        constexpr int kPer = 2 * kBMax;  // 16-byte loads per lane (B = 8)
        uint4 v[kPer];
        const uint64_t t0 = globaltimer();
        for (int spin = 0;; ++spin) {
          bool all = true;
#pragma unroll
          for (int q = 0; q < kPer; ++q) {
            const int i = lane + 32 * q;
            if (i < 64 * B) {
              const int b = i >> 6, u0 = 256 * w + 4 * (i & 63);
              asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                           : "=r"(v[q].x), "=r"(v[q].y), "=r"(v[q].z), "=r"(v[q].w)
                           : "l"(hx + (size_t)b * (kH / 2) + u0 / 2)
                           : "memory");
            }
          }
#pragma unroll
          for (int q = 0; q < kPer; ++q)
            if (lane + 32 * q < 64 * B) all = all && v[q].y == (uint32_t)t && v[q].w == (uint32_t)t;
          if (__all_sync(0xffffffffu, all)) break;
          if ((spin & 63) == 63 && globaltimer() - t0 > kTimeoutNs) {
            if (lane == 0) atomicOr(p.err, ERR_BIT_COMM);
            ok = false;
            break;
          }
        }
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
          const int i = lane + 32 * q;
          if (i < 64 * B) {
            const int b = i >> 6, u0 = 256 * w + 4 * (i & 63);
            *reinterpret_cast<uint2*>(sm.h_tile[cur] + tile_off(b, u0, kHTile)) = make_uint2(v[q].x, v[q].z);
          }
        }
        fence_proxy_async();
        __syncwarp();
      }
      tc_fence_after();
      const uint64_t bd0 = umma_desc(h_base0 + (uint32_t)cur * kHTile, 128, kHTile);
#pragma unroll
      for (int j = 0; j < 16; ++j) {  // K = 256w + 16j
        const int kk = 16 * w + j;
        if (kk * 16 < kKTmem)
          mma_ts(d_acc, tmem + 8u * (uint32_t)kk, bd0 + (uint64_t)(16 * kk), kIdescF16_N8, (uint32_t)j);
        else
          mma_ss(d_acc, umma_desc(a_s_base + (uint32_t)(kk * 16 - kKTmem) * 16u, 128, kASmemSBO),
                 bd0 + (uint64_t)(16 * kk), kIdescF16_N8, (uint32_t)j);
      }
      mma_commit(&sm.mma_bar);
      mbar_wait_parity(&sm.mma_bar, (uint32_t)(t & 1));
      tc_fence_after();
      uint32_t v[4][8];
#pragma unroll
      for (int a = 0; a < 4; ++a)
        tmem_ld8(tmem + ((uint32_t)(w * 32) << 16) + kKTmem / 2 + 8u * (uint32_t)a, v[a]);
      tmem_wait_ld();
      tc_fence_before();
      float acc[8];
#pragma unroll
      for (int e = 0; e < 8; ++e)
        acc[e] = (__uint_as_float(v[0][e]) + __uint_as_float(v[1][e])) + (__uint_as_float(v[2][e]) + __uint_as_float(v[3][e]));
      float gv[4][2];
#pragma unroll
      for (int g = 0; g < 4; ++g) gv[g][0] = gv[g][1] = 0.f;
#pragma unroll
      for (int bp = 0; bp < kBMax; ++bp) {
        if (bp < B) {
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            const float x = __shfl_sync(0xffffffffu, acc[bp], 8 * g + u8);
            if (bp == (lane >> 3)) gv[g][0] = x;
            if (bp == (lane >> 3) + 4) gv[g][1] = x;
          }
        }
      }
      float hv[2], cv[2], hin[2], cin[2];
      float4 ifgo[2];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int b = (lane >> 3) + 4 * j;
        const float ig = sigmoid_fast(gv[0][j] + gi[j][0] + bias[0]);
        const float fg = sigmoid_fast(gv[1][j] + gi[j][1] + bias[1]);
        const float gg = tanh_fast(gv[2][j] + gi[j][2] + bias[2]);
        const float og = sigmoid_fast(gv[3][j] + gi[j][3] + bias[3]);
        hin[j] = hown[j];
        cin[j] = cown[j];
        cv[j] = fg * cown[j] + ig * gg;
        hv[j] = og * tanh_fast(cv[j]);
        ifgo[j] = make_float4(ig, fg, gg, og);
        if (b < B && t + 1 < T_run) {
          const float m = smask[b * T_run + t + 1];
          hown[j] = m * hv[j];
          cown[j] = m * cv[j];
          reinterpret_cast<__half*>(sm.stage[w])[b * 8 + u8] = __float2half(m * hv[j]);
        }
      }
      if (t + 1 < T_run) {  // publish units [32c + 8w, +8) of env row b as 4 LL words (flag t + 1)
        __syncwarp();
        if (lane < 2 * B) {
          const int b = lane >> 1, half = lane & 1;
          const uint2 pk = *reinterpret_cast<const uint2*>(sm.stage[w] + 16 * b + 8 * half);
          uint2* hx = reinterpret_cast<uint2*>(p.hx) + (size_t)cur * kBMax * (kH / 2) + (size_t)b * (kH / 2) +
                      (gunit - u8) / 2 + 2 * half;
          st_ll2(hx, pk.x, pk.y, (uint32_t)(t + 1));
        }
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int b = (lane >> 3) + 4 * j;
        if (b < B) {
          const size_t o = ((size_t)b * T_run + t) * kH + gunit;
          p.Hs[o] = hv[j];
          p.Hin[o] = hin[j];
          p.Cin[o] = cin[j];
          p.Cs[o] = cv[j];
          p.IFGO[o] = ifgo[j];
          if (t + 1 < T_run) {
            const float* g0 = p.GI + (size_t)(b * T_run + t + 1) * kG4 + gunit;
#pragma unroll
            for (int g = 0; g < 4; ++g) gi[j][g] = g0[g * kH];
          }
        }
      }
    }
    (void)ok;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

// ------------------------------------------------------------------ backward (BPTT)
constexpr uint32_t kDgTile = (kRows / 8) * 128;   // [8 x 128] bf16 B tile
constexpr uint32_t kWtSBO = (kRows / 8) * 128;    // W^T tile [128 units][128 K] bf16: 2048 B / 8 rows
constexpr uint32_t kWtBytes = 16 * kWtSBO;        // 32 KB
constexpr int kTilesTmem = 6;                     // tiles 0..5 in TMEM (64 columns each), 6..7 in smem
constexpr uint32_t kBwdAcc0 = kTilesTmem * 64;    // 8 accumulators x 8 columns from column 384

struct BwdSmem {
  unsigned char wt_s[2][kWtBytes];  // W^T tiles 6, 7 (bf16)
  unsigned char dg_tile[kDgTile];   // dL/d(gates) (bf16) [8 env rows][128 own rows]
  uint64_t mma_bar;
  uint32_t tmem_slot;
};

__global__ void __launch_bounds__(kThreads, 1) lstm1024_bwd_kernel(LstmPtrs p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  BwdSmem& sm = *reinterpret_cast<BwdSmem*>(smem_raw);
  float* smask = reinterpret_cast<float*>(smem_raw + sizeof(BwdSmem));
  const int c = blockIdx.x;
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
    mbar_init(&sm.mma_bar, kMmaWarps);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc<512>(&sm.tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_slot;
  // A operand: tile q = units 128q.., lane = unit j, K = own gate row lr = g*32 + u (global row
  // g*1024 + 32c + u): A_q[j][lr] = W_hh[grow(lr)][128q + j].  Warp w (lane quarter w%4) handles
  // tiles q = w/4, w/4 + 2, ... (TMEM tiles) and the same lane rows of the smem tiles.
  {
    const int jl = (warp & 3) * 32 + lane;
#pragma unroll 1
    for (int q = warp >> 2; q < 8; q += 2) {
      const float* wcol = p.Whh + 128 * q + jl;
#pragma unroll 1
      for (int lr0 = 0; lr0 < kRows; lr0 += 32) {
        float w[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const int lr = lr0 + e;
          w[e] = wcol[(size_t)((lr / kUPC) * kH + c * kUPC + (lr % kUPC)) * kH];
        }
        if (q < kTilesTmem) {
#pragma unroll
          for (int sb = 0; sb < 2; ++sb) {
            uint32_t v[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) v[e] = pack_bf16(w[16 * sb + 2 * e], w[16 * sb + 2 * e + 1]);
            tmem_st8(tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(64 * q + lr0 / 2 + 8 * sb), v);
          }
        } else {
#pragma unroll
          for (int e8 = 0; e8 < 4; ++e8)
            *reinterpret_cast<uint4*>(sm.wt_s[q - kTilesTmem] + tile_off(jl, lr0 + 8 * e8, kWtSBO)) =
                make_uint4(pack_bf16(w[8 * e8], w[8 * e8 + 1]), pack_bf16(w[8 * e8 + 2], w[8 * e8 + 3]),
                           pack_bf16(w[8 * e8 + 4], w[8 * e8 + 5]), pack_bf16(w[8 * e8 + 6], w[8 * e8 + 7]));
        }
      }
    }
    tmem_wait_st();
  }
  const int ustride = B == 1 ? 1 : (B <= 2 ? 2 : (B <= 4 ? 4 : 8));  // LL words per (source, unit)
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  if (warp < kMmaWarps) {
    const int w = warp, u8 = lane & 7, u = 8 * w + u8, gunit = c * kUPC + u;
    // reduce-scatter slots: part[parity][owner][src][32 units][ustride]
    const size_t owner_stride = (size_t)kNCta * kUPC * ustride, parity_stride = (size_t)kNCta * owner_stride;
    float carry_h[2] = {0.f, 0.f}, carry_c[2] = {0.f, 0.f};
    float dH_t[2] = {0.f, 0.f}, c_t[2] = {0.f, 0.f}, c_in[2] = {0.f, 0.f};
    float4 ifgo[2] = {make_float4(0.f, 0.f, 0.f, 0.f), make_float4(0.f, 0.f, 0.f, 0.f)};
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int b = (lane >> 3) + 4 * j;
      if (b < B) {
        const size_t o = ((size_t)b * T_run + T_run - 1) * kH + gunit;
        dH_t[j] = p.dH[o];
        c_t[j] = p.Cs[o];
        c_in[j] = p.Cin[o];
        ifgo[j] = p.IFGO[o];
      }
    }
    const uint64_t bd0 = umma_desc(smem_u32(sm.dg_tile), 128, kDgTile);
    bool ok = true;
    for (int it = 0; it < T_run; ++it) {
      const int t = T_run - 1 - it, par = it & 1;
      float dgv[2][4];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int b = (lane >> 3) + 4 * j;
        const float dh = dH_t[j] + carry_h[j];
        const float ig = ifgo[j].x, fg = ifgo[j].y, gg = ifgo[j].z, og = ifgo[j].w;
        const float tc = tanhf(c_t[j]);
        const float dc = dh * og * (1.f - tc * tc) + carry_c[j];
        dgv[j][0] = dc * gg * ig * (1.f - ig);
        dgv[j][1] = dc * c_in[j] * fg * (1.f - fg);
        dgv[j][2] = dc * ig * (1.f - gg * gg);
        dgv[j][3] = dh * tc * og * (1.f - og);
        if (b < B) {
#pragma unroll
          for (int g = 0; g < 4; ++g)
            *reinterpret_cast<__nv_bfloat16*>(sm.dg_tile + tile_off(b, g * kUPC + u, kDgTile)) =
                __float2bfloat16(dgv[j][g]);
          carry_c[j] = smask[b * T_run + t] * dc * fg;
        }
      }
      fence_proxy_async();
      asm volatile("bar.sync 1, 128;" ::: "memory");  // the 4 MMA warps: dG tile complete
      tc_fence_after();
#pragma unroll
      for (int qi = 0; qi < 2; ++qi) {  // warp w: tiles 2w, 2w+1
        const int q = 2 * w + qi;
        const uint32_t d_q = tmem + kBwdAcc0 + 8u * (uint32_t)q;
#pragma unroll
        for (int kk = 0; kk < kRows / 16; ++kk) {
          if (q < kTilesTmem)
            mma_ts(d_q, tmem + 64u * (uint32_t)q + 8u * (uint32_t)kk, bd0 + (uint64_t)(16 * kk), kIdescBF16_N8,
                   (uint32_t)kk);
          else
            mma_ss(d_q, umma_desc(smem_u32(sm.wt_s[q - kTilesTmem]) + (uint32_t)kk * 256u, 128, kWtSBO),
                   bd0 + (uint64_t)(16 * kk), kIdescBF16_N8, (uint32_t)kk);
        }
      }
      mma_commit(&sm.mma_bar);
#pragma unroll
      for (int j = 0; j < 2; ++j) {  // off the chain while the MMAs run: save dG, prefetch step t-1
        const int b = (lane >> 3) + 4 * j;
        if (b < B) {
          const size_t og4 = ((size_t)b * T_run + t) * kG4 + gunit;
#pragma unroll
          for (int g = 0; g < 4; ++g) p.dG[og4 + g * kH] = dgv[j][g];
          if (t > 0) {
            const size_t o = ((size_t)b * T_run + t - 1) * kH + gunit;
            dH_t[j] = p.dH[o];
            c_t[j] = p.Cs[o];
            c_in[j] = p.Cin[o];
            ifgo[j] = p.IFGO[o];
          }
        }
      }
      mbar_wait_parity(&sm.mma_bar, (uint32_t)(it & 1));
      tc_fence_after();
      // partials of units 128q + 32w + lane (owner CTA 4q + w) into the owners' slots as LL words
      // {partial, it + 1}: word ((owner * 32 + src) * 32 + unit) * ustride + b
      uint2* part = reinterpret_cast<uint2*>(p.xpart) + (size_t)par * parity_stride;
      const uint32_t flag = (uint32_t)(it + 1);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        uint32_t a[8];
        tmem_ld8(tmem + ((uint32_t)(w * 32) << 16) + kBwdAcc0 + 8u * (uint32_t)q, a);
        tmem_wait_ld();
        uint2* dst = part + (size_t)(4 * q + w) * owner_stride + ((size_t)c * kUPC + lane) * ustride;
        if (B == 1) {
          st_ll1(dst, a[0], flag);
        } else {
#pragma unroll
          for (int e = 0; e < kBMax; e += 2)
            if (e < B) st_ll2(dst + e, a[e], a[e + 1], flag);
        }
      }
      tc_fence_before();
      // own units: all 32 sources' partials, summed in CTA order
      const uint2* mine = part + (size_t)c * owner_stride;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int b = (lane >> 3) + 4 * j;
        if (j == 1 && B <= 4) break;  // warp-uniform: slot 1 only exists for B > 4
        uint2 v[kNCta];
        const uint64_t t0 = globaltimer();
        for (int spin = 0;; ++spin) {  // all 32 sources' words in flight, re-read until every flag matches
          bool all = true;
          if (b < B) {
#pragma unroll
            for (int s2 = 0; s2 < kNCta; ++s2)
              asm volatile("ld.volatile.global.v2.u32 {%0, %1}, [%2];"
                           : "=r"(v[s2].x), "=r"(v[s2].y)
                           : "l"(mine + ((size_t)s2 * kUPC + u) * ustride + b)
                           : "memory");
#pragma unroll
            for (int s2 = 0; s2 < kNCta; ++s2) all = all && v[s2].y == flag;
          }
          if (__all_sync(0xffffffffu, all)) break;
          if ((spin & 63) == 63 && globaltimer() - t0 > kTimeoutNs) {
            if (lane == 0) atomicOr(p.err, ERR_BIT_COMM);
            ok = false;
            break;
          }
        }
        if (b < B) {
          float s = 0.f;
#pragma unroll
          for (int q = 0; q < kNCta; ++q) s += __uint_as_float(v[q].x);
          carry_h[j] = smask[b * T_run + t] * s;
        }
      }
    }
    (void)ok;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

ddppo_status launch_wide(ddppo_ctx* ctx, void (*kernel)(LstmPtrs), size_t smem, const LstmPtrs& p, cudaStream_t st,
                         void* ll, size_t ll_bytes) {
  DDPPO_CUDA_TRY(ctx, cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  DDPPO_CUDA_TRY(ctx, cudaMemsetAsync(ll, 0, ll_bytes, st));  // LL flags start below every step's
  kernel<<<kNCta, kThreads, smem, st>>>(p);
  ctx->count(1);
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  return DDPPO_OK;
}

}  // namespace

size_t lstm_wide_part_offset() { return kHxWords * 8; }

size_t lstm_wide_exchange_bytes() {
  // LL words (8 bytes): hx [2][8 rows][512 unit pairs]; partials [2][32 owners][32 sources][32 units][<= 8]
  return kHxWords * 8 + 2 * (size_t)kNCta * kNCta * kUPC * kBMax * 8 + 256;
}

ddppo_status launch_lstm1024_fwd(ddppo_ctx* ctx, const LstmPtrs& p, cudaStream_t st) {
  DDPPO_REQUIRE(ctx, p.hx && p.err, "lstm-1024: exchange buffers missing");
  DDPPO_REQUIRE(ctx, ctx->sm_count >= kNCta, "lstm-1024: needs 32 SMs");
  return launch_wide(ctx, lstm1024_fwd_kernel, sizeof(FwdSmem) + (size_t)p.B * p.T_run * sizeof(float), p, st, p.hx,
                     kHxWords * 8);
}

ddppo_status launch_lstm1024_bwd(ddppo_ctx* ctx, const LstmPtrs& p, cudaStream_t st) {
  DDPPO_REQUIRE(ctx, p.xpart && p.err, "lstm-1024: exchange buffers missing");
  DDPPO_REQUIRE(ctx, ctx->sm_count >= kNCta, "lstm-1024: needs 32 SMs");
  const int ustride = p.B == 1 ? 1 : (p.B <= 2 ? 2 : (p.B <= 4 ? 4 : 8));
  return launch_wide(ctx, lstm1024_bwd_kernel, sizeof(BwdSmem) + (size_t)p.B * p.T_run * sizeof(float), p, st,
                     p.xpart, 2 * (size_t)kNCta * kNCta * kUPC * ustride * 8);
}
