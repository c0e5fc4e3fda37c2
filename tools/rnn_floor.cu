// Floor microbenchmark of the 16-CTA cluster recurrence step:
// the pieces of one step of gps_gru_fwd_kernel / lstm_fwd_kernel timed in isolation, no gate math.
//
//   mode 0  exchange only: every CTA st.async's its h slice (B envs x 32 units fp16, 16-byte packets)
//           to all 16 CTAs, complete_tx on the receivers' mbarrier, waits for its own 16 slices
//   mode 1  MMA chain only: NMMA tcgen05.mma (M=128, N, K=16, A in TMEM) issued by 4 warps into
//           4 accumulators, commit, wait, tcgen05.ld of the accumulators, __syncthreads
//   mode 2  mode 0 + mode 1 in sequence (the r1 step skeleton)
//   mode 3  mode 2 with the MMAs of each group of 4 source CTAs issued as soon as that group's
//           slices arrived (per-group mbarriers)
//   mode 4  MMA chain only, ONE warp issuing all 32 MMAs into one accumulator (one commit)
//   mode 5  MMA chain only, 2 warps x 16 MMAs
//   mode 6  MMA chain only, 8 warps x 4 MMAs into 8 accumulators (each reader sums 8)
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1911_00357_b200/csrc \
//          tools/rnn_floor.cu -o tools/rnn_floor
// prints one line per (mode, N, B): cycles per step (CTA 0 clock64) and ns per step (%globaltimer).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "tc_util.cuh"

using namespace tcu;

namespace {
constexpr int kH = 512, kNC = 16, kUPC = 32, kThreads = 256;
constexpr uint32_t kSBO = (kH / 8) * 128;  // 8 rows x 512 K fp16 per 8-row group
struct Smem {
  unsigned char h_tile[2][2 * kSBO];
  unsigned char stage[2][512];
  uint64_t bar[2][4];
  uint64_t mma_bar;
  uint32_t tmem_slot;
};

__device__ __forceinline__ uint32_t htile_off(int r, int k) {
  return (uint32_t)((r >> 3) * kSBO + (k >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2);
}
__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <int MODE>
__global__ void __launch_bounds__(kThreads, 1) floor_kernel(int T, int B, int N, unsigned long long* out) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  const int c = (int)cluster_ctarank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int groups = MODE == 3 ? 4 : 1;
  for (int i = tid; i < (int)sizeof(sm.h_tile) / 16; i += kThreads)
    reinterpret_cast<uint4*>(sm.h_tile)[i] = make_uint4(0, 0, 0, 0);
  if (tid == 0) {
    for (int p = 0; p < 2; ++p)
      for (int g = 0; g < groups; ++g) mbar_init(&sm.bar[p][g], 1);
    mbar_init(&sm.mma_bar, MODE == 4 ? 1 : MODE == 5 ? 2 : MODE == 6 ? 8 : 4);
    fence_mbar_init_cluster();
  }
  if (warp == 0) tmem_alloc<512>(&sm.tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_slot;
  {
    uint32_t v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (warp < 4)
      for (int col = 0; col < 256; col += 8) tmem_st8(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)col, v);
    tmem_wait_st();
  }
  fence_proxy_async();
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  // packets: gate warp b, lane -> units 8*(lane%4) of env b to CTAs lane/4 and lane/4+8
  const bool gate_warp = warp < B;
  uint32_t pk_addr[2] = {0, 0}, pk_bar[2][2] = {{0, 0}, {0, 0}};
  if (gate_warp) {
    for (int j = 0; j < 2; ++j) {
      const uint32_t q = (uint32_t)(lane / 4 + 8 * j);
      pk_addr[j] = map_to_cta(sm.h_tile[0] + htile_off(warp, c * kUPC + 8 * (lane % 4)), q);
      const int g = MODE == 3 ? c / 4 : 0;
      pk_bar[j][0] = map_to_cta(&sm.bar[0][g], q);
      pk_bar[j][1] = map_to_cta(&sm.bar[1][g], q);
    }
  }
  const uint32_t tx_all = (uint32_t)(kNC * B * kUPC * 2), tx_grp = tx_all / 4;
  const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
  const uint32_t parity_bytes = (uint32_t)sizeof(sm.h_tile[0]);
  const uint32_t h_base0 = smem_u32(sm.h_tile[0]);
  const int nmma = kH / 16;  // 32 K steps of the hidden part
  __syncthreads();
  const long long c0 = clock64();
  const uint64_t g0 = gtimer();
  for (int t = 0; t < T; ++t) {
    const int cur = t & 1;
    if (MODE != 1 && MODE < 4 && t > 0 && warp < 4) {
      if (MODE == 3) {
        if (lane == 0) mbar_arrive_expect_tx(&sm.bar[cur][warp], tx_grp);
        mbar_wait_parity(&sm.bar[cur][warp], (uint32_t)(((t - 1) >> 1) & 1));
      } else {
        if (tid == 0) mbar_arrive_expect_tx(&sm.bar[cur][0], tx_all);
        mbar_wait_parity(&sm.bar[cur][0], (uint32_t)(((t - 1) >> 1) & 1));
      }
    }
    if (MODE == 0) __syncthreads();  // gate warps >= 4 (B = 8) wait for the slices too
    if (MODE == 6) {
      tc_fence_after();
      const uint64_t bd0 = umma_desc(h_base0 + (uint32_t)cur * parity_bytes, 128, kSBO);
      const uint32_t d_acc = tmem + 256u + 16u * (uint32_t)warp;
      for (int j = 0; j < nmma / 8; ++j) {
        const int kk = warp + 8 * j;
        mma_ts(d_acc, tmem + 8u * (uint32_t)kk, bd0 + (uint64_t)(16 * kk), idesc, (uint32_t)j);
      }
      mma_commit(&sm.mma_bar);
      if (warp < 4) {
        mbar_wait_parity(&sm.mma_bar, (uint32_t)(t & 1));
        tc_fence_after();
        uint32_t v[8][8];
        for (int a = 0; a < 8; ++a) tmem_ld8(tmem + ((uint32_t)(warp * 32) << 16) + 256u + 16u * (uint32_t)a, v[a]);
        tmem_wait_ld();
        if (v[0][0] == 12345u && v[7][7] == 54321u) out[1] = 1;
        tc_fence_before();
      }
      __syncthreads();
    } else if (MODE >= 4) {
      const int nw = MODE == 4 ? 1 : 2;
      if (warp < nw) {
        tc_fence_after();
        const uint64_t bd0 = umma_desc(h_base0 + (uint32_t)cur * parity_bytes, 128, kSBO);
        const uint32_t d_acc = tmem + 256u + 16u * (uint32_t)warp;
        for (int j = 0; j < nmma / nw; ++j) {
          const int kk = warp * (nmma / nw) + j;
          mma_ts(d_acc, tmem + 8u * (uint32_t)kk, bd0 + (uint64_t)(16 * kk), idesc, (uint32_t)j);
        }
        mma_commit(&sm.mma_bar);
      }
      if (warp < 4) {
        mbar_wait_parity(&sm.mma_bar, (uint32_t)(t & 1));
        tc_fence_after();
        uint32_t v[2][8];
        for (int a = 0; a < nw; ++a) tmem_ld8(tmem + ((uint32_t)(warp * 32) << 16) + 256u + 16u * (uint32_t)a, v[a]);
        tmem_wait_ld();
        if (v[0][0] == 12345u && v[nw - 1][7] == 54321u) out[1] = 1;
        tc_fence_before();
      }
      __syncthreads();
    } else if (MODE != 0) {
      if (warp < 4) {
        fence_proxy_async();
        tc_fence_after();
        const uint64_t bd0 = umma_desc(h_base0 + (uint32_t)cur * parity_bytes, 128, kSBO);
        const uint32_t d_acc = tmem + 256u + 16u * (uint32_t)warp;
        for (int j = 0; j < nmma / 4; ++j) {
          const int kk = MODE == 3 ? warp * (nmma / 4) + j : warp + 4 * j;
          mma_ts(d_acc, tmem + 8u * (uint32_t)kk, bd0 + (uint64_t)(16 * kk), idesc, (uint32_t)j);
        }
        mma_commit(&sm.mma_bar);
        mbar_wait_parity(&sm.mma_bar, (uint32_t)(t & 1));
        tc_fence_after();
        uint32_t v[4][8];
        for (int a = 0; a < 4; ++a) tmem_ld8(tmem + ((uint32_t)(warp * 32) << 16) + 256u + 16u * (uint32_t)a, v[a]);
        tmem_wait_ld();
        if (v[0][0] == 12345u && v[3][7] == 54321u) out[1] = 1;  // keep the loads
        tc_fence_before();
      }
      __syncthreads();
    }
    if (MODE != 1 && MODE < 4 && gate_warp && t + 1 < T) {
      __half* st = reinterpret_cast<__half*>(sm.stage[cur]) + warp * kUPC;
      st[lane] = __float2half((float)t);
      __syncwarp();
      const uint4 pkt = *reinterpret_cast<const uint4*>(st + 8 * (lane % 4));
      const uint32_t off = (uint32_t)(cur ^ 1) * parity_bytes;
      st_async_v4(pk_addr[0] + off, pkt, pk_bar[0][cur ^ 1]);
      st_async_v4(pk_addr[1] + off, pkt, pk_bar[1][cur ^ 1]);
    }
  }
  __syncthreads();
  const long long c1 = clock64();
  const uint64_t g1 = gtimer();
  if (c == 0 && tid == 0) {
    out[0] = (unsigned long long)(c1 - c0);
    out[2] = g1 - g0;
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

template <int MODE>
void run(int T, int B, int N, unsigned long long* d_out) {
  auto k = floor_kernel<MODE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem));
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kNC);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = sizeof(Smem);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kNC;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  unsigned long long h[3];
  double best_c = 1e30, best_ns = 1e30;
  for (int rep = 0; rep < 5; ++rep) {
    cudaError_t e = cudaLaunchKernelEx(&cfg, k, T, B, N, d_out);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("mode %d: %s\n", MODE, cudaGetErrorString(e));
      exit(1);
    }
    cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
    if ((double)h[0] / T < best_c) best_c = (double)h[0] / T;
    if ((double)h[2] / T < best_ns) best_ns = (double)h[2] / T;
  }
  static const char* names[7] = {"exchange only", "MMA chain only", "exchange + MMA (serial)",
                                 "exchange + MMA (per-group overlap)", "MMA chain, 1 issuing warp",
                                 "MMA chain, 2 issuing warps", "MMA chain, 8 issuing warps"};
  printf("mode %d %-36s N=%2d B=%d : %7.1f cycles/step  %7.1f ns/step\n", MODE, names[MODE], N, B, best_c, best_ns);
}
}  // namespace

int main() {
  unsigned long long* d_out;
  cudaMalloc(&d_out, 64);
  const int T = 4096;
  for (int N : {16, 8}) {
    run<4>(T, 2, N, d_out);
    run<5>(T, 2, N, d_out);
    run<1>(T, 2, N, d_out);
    run<6>(T, 2, N, d_out);
  }
  for (int B : {2, 8}) {
    run<0>(T, B, 16, d_out);
    for (int N : {16, 8}) {
      run<1>(T, B, N, d_out);
      run<2>(T, B, N, d_out);
      run<3>(T, B, N, d_out);
    }
  }
  return 0;
}
