// a8 over NVLink peer memory (K16 v2): the gradient AllReduce-mean fused with the clip norm, then
// the Adam update -- no NCCL on the learner's critical path.
//
// P:L150-158 (Eq. 3): every worker applies ParamUpdate(theta, (1/N) sum_i grad_i).  Here each rank
// exposes its learner workspace to the others through CUDA IPC (handles exchanged once with an
// NCCL all-gather); per minibatch every rank
//   1. signals "my gradient is final" into every peer's flag slot (st.release.sys) and waits for
//      all N signals (ld.acquire.sys, bounded spin -> error flag instead of a hang) -- one warp,
//      so the reduction kernel behind it starts only when every gradient is final,
//   2. reads the N gradients over NVLink and sums them in rank order 0..N-1 (so every rank holds
//      bit-identical sums: parameters stay identical without a broadcast), accumulating the
//      squared norm of the mean in fp64 with the fixed-order last-block reduction,
//   3. runs the existing fused Adam kernel on the summed gradient (adam.cu).
// The gradient buffers are double-buffered by minibatch parity: a rank overwrites gradient buffer
// k%2 only in minibatch k+2, after minibatch k+1's barrier proved that every peer has finished
// reading it.
#include <string.h>

#include <vector>

#include "common.cuh"

namespace {

constexpr int kThreads = 256;
constexpr long long kSpinLimit = 1LL << 31;  // ~seconds: a peer that never arrives sets the error flag

__device__ __forceinline__ void st_release_sys(unsigned int* p, unsigned int v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned int ld_acquire_sys(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

struct PeerArgs {
  const float* grad[kMaxPeers];        // rank j's gradient buffer (this minibatch's parity)
  unsigned int* flags[kMaxPeers];      // rank j's flag array [kMaxPeers]
};

// one warp: lane j signals rank j ("my gradient is final") and then waits for rank j's signal
__global__ void peer_barrier_kernel(const PeerArgs args, int world, int rank, unsigned int* d_epoch, int* err) {
  const int j = threadIdx.x;
  unsigned int epoch = 0;
  if (j == 0) {
    epoch = *d_epoch + 1;  // every rank advances its own counter identically (one barrier per minibatch)
    *d_epoch = epoch;
  }
  epoch = __shfl_sync(0xffffffffu, epoch, 0);
  if (j < world) {
    __threadfence_system();  // this rank's gradient (earlier kernels) before the signal
    st_release_sys(args.flags[j] + rank, epoch);
    long long spins = 0;
    while ((int)(ld_acquire_sys(args.flags[rank] + j) - epoch) < 0) {
      if (++spins > kSpinLimit) {
        atomicOr(err, ERR_BIT_COMM);
        break;
      }
    }
  }
}

__global__ void __launch_bounds__(kThreads)
peer_reduce_norm_kernel(const PeerArgs args, int world, int64_t P, float inv_world, float max_norm,
                        float* __restrict__ gsum, double* partials, unsigned int* counter, float* scalars,
                        float* grad_norm_out, int* err) {
  __shared__ double red[kThreads / 32];
  __shared__ double fin[1];
  double acc[1] = {0.0};
  const int64_t P4 = P / 4, stride = (int64_t)gridDim.x * blockDim.x;
  float s = 0.f;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P4; i += stride) {
    float4 u[kMaxPeers];
#pragma unroll
    for (int j = 0; j < kMaxPeers; ++j)  // all loads in flight before the (rank-ordered) sums
      if (j < world) u[j] = __ldcg(reinterpret_cast<const float4*>(args.grad[j]) + i);
    float4 t = u[0];
#pragma unroll
    for (int j = 1; j < kMaxPeers; ++j)
      if (j < world) {
        t.x += u[j].x;
        t.y += u[j].y;
        t.z += u[j].z;
        t.w += u[j].w;
      }
    reinterpret_cast<float4*>(gsum)[i] = t;
    const float a = t.x * inv_world, b = t.y * inv_world, c = t.z * inv_world, d = t.w * inv_world;
    s += a * a + b * b + c * c + d * d;
  }
  for (int64_t i = P4 * 4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += stride) {
    float t = __ldcg(args.grad[0] + i);
    for (int j = 1; j < world; ++j) t += __ldcg(args.grad[j] + i);
    gsum[i] = t;
    s += (t * inv_world) * (t * inv_world);
  }
  acc[0] = (double)s;
  if (last_block_reduce<1>(acc, partials, counter, fin, red)) {
    if (threadIdx.x == 0) {
      const double total = sqrt(fin[0]);
      double coef = 1.0;
      if (max_norm > 0.f) coef = fmin(1.0, (double)max_norm / (total + 1e-6));
      scalars[0] = (float)coef * inv_world;
      scalars[1] = (float)total;
      if (grad_norm_out) grad_norm_out[0] = (float)total;
      if (!isfinite(total)) atomicOr(err, ERR_BIT_GRAD);
    }
  }
}

// base address of the device allocation holding p (driver API through the runtime's entry point)
typedef int (*MemGetAddressRange)(unsigned long long*, size_t*, unsigned long long);
ddppo_status allocation_base(ddppo_ctx* ctx, const void* p, char** base) {
  static MemGetAddressRange fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    DDPPO_CUDA_TRY(ctx, cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q));
    DDPPO_REQUIRE(ctx, f != nullptr && q == cudaDriverEntryPointSuccess, "peer: cuMemGetAddressRange unavailable");
    fn = reinterpret_cast<MemGetAddressRange>(f);
  }
  unsigned long long b = 0;
  size_t sz = 0;
  DDPPO_REQUIRE(ctx, fn(&b, &sz, (unsigned long long)(uintptr_t)p) == 0, "peer: address is not device memory");
  *base = reinterpret_cast<char*>(b);
  return DDPPO_OK;
}

// One IPC-shared area per rank: the learner barrier's flags (first, peer_flags[j] points here), the
// counts exchange's flags and its values, double-buffered by epoch parity: rank r writes slot
// [e & 1][r] of every peer's area, then signals; a rank can only reach epoch e + 2 after every peer
// signalled e + 1, i.e. after every peer finished reading epoch e's values.
struct PeerArea {
  unsigned int flags[kMaxPeers];
  unsigned int cnt_flags[kMaxPeers];
  long long vals[2][kMaxPeers][kMaxCountVals];
};

struct CountArgs {
  PeerArea* area[kMaxPeers];
  long long v[kMaxCountVals];
};

__global__ void peer_counts_kernel(const CountArgs a, int world, int rank, int n, unsigned int* d_epoch,
                                   long long* out, int* err) {
  __shared__ unsigned int s_epoch;
  if (threadIdx.x == 0) {
    s_epoch = *d_epoch + 1;
    *d_epoch = s_epoch;
  }
  __syncthreads();
  const unsigned int epoch = s_epoch;
  const int par = (int)(epoch & 1u);
  const int j = threadIdx.x;
  if (j < world) {
    for (int i = 0; i < n; ++i) a.area[j]->vals[par][rank][i] = a.v[i];
    __threadfence_system();
    st_release_sys(&a.area[j]->cnt_flags[rank], epoch);
    long long spins = 0;
    while ((int)(ld_acquire_sys(&a.area[rank]->cnt_flags[j]) - epoch) < 0) {
      if (++spins > kSpinLimit) {
        atomicOr(err, ERR_BIT_COMM);
        break;
      }
    }
  }
  __syncthreads();
  if (j < n) {
    long long t = 0;
    for (int r = 0; r < world; ++r) t += ((volatile long long*)a.area[rank]->vals[par][r])[j];  // rank order
    out[j] = t;
  }
}

struct Shared {
  cudaIpcMemHandle_t handle;
  unsigned long long offset;
};

}  // namespace

// Exchange IPC handles of the allocations holding `local` (this rank) so that out[j] is rank j's
// corresponding address; out[rank] = local.  Collective.
ddppo_status peer_exchange(ddppo_ctx* ctx, void* local, void** out) {
  char* base = nullptr;
  ddppo_status s = allocation_base(ctx, local, &base);
  if (s != DDPPO_OK) return s;
  Shared mine;
  memset(&mine, 0, sizeof(mine));
  DDPPO_CUDA_TRY(ctx, cudaIpcGetMemHandle(&mine.handle, base));
  mine.offset = (unsigned long long)((char*)local - base);
  const int W = ctx->world;
  std::vector<Shared> all(W);
  char* dbuf = nullptr;
  DDPPO_CUDA_TRY(ctx, cudaMalloc(&dbuf, sizeof(Shared) * W));
  DDPPO_CUDA_TRY(ctx, cudaMemcpy(dbuf + sizeof(Shared) * ctx->rank, &mine, sizeof(Shared), cudaMemcpyHostToDevice));
  ncclResult_t nr = ncclAllGather(dbuf + sizeof(Shared) * ctx->rank, dbuf, sizeof(Shared), ncclChar, ctx->comm, 0);
  if (nr != ncclSuccess) {
    cudaFree(dbuf);
    ctx->last_error = std::string("peer exchange: ") + ncclGetErrorString(nr);
    return DDPPO_ERR_COMM;
  }
  DDPPO_CUDA_TRY(ctx, cudaMemcpy(all.data(), dbuf, sizeof(Shared) * W, cudaMemcpyDeviceToHost));
  cudaFree(dbuf);
  for (int j = 0; j < W; ++j) {
    if (j == ctx->rank) {
      out[j] = local;
      continue;
    }
    void* pb = nullptr;
    DDPPO_CUDA_TRY(ctx, cudaIpcOpenMemHandle(&pb, all[j].handle, cudaIpcMemLazyEnablePeerAccess));
    ctx->ipc_opened.push_back(pb);
    out[j] = (char*)pb + all[j].offset;
  }
  return DDPPO_OK;
}

ddppo_status peer_setup_flags(ddppo_ctx* ctx) {
  if (ctx->peer_flags[ctx->rank]) return DDPPO_OK;
  unsigned int* f = nullptr;
  DDPPO_CUDA_TRY(ctx, cudaMalloc(&f, sizeof(PeerArea)));
  DDPPO_CUDA_TRY(ctx, cudaMemset(f, 0, sizeof(PeerArea)));
  DDPPO_CUDA_TRY(ctx, cudaDeviceSynchronize());
  ctx->own_flags = f;
  DDPPO_CUDA_TRY(ctx, cudaMalloc(&ctx->d_peer_epoch, 2 * sizeof(unsigned int)));
  DDPPO_CUDA_TRY(ctx, cudaMemset(ctx->d_peer_epoch, 0, 2 * sizeof(unsigned int)));
  ctx->d_cnt_epoch = ctx->d_peer_epoch + 1;
  DDPPO_CUDA_TRY(ctx, cudaDeviceSynchronize());
  void* out[kMaxPeers] = {};
  ddppo_status s = peer_exchange(ctx, f, out);
  if (s != DDPPO_OK) return s;
  for (int j = 0; j < ctx->world; ++j) ctx->peer_flags[j] = reinterpret_cast<unsigned int*>(out[j]);
  return DDPPO_OK;
}

// sum over ranks (rank order) of grad buffers peers[j] -> gsum, clip coefficient -> ctx scalars
ddppo_status launch_peer_reduce_norm(ddppo_ctx* ctx, float* const* peers, float* gsum, int64_t P, float max_norm,
                                     float* grad_norm, cudaStream_t st) {
  DDPPO_REQUIRE(ctx, ctx->world <= kMaxPeers && ctx->peer_flags[ctx->rank], "peer: flags not set up");
  PeerArgs a;
  for (int j = 0; j < ctx->world; ++j) {
    a.grad[j] = peers[j];
    a.flags[j] = ctx->peer_flags[j];
    DDPPO_REQUIRE(ctx, (uintptr_t)peers[j] % 16 == 0, "peer: gradient buffers must be 16-byte aligned");
  }
  peer_barrier_kernel<<<1, 32, 0, st>>>(a, ctx->world, ctx->rank, ctx->d_peer_epoch, ctx->d_err);
  const int blocks = grid_for((int)std::min<int64_t>((P + 3) / 4, 1 << 30), kThreads, ctx->sm_count * 4);
  peer_reduce_norm_kernel<<<blocks, kThreads, 0, st>>>(a, ctx->world, P, 1.f / (float)ctx->world, max_norm, gsum,
                                                       ctx->d_partials, ctx->d_counters + CNT_NORM, ctx->d_scalars,
                                                       grad_norm, ctx->d_err);
  ctx->count(2);
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  return DDPPO_OK;
}

ddppo_status peer_allreduce_counts(ddppo_ctx* ctx, int64_t* host_vals, int n) {
  DDPPO_REQUIRE(ctx, ctx->world <= kMaxPeers && ctx->peer_flags[ctx->rank] && n <= kMaxCountVals,
                "peer counts: flags not set up");
  if (!ctx->cnt_stream) {
    DDPPO_CUDA_TRY(ctx, cudaStreamCreateWithFlags(&ctx->cnt_stream, cudaStreamNonBlocking));
    DDPPO_CUDA_TRY(ctx, cudaMallocHost(&ctx->h_cnt, kMaxCountVals * sizeof(int64_t)));
  }
  CountArgs a;
  memset(&a, 0, sizeof(a));
  for (int j = 0; j < ctx->world; ++j) a.area[j] = reinterpret_cast<PeerArea*>(ctx->peer_flags[j]);
  for (int i = 0; i < n; ++i) a.v[i] = (long long)host_vals[i];
  peer_counts_kernel<<<1, 64, 0, ctx->cnt_stream>>>(a, ctx->world, ctx->rank, n, ctx->d_cnt_epoch,
                                                     reinterpret_cast<long long*>(ctx->d_i64), ctx->d_err);
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  DDPPO_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->h_cnt, ctx->d_i64, n * sizeof(int64_t), cudaMemcpyDeviceToHost,
                                      ctx->cnt_stream));
  DDPPO_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->cnt_stream));
  for (int i = 0; i < n; ++i) host_vals[i] = ctx->h_cnt[i];
  return DDPPO_OK;
}
