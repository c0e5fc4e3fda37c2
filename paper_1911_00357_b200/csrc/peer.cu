// a8 over NVLink peer memory: the gradient AllReduce-mean fused with the clip norm and Adam -- no
// NCCL on the learner's critical path.
//
// P:L150-158 (Eq. 3): every worker applies ParamUpdate(theta, (1/N) sum_i grad_i).  Each rank
// exposes its learner workspace to the others through CUDA IPC (handles exchanged once with an NCCL
// all-gather) plus one small flag area (PeerArea).  Per minibatch:
//
//   barrier      one warp: lane j signals "my gradient is final" into rank j's flag slot
//                (st.release.sys) and waits for rank j's signal (ld.acquire.sys, bounded by
//                %globaltimer -> ERR_BIT_COMM instead of a hang; every later kernel of the exchange
//                then leaves the parameters untouched and ddppo_check reports ERR_COMM).
//
//   v1 (all-read, DDPPO_A8_ALLREAD): every rank reads all N gradients over NVLink, sums them in rank
//      order 0..N-1 (bit-identical sums everywhere, so parameters stay identical without a
//      broadcast) with the clip norm in the same pass, then the full Adam: (N-1)*4P bytes read
//      per rank, the whole Adam on every rank.
//
//   v2 (sharded, DDPPO_A8_SHARDED, default; the ZeRO-1 form of NEXT-2): rank r owns the 1/N shard
//      [lo_r, hi_r) of the flat parameter vector.
//      rs_norm    reduce-scatter: rank r sums the N ranks' gradient shards in rank order (the same
//                 per-element arithmetic as v1) and its shard's sum of squares (fixed-order
//                 last-block reduction); the last block pushes that fp64 partial into every peer's
//                 area and releases a flag
//      adam_shard waits for the N partials, adds them in rank order (every rank the same coef),
//                 applies clip + Adam to its shard only (m / v are meaningful on the owned shard),
//                 stages the updated shard in its workspace and releases a flag
//      ag         all-gather: waits for the N flags and copies every other rank's updated shard
//                 from that rank's workspace into its own parameters.
//      NVLink bytes per rank: 2(N-1)/N * 4P (ring-allreduce volume) instead of (N-1) * 4P, and
//      Adam runs on P/N elements.
//
// Buffer reuse (why no extra barrier is needed): gradient buffers are double-buffered by
// minibatch parity -- a rank rewrites buffer k%2 in minibatch k+2, after minibatch k+1's barrier,
// which every peer passes only after its minibatch-k reads.  The norm partial slots are
// double-buffered by epoch parity (a rank writes epoch e+2's slot only after the barrier of
// e+2, i.e. after every peer consumed epoch e's partials in its adam_shard).  The staged shard
// (pgather) of minibatch k is read by the peers' ag of minibatch k, which precedes (stream
// order) their minibatch-(k+1) barrier signal, which the owner's adam_shard of k+1 waits for.
#include <string.h>

#include <vector>

#include "common.cuh"

namespace {

constexpr int kThreads = 256;
constexpr unsigned long long kTimeoutNs = 30ull * 1000 * 1000 * 1000;  // a peer that never arrives

__device__ __forceinline__ void st_release_sys(unsigned int* p, unsigned int v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned int ld_acquire_sys(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// wait until *flag has reached epoch (wrap-safe); false (and ERR_BIT_COMM) after kTimeoutNs
__device__ __forceinline__ bool wait_epoch(const unsigned int* flag, unsigned int epoch, int* err) {
  if ((int)(ld_acquire_sys(flag) - epoch) >= 0) return true;
  const unsigned long long t0 = globaltimer();
  for (;;) {
    for (int i = 0; i < 64; ++i)
      if ((int)(ld_acquire_sys(flag) - epoch) >= 0) return true;
    if (globaltimer() - t0 > kTimeoutNs) {
      atomicOr(err, ERR_BIT_COMM);
      return false;
    }
  }
}
__device__ __forceinline__ bool comm_failed(const int* err) {
  return (*(volatile const int*)err & (ERR_BIT_COMM | ERR_BIT_GRAD)) != 0;
}

}  // namespace

// One IPC-shared area per rank.  flags: the gradient barrier; norm_flags / norm_part: the sharded
// clip-norm partials (slot [epoch & 1][rank]); ag_flags: "my updated shard is staged"; cnt_*: the
// a10 counts exchange (values double-buffered by epoch parity).
struct PeerArea {
  unsigned int flags[kMaxPeers];
  unsigned int cnt_flags[kMaxPeers];
  unsigned int norm_flags[kMaxPeers];
  unsigned int ag_flags[kMaxPeers];
  double norm_part[2][kMaxPeers];
  long long vals[2][kMaxPeers][kMaxCountVals];
};

namespace {

struct PeerArgs {
  const float* grad[kMaxPeers];  // rank j's gradient buffer (this minibatch's parity)
  const float* pg[kMaxPeers];    // rank j's staged updated shard (v2)
  PeerArea* area[kMaxPeers];
};

// shard of rank r in float4 units: [q_lo, q_hi); the last shard also owns the scalar tail
__host__ __device__ __forceinline__ int64_t shard_q(int64_t Q, int world, int r) { return Q * r / world; }

// one warp per emulated rank (production: one warp, rank_base = rank): lane j signals rank j and
// waits for rank j's signal.  d_epoch[w] is rank (rank_base + w)'s barrier epoch.
__global__ void peer_barrier_kernel(const PeerArgs args, int world, int rank_base, unsigned int* d_epoch, int* err) {
  const int w = threadIdx.x >> 5, j = threadIdx.x & 31, rank = rank_base + w;
  unsigned int epoch = 0;
  if (j == 0) {
    epoch = d_epoch[w] + 1;  // every rank advances its own counter identically (one barrier per minibatch)
    d_epoch[w] = epoch;
  }
  epoch = __shfl_sync(0xffffffffu, epoch, 0);
  if (j < world) {
    __threadfence_system();  // this rank's gradient (earlier kernels) before the signal
    st_release_sys(&args.area[j]->flags[rank], epoch);
    wait_epoch(&args.area[rank]->flags[j], epoch, err);
  }
}

// v1: gsum = sum_j grad_j (rank order) over all P, clip coefficient -> scalars
__global__ void __launch_bounds__(kThreads)
peer_reduce_norm_kernel(const PeerArgs args, int world, int64_t P, float inv_world, float max_norm,
                        float* __restrict__ gsum, double* partials, unsigned int* counter, float* scalars,
                        float* grad_norm_out, int* err) {
  __shared__ double red[kThreads / 32];
  __shared__ double fin[1];
  if (comm_failed(err)) return;
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

// v2 reduce-scatter: gsum[shard] = sum_j grad_j[shard] (rank order); the shard's sum of squares of
// the mean goes to every rank's norm_part[epoch & 1][rank], then norm_flags[rank] = epoch.
__global__ void __launch_bounds__(kThreads)
peer_rs_norm_kernel(const PeerArgs args, int world, int rank, int64_t P, float inv_world, float* __restrict__ gsum,
                    double* partials, unsigned int* counter, const unsigned int* d_epoch, int* err) {
  __shared__ double red[kThreads / 32];
  __shared__ double fin[1];
  if (comm_failed(err)) return;
  const int64_t Q = P / 4, q0 = shard_q(Q, world, rank), q1 = shard_q(Q, world, rank + 1);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  float s = 0.f;
  for (int64_t i = q0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < q1; i += stride) {
    float4 u[kMaxPeers];
#pragma unroll
    for (int j = 0; j < kMaxPeers; ++j)
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
  if (rank == world - 1)
    for (int64_t i = Q * 4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += stride) {
      float t = __ldcg(args.grad[0] + i);
      for (int j = 1; j < world; ++j) t += __ldcg(args.grad[j] + i);
      gsum[i] = t;
      s += (t * inv_world) * (t * inv_world);
    }
  double acc[1] = {(double)s};
  if (last_block_reduce<1>(acc, partials, counter, fin, red)) {
    if (threadIdx.x == 0) {
      const unsigned int epoch = *d_epoch;
      for (int j = 0; j < world; ++j) args.area[j]->norm_part[epoch & 1u][rank] = fin[0];
      __threadfence_system();
      for (int j = 0; j < world; ++j) st_release_sys(&args.area[j]->norm_flags[rank], epoch);
    }
  }
}

// v2: clip coefficient from the N shard partials (rank order), Adam on the owned shard, the updated
// shard staged in pgather (own workspace), then ag_flags[rank] = epoch in every rank's area.
__global__ void __launch_bounds__(kThreads)
peer_adam_shard_kernel(const PeerArgs args, int world, int rank, int64_t P, const float* __restrict__ gsum,
                       float* __restrict__ p, float* __restrict__ m, float* __restrict__ v, float* __restrict__ pgather,
                       float inv_world, float max_norm, float b1, float b2, float lr, float eps, const int* dstep,
                       int step_add, const unsigned int* d_epoch, unsigned int* counter, float* grad_norm_out,
                       int* err, const uint8_t* __restrict__ freeze, int64_t frz_end) {
  __shared__ float sc[3];
  __shared__ int ok;
  __shared__ bool am_last;
  if (threadIdx.x == 0) {
    ok = 0;
    if (!comm_failed(err)) {
      const unsigned int epoch = *d_epoch;
      bool all = true;
      for (int j = 0; j < world && all; ++j) all = wait_epoch(&args.area[rank]->norm_flags[j], epoch, err);
      if (all) {
        double sq = 0.0;
        for (int j = 0; j < world; ++j) sq += ((volatile double*)args.area[rank]->norm_part[epoch & 1u])[j];
        const double total = sqrt(sq);
        double coef = 1.0;
        if (max_norm > 0.f) coef = fmin(1.0, (double)max_norm / (total + 1e-6));
        const int step = (dstep ? *dstep : 0) + step_add;
        const double bc1 = 1.0 - pow((double)b1, (double)step), bc2 = 1.0 - pow((double)b2, (double)step);
        sc[0] = (float)coef * inv_world;
        sc[1] = (float)((double)lr / bc1);
        sc[2] = (float)(1.0 / sqrt(bc2));
        if (blockIdx.x == 0 && grad_norm_out) grad_norm_out[0] = (float)total;
        if (isfinite(total)) ok = 1;
        else atomicOr(err, ERR_BIT_GRAD);  // identical on every rank: nobody updates
      }
    }
  }
  __syncthreads();
  if (!ok) return;
  const float scale = sc[0], step_size = sc[1], inv_sqrt_bc2 = sc[2];
  const int64_t Q = P / 4, q0 = shard_q(Q, world, rank), q1 = shard_q(Q, world, rank + 1);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = q0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < q1; i += stride) {
    float4 pp = reinterpret_cast<float4*>(p)[i];
    if (i < frz_end / 4) {  // frozen prefix: staged unchanged (the peers copy it back)
      reinterpret_cast<float4*>(pgather)[i] = pp;
      continue;
    }
    const float4 gg = reinterpret_cast<const float4*>(gsum)[i];
    float4 mm = reinterpret_cast<float4*>(m)[i];
    float4 vv = reinterpret_cast<float4*>(v)[i];
    const float4 po = pp, mo = mm, vo = vv;
    adam_one(pp.x, mm.x, vv.x, gg.x * scale, b1, b2, step_size, inv_sqrt_bc2, eps);
    adam_one(pp.y, mm.y, vv.y, gg.y * scale, b1, b2, step_size, inv_sqrt_bc2, eps);
    adam_one(pp.z, mm.z, vv.z, gg.z * scale, b1, b2, step_size, inv_sqrt_bc2, eps);
    adam_one(pp.w, mm.w, vv.w, gg.w * scale, b1, b2, step_size, inv_sqrt_bc2, eps);
    if (freeze) {
      const uint32_t fr = reinterpret_cast<const uint32_t*>(freeze)[i];
      if (fr & 0xffu) { pp.x = po.x; mm.x = mo.x; vv.x = vo.x; }
      if (fr & 0xff00u) { pp.y = po.y; mm.y = mo.y; vv.y = vo.y; }
      if (fr & 0xff0000u) { pp.z = po.z; mm.z = mo.z; vv.z = vo.z; }
      if (fr & 0xff000000u) { pp.w = po.w; mm.w = mo.w; vv.w = vo.w; }
    }
    reinterpret_cast<float4*>(p)[i] = pp;
    reinterpret_cast<float4*>(m)[i] = mm;
    reinterpret_cast<float4*>(v)[i] = vv;
    reinterpret_cast<float4*>(pgather)[i] = pp;
  }
  if (rank == world - 1)
    for (int64_t i = Q * 4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += stride) {
      if (freeze && freeze[i]) {
        pgather[i] = p[i];
        continue;
      }
      float pp = p[i], mm = m[i], vv = v[i];
      adam_one(pp, mm, vv, gsum[i] * scale, b1, b2, step_size, inv_sqrt_bc2, eps);
      p[i] = pp;
      m[i] = mm;
      v[i] = vv;
      pgather[i] = pp;
    }
  // the last block to finish publishes the staged shard
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    am_last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (am_last && threadIdx.x == 0) {
    *counter = 0u;
    __threadfence_system();
    const unsigned int epoch = *d_epoch;
    for (int j = 0; j < world; ++j) st_release_sys(&args.area[j]->ag_flags[rank], epoch);
  }
}

// v2 all-gather: params[shard j] = rank j's staged shard, for every j != rank
__global__ void __launch_bounds__(kThreads)
peer_ag_kernel(const PeerArgs args, int world, int rank, int64_t P, float* __restrict__ p,
               const unsigned int* d_epoch, int* err) {
  __shared__ int ok;
  if (threadIdx.x == 0) {
    ok = 0;
    if (!comm_failed(err)) {
      const unsigned int epoch = *d_epoch;
      bool all = true;
      for (int j = 0; j < world && all; ++j)
        if (j != rank) all = wait_epoch(&args.area[rank]->ag_flags[j], epoch, err);
      ok = all ? 1 : 0;
    }
  }
  __syncthreads();
  if (!ok) return;
  const int64_t Q = P / 4, stride = (int64_t)gridDim.x * blockDim.x;
  for (int j = 0; j < world; ++j) {
    if (j == rank) continue;
    const int64_t q0 = shard_q(Q, world, j), q1 = shard_q(Q, world, j + 1);
    for (int64_t i = q0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < q1; i += stride)
      reinterpret_cast<float4*>(p)[i] = __ldcg(reinterpret_cast<const float4*>(args.pg[j]) + i);
    if (j == world - 1)
      for (int64_t i = Q * 4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += stride)
        p[i] = __ldcg(args.pg[j] + i);
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

struct CountArgs {
  PeerArea* area[kMaxPeers];
  long long v[kMaxPeers][kMaxCountVals];  // row b: the values of emulated rank rank_base + b (row 0 in production)
};

// one block per emulated rank (production: one block, rank_base = rank): push this rank's values into
// every peer's area (slot [epoch & 1][rank]), signal, wait for every peer's signal, sum in rank order
__global__ void peer_counts_kernel(const CountArgs a, int world, int rank_base, int n, unsigned int* d_epoch,
                                   long long* out, int* err) {
  __shared__ unsigned int s_epoch;
  __shared__ int ok;
  const int b = blockIdx.x, rank = rank_base + b;
  if (threadIdx.x == 0) {
    s_epoch = d_epoch[b] + 1;
    d_epoch[b] = s_epoch;
    ok = 1;
  }
  __syncthreads();
  const unsigned int epoch = s_epoch;
  const int par = (int)(epoch & 1u);
  const int j = threadIdx.x;
  if (j < world) {
    for (int i = 0; i < n; ++i) a.area[j]->vals[par][rank][i] = a.v[b][i];
    __threadfence_system();
    st_release_sys(&a.area[j]->cnt_flags[rank], epoch);
    if (!wait_epoch(&a.area[rank]->cnt_flags[j], epoch, err)) ok = 0;
  }
  __syncthreads();
  if (j < n && ok) {
    long long t = 0;
    for (int r = 0; r < world; ++r) t += ((volatile long long*)a.area[rank]->vals[par][r])[j];  // rank order
    out[(size_t)b * kMaxCountVals + j] = t;
  }
}

struct Shared {
  cudaIpcMemHandle_t handle;
  unsigned long long offset;
};

int a8_blocks(ddppo_ctx* ctx, int64_t n) {
  return grid_for((int)std::min<int64_t>((n + 3) / 4, 1 << 30), kThreads, ctx->sm_count * 4);
}

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

// The whole a8 of one minibatch for `rank` over N ranks' buffers.  grads[j] / pgs[j]: rank j's
// gradient / staged-shard buffer as addressed from this rank; areas[j]: rank j's PeerArea.
// barrier: whether to run the barrier kernel (the single-device emulation runs it once for all).
static ddppo_status a8_rank(ddppo_ctx* ctx, int mode, int world, int rank, float* const* grads, float* const* pgs,
                            PeerArea* const* areas, unsigned int* d_epoch, bool barrier, float* gsum, float* params,
                            float* m, float* v, int64_t P, const ddppo_adam_cfg& cfg, const int* dstep, int step_add,
                            float* grad_norm, cudaStream_t st, const uint8_t* freeze = nullptr,
                            int64_t frz_end = 0) {
  PeerArgs a;
  memset(&a, 0, sizeof(a));
  for (int j = 0; j < world; ++j) {
    a.grad[j] = grads[j];
    a.pg[j] = pgs ? pgs[j] : nullptr;
    a.area[j] = areas[j];
    DDPPO_REQUIRE(ctx, (uintptr_t)grads[j] % 16 == 0, "peer: gradient buffers must be 16-byte aligned");
  }
  if (barrier) {
    peer_barrier_kernel<<<1, 32, 0, st>>>(a, world, rank, d_epoch, ctx->d_err);
    ctx->count(1);
  }
  const float inv_world = 1.f / (float)world;
  if (mode == DDPPO_A8_ALLREAD) {
    peer_reduce_norm_kernel<<<a8_blocks(ctx, P), kThreads, 0, st>>>(a, world, P, inv_world, cfg.max_grad_norm, gsum,
                                                                    ctx->d_partials, ctx->d_counters + CNT_NORM,
                                                                    ctx->d_scalars, grad_norm, ctx->d_err);
    ctx->count(1);
    DDPPO_CUDA_TRY(ctx, cudaGetLastError());
    return launch_adam_only(ctx, gsum, params, m, v, freeze, P, cfg, dstep, step_add, st, frz_end);
  }
  DDPPO_REQUIRE(ctx, pgs != nullptr, "peer: sharded a8 needs staged-shard buffers");
  const int64_t shard = (P + world - 1) / world;
  const int blocks = a8_blocks(ctx, shard);
  peer_rs_norm_kernel<<<blocks, kThreads, 0, st>>>(a, world, rank, P, inv_world, gsum, ctx->d_partials,
                                                   ctx->d_counters + CNT_NORM, d_epoch, ctx->d_err);
  {
    ProfScope ps(ctx, DDPPO_K_ADAM, st, 0);
    peer_adam_shard_kernel<<<blocks, kThreads, 0, st>>>(a, world, rank, P, gsum, params, m, v, pgs[rank], inv_world,
                                                        cfg.max_grad_norm, cfg.beta1, cfg.beta2, cfg.lr, cfg.eps, dstep,
                                                        step_add, d_epoch, ctx->d_counters + CNT_MISC, grad_norm,
                                                        ctx->d_err, freeze, frz_end);
  }
  peer_ag_kernel<<<a8_blocks(ctx, P - shard), kThreads, 0, st>>>(a, world, rank, P, params, d_epoch, ctx->d_err);
  ctx->count(3);
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  return DDPPO_OK;
}

ddppo_status launch_peer_a8(ddppo_ctx* ctx, float* const* peers, float* const* pgs, float* gsum, float* params,
                            float* m, float* v, int64_t P, const ddppo_adam_cfg& cfg, const int* dstep, int step_add,
                            cudaStream_t st, const uint8_t* freeze, int64_t frz_end) {
  DDPPO_REQUIRE(ctx, ctx->world <= kMaxPeers && ctx->peer_flags[ctx->rank], "peer: flags not set up");
  PeerArea* areas[kMaxPeers];
  for (int j = 0; j < ctx->world; ++j) areas[j] = reinterpret_cast<PeerArea*>(ctx->peer_flags[j]);
  int mode = ctx->a8_mode;
  if (mode == DDPPO_A8_AUTO) {  // include/ddppo.h: the cheaper form under the bytes + synchronisation model
    const double N = ctx->world;
    const double extra_read_s = (N - 1.0) * (1.0 - 2.0 / N) * 4.0 * (double)P / 770e9;
    const double adam_saved_s = (1.0 - 1.0 / N) * 28.0 * (double)P / 6.5e12;
    mode = extra_read_s + adam_saved_s > 20e-6 ? DDPPO_A8_SHARDED : DDPPO_A8_ALLREAD;
  }
  return a8_rank(ctx, mode, ctx->world, ctx->rank, peers, pgs, areas, ctx->d_peer_epoch, true, gsum, params,
                 m, v, P, cfg, dstep, step_add, nullptr, st, freeze, frz_end);
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
  for (int i = 0; i < n; ++i) a.v[0][i] = (long long)host_vals[i];
  peer_counts_kernel<<<1, 64, 0, ctx->cnt_stream>>>(a, ctx->world, ctx->rank, n, ctx->d_cnt_epoch,
                                                     reinterpret_cast<long long*>(ctx->d_i64), ctx->d_err);
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  DDPPO_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->h_cnt, ctx->d_i64, n * sizeof(int64_t), cudaMemcpyDeviceToHost,
                                      ctx->cnt_stream));
  DDPPO_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->cnt_stream));
  int err = 0;
  DDPPO_CUDA_TRY(ctx, cudaMemcpy(&err, ctx->d_err, sizeof(int), cudaMemcpyDeviceToHost));
  if (err & ERR_BIT_COMM) {
    ctx->last_error = "counts exchange timed out (a rank did not reach ddppo_allreduce_counts)";
    return DDPPO_ERR_COMM;
  }
  for (int i = 0; i < n; ++i) host_vals[i] = ctx->h_cnt[i];
  return DDPPO_OK;
}

// ------------------------------------------------------------------ single-device emulation (tests)
extern "C" ddppo_status ddppo_debug_peer_a8(ddppo_ctx* ctx, int N, int mode, float* const* host_grads,
                                            float* const* host_params, float* const* host_m, float* const* host_v,
                                            int64_t P, const ddppo_adam_cfg* host_cfg, float* const* host_gsum,
                                            void* scratch, size_t scratch_bytes, size_t* host_need, void* stream) {
  if (!ctx) return DDPPO_ERR_CONFIG;
  DDPPO_REQUIRE(ctx, N >= 1 && N <= kMaxPeers && P >= 1 && host_cfg, "debug_peer_a8: 1 <= N <= 8, P >= 1");
  DDPPO_REQUIRE(ctx, mode == DDPPO_A8_ALLREAD || mode == DDPPO_A8_SHARDED, "debug_peer_a8: bad mode");
  const size_t area_b = align_up(sizeof(PeerArea), 256), pg_b = align_up((size_t)P * 4, 256);
  const size_t need = N * (area_b + pg_b) + 256;
  if (host_need) *host_need = need;
  if (!scratch) return DDPPO_OK;
  DDPPO_REQUIRE(ctx, scratch_bytes >= need && host_grads && host_params && host_m && host_v && host_gsum,
                "debug_peer_a8: bad buffers");
  cudaStream_t st = as_stream(stream);
  char* b = reinterpret_cast<char*>(scratch);
  DDPPO_CUDA_TRY(ctx, cudaMemsetAsync(b, 0, need, st));
  PeerArea* areas[kMaxPeers];
  float* pgs[kMaxPeers];
  for (int j = 0; j < N; ++j) areas[j] = reinterpret_cast<PeerArea*>(b + j * area_b);
  for (int j = 0; j < N; ++j) pgs[j] = reinterpret_cast<float*>(b + N * area_b + j * pg_b);
  unsigned int* epochs = reinterpret_cast<unsigned int*>(b + N * (area_b + pg_b));
  ProfScope ps(ctx, DDPPO_K_OTHER, st, 0);
  // the barrier of all N ranks at once (one warp each, one block: they run concurrently)
  PeerArgs a;
  memset(&a, 0, sizeof(a));
  for (int j = 0; j < N; ++j) a.area[j] = areas[j];
  peer_barrier_kernel<<<1, 32 * N, 0, st>>>(a, N, 0, epochs, ctx->d_err);
  ctx->count(1);
  ddppo_adam_cfg cfg = *host_cfg;
  // then every phase rank by rank: each phase's flags are all set before any rank waits on them
  if (mode == DDPPO_A8_ALLREAD) {
    for (int r = 0; r < N; ++r) {
      ddppo_status s = a8_rank(ctx, mode, N, r, host_grads, nullptr, areas, epochs + r, false, host_gsum[r],
                               host_params[r], host_m[r], host_v[r], P, cfg, nullptr, cfg.step, nullptr, st);
      if (s != DDPPO_OK) return s;
    }
  } else {
    const int64_t shard = (P + N - 1) / N;
    const int blocks = a8_blocks(ctx, shard);
    PeerArgs pa = a;
    for (int j = 0; j < N; ++j) {
      pa.grad[j] = host_grads[j];
      pa.pg[j] = pgs[j];
    }
    for (int r = 0; r < N; ++r)
      peer_rs_norm_kernel<<<blocks, kThreads, 0, st>>>(pa, N, r, P, 1.f / N, host_gsum[r], ctx->d_partials,
                                                       ctx->d_counters + CNT_NORM, epochs + r, ctx->d_err);
    for (int r = 0; r < N; ++r)
      peer_adam_shard_kernel<<<blocks, kThreads, 0, st>>>(pa, N, r, P, host_gsum[r], host_params[r], host_m[r],
                                                          host_v[r], pgs[r], 1.f / N, cfg.max_grad_norm, cfg.beta1,
                                                          cfg.beta2, cfg.lr, cfg.eps, nullptr, cfg.step, epochs + r,
                                                          ctx->d_counters + CNT_MISC, nullptr, ctx->d_err, nullptr, 0);
    for (int r = 0; r < N; ++r)
      peer_ag_kernel<<<a8_blocks(ctx, P - shard), kThreads, 0, st>>>(pa, N, r, P, host_params[r], epochs + r,
                                                                     ctx->d_err);
    ctx->count(3 * N);
  }
  DDPPO_CUDA_TRY(ctx, cudaGetLastError());
  return DDPPO_OK;
}

extern "C" ddppo_status ddppo_debug_peer_counts(ddppo_ctx* ctx, int N, const int64_t* host_vals, int n,
                                                int64_t* host_out, void* scratch, size_t scratch_bytes,
                                                size_t* host_need) {
  if (!ctx) return DDPPO_ERR_CONFIG;
  DDPPO_REQUIRE(ctx, N >= 1 && N <= kMaxPeers && n >= 0 && n <= kMaxCountVals, "debug_peer_counts: bad sizes");
  const size_t area_b = align_up(sizeof(PeerArea), 256);
  const size_t need = N * area_b + 256 + (size_t)N * kMaxCountVals * 8;
  if (host_need) *host_need = need;
  if (!scratch) return DDPPO_OK;
  DDPPO_REQUIRE(ctx, scratch_bytes >= need && host_vals && host_out, "debug_peer_counts: bad buffers");
  char* b = reinterpret_cast<char*>(scratch);
  DDPPO_CUDA_TRY(ctx, cudaMemset(b, 0, need));
  CountArgs a;
  memset(&a, 0, sizeof(a));
  for (int j = 0; j < N; ++j) a.area[j] = reinterpret_cast<PeerArea*>(b + j * area_b);
  for (int j = 0; j < N; ++j)
    for (int i = 0; i < n; ++i) a.v[j][i] = (long long)host_vals[j * n + i];
  unsigned int* epochs = reinterpret_cast<unsigned int*>(b + N * area_b);
  long long* out = reinterpret_cast<long long*>(b + N * area_b + 256);
  // the N ranks as N co-resident blocks (cooperative launch: they wait on one another)
  int world = N, rank_base = 0;
  int* err = ctx->d_err;
  void* args[] = {&a, &world, &rank_base, &n, &epochs, &out, &err};
  DDPPO_CUDA_TRY(ctx, cudaLaunchCooperativeKernel((const void*)peer_counts_kernel, dim3(N), dim3(64), args, 0, 0));
  ctx->count(1);
  DDPPO_CUDA_TRY(ctx, cudaDeviceSynchronize());
  std::vector<long long> h((size_t)N * kMaxCountVals);
  DDPPO_CUDA_TRY(ctx, cudaMemcpy(h.data(), out, h.size() * 8, cudaMemcpyDeviceToHost));
  for (int j = 0; j < N; ++j)
    for (int i = 0; i < n; ++i) host_out[j * n + i] = h[(size_t)j * kMaxCountVals + i];
  return DDPPO_OK;
}
