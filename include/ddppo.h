/*
 * ddppo.h -- C ABI of the B200-native DD-PPO learner step (libddppo.so).
 *
 * Method: Decentralized Distributed PPO, arXiv 1911.00357 (/root/reference/PAPER.md,
 * cited as P:Lnn = line nn).  One process per GPU runs a worker; every worker owns its
 * rollout, computes grad J^PPO locally, the gradients are AllReduce-averaged and the same
 * Adam update is applied everywhere (Eq. 3/4); stragglers' collection is
 * preempted once p% of the workers are done.
 *
 * Conventions (every entry point):
 *  - Pointers are DEVICE pointers unless the parameter name starts with `host_`.
 *    The caller owns every buffer; the library never allocates or frees in the hot path.
 *    The library owns only the opaque ddppo_ctx (NCCL communicator, small scratch, a
 *    device error word).
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  Calls are
 *    stream-ordered and asynchronous except the ones marked "blocking".
 *  - Calls marked "collective" must be issued by every rank in the same order (a mismatch
 *    deadlocks).  With world == 1 they perform no communication.
 *  - One ctx must not be used from two streams concurrently (scratch is per ctx).
 *  - Per-step rollout arrays are env-major [E][ld] (ld = row stride in elements, ld >= T+1,
 *    ld % 4 == 0 enables 16-byte vector loads).  The value row holds T+1 slots: slot L_n is
 *    the bootstrap value V(s_{L_n}) of an env truncated at length L_n (P:L171 preemption).
 *  - Errors: every function returns ddppo_status; ddppo_last_error(ctx) gives the message.
 *    Non-finite losses/gradients set a device flag that ddppo_check() reports as
 *    DDPPO_ERR_NUMERICAL.
 */
#ifndef DDPPO_H_
#define DDPPO_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DDPPO_ABI_VERSION 1

typedef enum {
  DDPPO_OK = 0,
  DDPPO_ERR_CONFIG = 1,      /* shape / dim / alignment / enum problem                */
  DDPPO_ERR_NUMERICAL = 2,   /* non-finite loss or gradient detected on the device     */
  DDPPO_ERR_PROTOCOL = 3,    /* ranks disagree (layout hash, lengths)                  */
  DDPPO_ERR_COMM = 4,        /* NCCL error -- fatal to the job (no elasticity) */
  DDPPO_ERR_CUDA = 5,        /* CUDA runtime error                                     */
  DDPPO_ERR_UNSUPPORTED = 6  /* device is not sm_100 / feature not built               */
} ddppo_status;

typedef struct ddppo_ctx ddppo_ctx;

int ddppo_abi_version(void);
const char* ddppo_status_string(ddppo_status s);

/* ------------------------------------------------------------------ context
 * Rank 0 calls ddppo_get_unique_id, broadcasts the 128 bytes (e.g. over a torch process
 * group), then every rank calls ddppo_ctx_create (collective when world > 1). */
ddppo_status ddppo_get_unique_id(uint8_t host_id[128]);
ddppo_status ddppo_ctx_create(int rank, int world, const uint8_t* host_id /* NULL if world==1 */,
                              int device, ddppo_ctx** host_out);
ddppo_status ddppo_ctx_destroy(ddppo_ctx* ctx);
const char* ddppo_last_error(const ddppo_ctx* ctx);
/* blocking: synchronises `stream`, then reads and clears the device error word. */
ddppo_status ddppo_check(ddppo_ctx* ctx, void* stream);

/* ------------------------------------------------------------------ a2: GAE
 * P:L218 (sec.4): GAE with discount gamma (0.99) and GAE parameter tau (0.95); per env n,
 * for t = L_n-1 .. 0:  delta_t = r_t + gamma*V_{t+1}*(1-done_t) - V_t,
 *                      A_t = delta_t + gamma*tau*(1-done_t)*A_{t+1}, A_{L_n} = 0,
 *                      R_t = A_t + V_t;  A_t = R_t = 0 for L_n <= t < T.
 * rew, done, adv, ret: [E][ld]; val: [E][ld] with T+1 meaningful slots; len: [E] (1..T).
 * stats3 (nullable, device double[3]) receives the local {sum A, sum A^2, n} over valid t
 * (deterministic fixed-order reduction), the input of ddppo_adv_norm. */
ddppo_status ddppo_gae(ddppo_ctx* ctx, const float* rew, const float* val, const uint8_t* done,
                       const int32_t* len, int E, int T, int ld, float gamma, float tau,
                       float* adv, float* ret, double* stats3, void* stream);

/* ------------------------------------------------------------------ a3: advantage normalisation
 * Not in the paper (P:L219 says advantages are NOT normalised); required by the north_star.
 * collective: stats3 (device double[3]) is allreduced (sum) in place across ranks, then
 * mean_invstd (device float[2]) = { mu = S/n, 1/(sigma + eps) }, sigma^2 = (Q - n mu^2)/(n-1).
 * The normalisation itself is applied on the fly by ddppo_ppo_loss_grad. */
ddppo_status ddppo_adv_norm(ddppo_ctx* ctx, double* stats3, float eps, float* mean_invstd,
                            void* stream);

/* ------------------------------------------------------------------ model description
 * P:L582-593 (App. C) agent: goal [d, cos th, sin th] -> FC 32; previous-action embedding 32
 * (start token = num_actions); recurrent policy; FC -> softmax over actions + value.
 *   DDPPO_ARCH_TOY_MLP : goal -> Linear(3,64) -> tanh -> Linear(64, A+1)        (configs[0])
 *   DDPPO_ARCH_GPS_GRU : goal -> Linear(3,32); Embedding(A+1,32); x = [goal, act] ->
 *                        GRU(64, hidden=512) -> Linear(hidden, A+1)              (configs[1])
 *   DDPPO_ARCH_DEPTH_R18_LSTM : depth [1][64][64] -> half-width ResNet18 with GroupNorm(16)
 *                         -> 128x2x2 -> flatten (c,h,w) -> Linear(512,512)+ReLU;
 *                        x = [visual, Linear(3,32)(goal), Embedding(A+1,32)] -> LSTM(576,
 *                        hidden=512) -> Linear(hidden, A+1)                      (configs[2])
 *   DDPPO_ARCH_RGBD_R50_LSTM2 : RGB-D [4][256][256] (RGB in [0,255] normalised channel-wise,
 *                        P:L367) -> 2x2 avg-pool -> half-width ResNet50 (bottlenecks 3/4/6/3,
 *                        P:L212) -> 128x4x4 -> Linear(2048,512)+ReLU; [visual, goal, action] ->
 *                        2-layer LSTM-512 -> Linear(hidden, A+1)                 (configs[3])
 * Flat parameter layout: the tensors below in this order, row-major, each starting at an
 * offset rounded up to a multiple of 4 floats (PyTorch shapes/conventions):
 *   TOY: fc1.weight[64][3] fc1.bias[64] head.weight[A+1][64] head.bias[A+1]
 *   GPS: goal_fc.weight[32][3] goal_fc.bias[32] act_embed.weight[A+1][32]
 *        rnn.weight_ih[3H][64] rnn.weight_hh[3H][H] rnn.bias_ih[3H] rnn.bias_hh[3H]
 *        head.weight[A+1][H] head.bias[A+1]           (GRU gate rows r, z, n)
 *   DEPTH: the encoder (enc.stem.conv.weight[32][1][7][7], enc.stem.gn.{weight,bias}[32], then
 *        per residual block enc.layer{1..4}.{0,1}.{conv1,gn1,conv2,gn2[,down.conv,down.gn]},
 *        enc.compress.conv.weight[128][256][3][3], enc.compress.gn.*; widths 32/64/128/256,
 *        conv weights [Co][Ci][k][k]), visual_fc.weight[512][512] visual_fc.bias[512],
 *        goal_fc.*, act_embed.weight[A+1][32], rnn.weight_ih[4H][576] rnn.weight_hh[4H][H]
 *        rnn.bias_ih[4H] rnn.bias_hh[4H] head.*       (LSTM gate rows i, f, g, o)
 *   RGBD: enc.stem.conv.weight[32][4][7][7], enc.stem.gn.*, per bottleneck enc.layer{1..4}.{b}.
 *        {conv1,gn1,conv2,gn2,conv3,gn3[,down.conv,down.gn]} (1x1, 3x3 with the stride, 1x1),
 *        enc.compress.conv.weight[128][1024][3][3], enc.compress.gn.*, visual_fc.weight[512][2048]
 *        visual_fc.bias, goal_fc.*, act_embed.*, rnn.{weight_ih,weight_hh,bias_ih,bias_hh}_l{0,1}
 *        (weight_ih_l0 [4H][576], weight_ih_l1 [4H][H]), head.*
 * head rows 0..A-1 are the action logits, row A the value.  num_actions must be 4;
 * GPS requires hidden == 512; the visual agents take hidden 512 or 1024 (NEXT-3: "a 2-layer LSTM
 * with either a 512-dimensional or 1024-dimensional hidden dimension", P:L593 -- the best agent of
 * P:L334 is SE-ResNeXt101 + 1024-d LSTM).  hidden 1024 runs 32-CTA recurrences that exchange
 * through L2 (lstm_wide.cu); it needs 32 SMs free at once while a recurrence runs (a timeout of the
 * bounded exchange waits sets the device error word: ddppo_check returns DDPPO_ERR_COMM). */
typedef enum {
  DDPPO_ARCH_TOY_MLP = 0, DDPPO_ARCH_GPS_GRU = 1, DDPPO_ARCH_DEPTH_R18_LSTM = 2, DDPPO_ARCH_RGBD_R50_LSTM2 = 3,
  /* NEXT-3: the RGB-D agent with the half-width SE-ResNeXt50 encoder --
   * ResNet50/2's topology, each bottleneck's 3x3 conv grouped (cardinality 16, inner width 2 x planes)
   * and a squeeze-excitation module (reduction 16) before the residual addition (reading R9) */
  DDPPO_ARCH_RGBD_SERX50_LSTM2 = 4,
  DDPPO_ARCH_RGBD_SERX101_LSTM2 = 5   /* the same with SE-ResNeXt101's block counts [3, 4, 23, 3] */
} ddppo_arch;

typedef struct {
  int32_t arch;        /* ddppo_arch */
  int32_t hidden;      /* 64 (toy) / 512 (gps) / 512 or 1024 (visual agents) */
  int32_t num_actions; /* 4 */
  int32_t reserved[5];
} ddppo_model_desc;

typedef struct {
  char name[48];
  int64_t offset;   /* in floats */
  int64_t numel;
  int32_t ndim;
  int32_t fan_in;   /* used by the default initialiser U(-1/sqrt(fan_in), 1/sqrt(fan_in)) */
  int64_t shape[4];
} ddppo_tensor_info;

ddppo_status ddppo_model_param_count(const ddppo_model_desc* host_desc, int64_t* host_P);
ddppo_status ddppo_model_param_layout(const ddppo_model_desc* host_desc, ddppo_tensor_info* host_out,
                                      int cap, int* host_n);
/* bytes of device workspace ddppo_policy_fwd/bwd need for minibatches of <= max_B envs and
 * <= T steps (16-byte aligned base required). */
ddppo_status ddppo_workspace_size(const ddppo_model_desc* host_desc, int max_B, int T,
                                  size_t* host_bytes);

/* One PPO minibatch = B whole env trajectories (reading Z13: minibatches partition envs,
 * P:L219).  Samples are ordered m = b*T_run + t (b-th env of env_idx, time t). */
typedef struct {
  const float* goal;          /* [E][T][3]   (d, cos th, sin th)            */
  const int32_t* prev_action; /* [E][ld]     start token = num_actions         */
  const float* mask;          /* [E][ld]     1 - done_{t-1}; state is multiplied by it */
  const float* h0;            /* [E][layers*hidden] recurrent state before step 0 (no   */
                              /* grad; layer-major; layers = 2 for RGBD, else 1)           */
  const int32_t* len;         /* [E]         valid steps per env                        */
  const int32_t* env_idx;     /* [B]         env ids of this minibatch                  */
  int32_t E, T, ld, B;
  int32_t T_run;              /* steps to run: max len over the minibatch (host value)  */
  int32_t n_valid;            /* sum over the B envs of min(len, T_run) (host value)    */
  const uint16_t* obs;        /* depth frames as bf16 bits, values in [0, 1]:     */
                              /* DEPTH [E][T][1][64][64]; RGBD [E][T][1][256][256]; else NULL */
  const float* c0;            /* LSTM cell state before step 0, like h0 (DEPTH / RGBD)      */
  const uint8_t* obs_rgb;     /* RGBD: camera bytes [E][T][3][256][256] (normalised channel-   */
                              /* wise on the device); else NULL                        */
  /* transfer-learning mechanics (NEXT-4), both optional (0 / NULL):                 */
  float* dgoal;               /* DEPTH / RGBD backward output [B*T_run][3]: dL/d(goal input), the */
                              /* gradient a planner receives through a frozen "differentiable    */
                              /* neural controller"                                  */
  int32_t flags;              /* DDPPO_BATCH_FREEZE_ENCODER: the visual encoder (enc.* tensors) is */
                              /* frozen -- no encoder backward runs, its gradient entries are 0    */
  int32_t reserved_flags;
} ddppo_batch;
#define DDPPO_BATCH_FREEZE_ENCODER 1

/* a5: logits [B][T_run][A], values [B][T_run]; saves activations in ws for the backward. */
ddppo_status ddppo_policy_fwd(ddppo_ctx* ctx, const ddppo_model_desc* host_desc, const float* params,
                              const ddppo_batch* host_batch, float* logits, float* values,
                              void* ws, size_t ws_bytes, void* stream);
/* a7: grad [P] is OVERWRITTEN with dL/dparams given dL/dlogits, dL/dvalues (same layout as
 * the forward outputs); requires the ws of the matching ddppo_policy_fwd call. */
ddppo_status ddppo_policy_bwd(ddppo_ctx* ctx, const ddppo_model_desc* host_desc, const float* params,
                              const ddppo_batch* host_batch, const float* dlogits,
                              const float* dvalues, float* grad, void* ws, size_t ws_bytes,
                              void* stream);

/* ------------------------------------------------------------------ a6: fused PPO loss + gradient
 * P:L129-138 (Eq. 2) clipped surrogate on r_t = exp(lp - lp_old); value loss
 * 0.5*max((v-R)^2, (v_clip-R)^2) with v_clip = v_old + clip(v - v_old, +-vclip_eps) (or
 * 0.5*(v-R)^2 when use_value_clip == 0); entropy bonus.  Per-worker mean over the n_valid
 * valid samples (P:L171 equal weighting).  L = L_pi + c_v L_v - c_e H.
 * Tie conventions are torch's (min/max split 1/2-1/2, clamp passes on the closed interval).
 * stats (device float[8]) = {policy_loss, value_loss, entropy, clip_frac, approx_kl, total,
 * n_valid, 0}.  dlogits/dvalues have the logits/values layout; invalid samples get 0. */
typedef struct {
  const int32_t* action;    /* [E][ld] */
  const float* logp_old;    /* [E][ld] log pi_old(a_t|o_t) */
  const float* value_old;   /* [E][ld] V_hat_t of the rollout (the value row)   */
  const float* ret;         /* [E][ld] R_t (ddppo_gae) */
  const float* adv;         /* [E][ld] A_t (ddppo_gae, un-normalised) */
} ddppo_loss_inputs;

typedef struct {
  float clip_eps;        /* 0.2   */
  float vclip_eps;       /* 0.2   */
  float c_v;             /* 0.5   */
  float c_e;             /* 0.01  */
  int32_t use_value_clip;
  int32_t normalize_adv; /* if set, mean_invstd must be non-NULL */
} ddppo_loss_cfg;

ddppo_status ddppo_ppo_loss_grad(ddppo_ctx* ctx, const float* logits, const float* values,
                                 const ddppo_batch* host_batch, const ddppo_loss_inputs* host_in,
                                 const float* mean_invstd, const ddppo_loss_cfg* host_cfg,
                                 float* dlogits, float* dvalues, float* stats, void* stream);

/* ------------------------------------------------------------------ a8: AllReduce-mean + clip + Adam
 * P:L150-158 (Eq. 3), P:L219 (Adam, lr 2.5e-4).  collective.  grad [P] is summed over ranks in
 * place (NCCL, fp32), then one fused pass: g = sum/N; c = min(1, max_grad_norm/(||g||_2+1e-6))
 * (skipped if max_grad_norm <= 0); Adam (PyTorch form, bias-corrected, `step` = 1-based index
 * of this update) on every entry whose freeze_mask byte is 0 (freeze_mask nullable).
 * grad_norm (nullable, device float[1]) receives ||g|| before clipping. */
typedef struct {
  float lr, beta1, beta2, eps, max_grad_norm;
  int32_t step;
} ddppo_adam_cfg;

ddppo_status ddppo_grad_allreduce_step(ddppo_ctx* ctx, float* grad, float* params, float* m, float* v,
                                       const uint8_t* freeze_mask, int64_t P,
                                       const ddppo_adam_cfg* host_cfg, float* grad_norm, void* stream);

/* ------------------------------------------------------------------ a9: preemption protocol
 * stragglers stop collecting once p% of the workers have finished, but never before
 * one-fourth of the maximum steps.  Readings: K = ceil(p*N/100) (other_workers: ceil(p*(N-1)/100),
 * clamped >= 1); min_steps = ceil(T/4) unless overridden (> 0).  Decision after completing a
 * step: stop iff my_steps >= T, or (my_steps >= min_steps and finished_count >= K). */
typedef struct {
  int32_t p_percent;     /* 1..100 (60 works well) */
  int32_t T;             /* rollout capacity */
  int32_t min_steps;     /* 0 => ceil(T/4) */
  int32_t other_workers; /* alternate reading of "p% of the other workers" */
} ddppo_preempt_cfg;

/* pure host arithmetic (no ctx, no GPU) */
ddppo_status ddppo_preempt_threshold(const ddppo_preempt_cfg* host_cfg, int world, int* host_K,
                                     int* host_min_steps);
ddppo_status ddppo_preempt_decide(const ddppo_preempt_cfg* host_cfg, int world, int my_steps,
                                  int finished_count, int* host_should_stop);
/* collective, blocking: allreduce(sum) of {finished (0/1: this rank completed T steps),
 * active (0/1: still collecting)} across ranks (the paper's TCPStore counter, P:L176/P:L637,
 * realised as an int32 allreduce per poll tick), then the decision above for this rank. */
ddppo_status ddppo_preempt_poll(ddppo_ctx* ctx, int my_steps, int finished, int active,
                                const ddppo_preempt_cfg* host_cfg, int* host_should_stop,
                                int* host_finished_count, int* host_active_count);

/* a10: collective, blocking int64 sum of n host values (step accounting). */
ddppo_status ddppo_allreduce_counts(ddppo_ctx* ctx, int64_t* host_vals, int n);
/* a10 input of one rank: the experience steps its rollout holds, sum_e min(len[e], T) (the steps a
 * learner step trains on; a preempted env contributes its L_w).  host_len: [E] int32 host
 * array; ERR_CONFIG on E < 1, T < 1 or a negative length. */
ddppo_status ddppo_rollout_steps(const int32_t* host_len, int E, int T, int64_t* host_steps);

/* ------------------------------------------------------------------ the whole learner step
 * a2..a8 for one rollout on this rank: GAE -> (adv norm) -> epochs x minibatches of
 * {policy_fwd, ppo_loss_grad, policy_bwd, grad_allreduce_step}.  collective. */
typedef struct {
  const float* rew; const float* val; const uint8_t* done; const int32_t* len;
  const float* goal; const int32_t* prev_action; const float* mask; const float* h0;
  const int32_t* action; const float* logp_old;
  const int32_t* perms;       /* [epochs][E] device: env permutation per epoch (a4 input) */
  const int32_t* host_len;    /* [E] host copy of len */
  const int32_t* host_perms;  /* [epochs][E] host copy of perms */
  int32_t E, T, ld;
  const uint16_t* obs;        /* as ddppo_batch::obs (DEPTH / RGBD, else NULL) */
  const float* c0;            /* as ddppo_batch::c0  (DEPTH / RGBD, else NULL) */
  const uint8_t* obs_rgb;     /* as ddppo_batch::obs_rgb (RGBD, else NULL) */
} ddppo_rollout;

typedef struct {
  float gamma, tau, adv_eps;
  int32_t normalize_adv;
  int32_t epochs, minibatches;
  ddppo_loss_cfg loss;
  ddppo_adam_cfg adam;        /* adam.step = number of updates already taken */
  /* NEXT-4: freeze_mask (device uint8 [P], nullable, 4-byte aligned): entries != 0 keep
   * params / m / v bit-identical; freeze_encoder != 0: the visual encoder's backward is
   * skipped, its gradient entries are 0 (excluded from the clip norm) and its parameters frozen. */
  const uint8_t* freeze_mask;
  int32_t freeze_encoder;
  int32_t reserved;
} ddppo_learner_cfg;

ddppo_status ddppo_learner_workspace_size(const ddppo_model_desc* host_desc, int E, int T, int ld,
                                          int minibatches, int epochs, size_t* host_bytes);
/* collective: make this workspace (allocated for the learner_step configuration every rank uses)
 * visible to all ranks over NVLink (CUDA IPC handles exchanged with an NCCL all-gather).  After
 * it, ddppo_learner_step on this ws performs a8 over peer memory instead of NCCL: every rank sums
 * all ranks' gradients in rank order 0..N-1 (bit-identical on every rank), computes the clip norm
 * in the same pass and applies Adam; a flag barrier per minibatch (release/acquire at system
 * scope, bounded wait -> ddppo_check reports a communication error).  The workspace must stay
 * allocated while the context lives.  World size 1: no-op.  At most one workspace per context. */
ddppo_status ddppo_learner_register(ddppo_ctx* ctx, void* ws, size_t ws_bytes);

/* ------------------------------------------------------------------ collection side (NEXT-1)
 * Batched single-step policy inference ("collect experience with pi_theta"; P:L461 batching
 * across a GPU's environments): step t of E envs at once, the recurrent state carried in
 * h_in/c_in -> h_out/c_out, an action sampled per env.
 * Inputs use the rollout layout with T = 1 slot (or a rollout's column t through pointer offsets):
 * goal [E][T][3], prev_action / mask [E][ld] (column t), obs (bf16 depth) [E][T][1][H][W], obs_rgb
 * (RGBD) [E][T][3][H][W]; the step read is t.  h_in / c_in [E][layers*hidden] (c: visual agents).
 * Sampling (both the kernels and the oracle implement it): u_e = (splitmix64(seed *
 * 0x9E3779B97F4A7C15 + counter * 0xD1B54A32D192ED03 + e) >> 40) * 2^-24; with m = max_a z_a,
 * w_a = expf(z_a - m), S = ((w_0 + w_1) + w_2) + w_3 (fp32, this order), the action is the first a
 * whose running sum w_0 + .. + w_a exceeds u_e * S (else A-1); logp = (z_a - m) - logf(S).
 * greedy != 0: the first argmax instead.  Outputs (device, [E]): actions, logp, values; logits
 * [E][A] nullable.  The workspace (ddppo_act_workspace_size) holds the forward's activations. */
typedef struct {
  const float* goal; const int32_t* prev_action; const float* mask;
  const uint16_t* obs; const uint8_t* obs_rgb;
  int32_t E, T, ld, t;
  const float* h_in; const float* c_in;
  float* h_out; float* c_out;
  uint64_t seed; int64_t counter;
  int32_t greedy; int32_t reserved;
} ddppo_act_batch;
ddppo_status ddppo_act_workspace_size(const ddppo_model_desc* host_desc, int E, size_t* host_bytes);
ddppo_status ddppo_policy_act(ddppo_ctx* ctx, const ddppo_model_desc* host_desc, const float* params,
                              const ddppo_act_batch* host_batch, int32_t* actions, float* logp, float* values,
                              float* logits, void* ws, size_t ws_bytes, void* stream);

/* Critic re-initialisation ("critic layers are reinitialized"): the value head
 * (row num_actions of head.weight and head.bias[num_actions]) is resampled from the default
 * initialiser U(-1/sqrt(fan_in), 1/sqrt(fan_in)) with a counter-based generator (element i of the
 * head row / bias: u = splitmix64(seed * 0x9E3779B97F4A7C15 + i) >> 40, value = (u * 2^-23 - 1) *
 * (1 / sqrtf(fan_in)) in fp32; the bias uses i = fan_in); m / v of those entries are zeroed (a fresh
 * optimiser state); every other entry is untouched.  params / m / v device [P]; stream-ordered. */
ddppo_status ddppo_reinit_critic(ddppo_ctx* ctx, const ddppo_model_desc* host_desc, float* params, float* m,
                                 float* v, uint64_t seed, void* stream);

/* Layout agreement at rendezvous ("layout is identical across all workers ... checked at
 * rendezvous by exchanging a layout hash"; S:L329 length mismatch -> fatal protocol error).
 * ddppo_layout_hash (pure host): 64-bit FNV-1a over the flat parameter layout of desc (every tensor's
 * name, offset, numel, shape, in order) and the learner geometry (E, T, ld, minibatches, epochs).
 * ddppo_layout_check (collective): all-gathers every rank's hash over NCCL; DDPPO_ERR_PROTOCOL (on
 * every rank, ddppo_last_error lists the disagreeing ranks) if any differs.  World size 1: OK. */
ddppo_status ddppo_layout_hash(const ddppo_model_desc* host_desc, int E, int T, int ld, int minibatches,
                               int epochs, uint64_t* host_hash);
ddppo_status ddppo_layout_check(ddppo_ctx* ctx, const ddppo_model_desc* host_desc, int E, int T, int ld,
                                int minibatches, int epochs);

/* a8 over peer memory (after ddppo_learner_register), Eq. 3:
 *   DDPPO_A8_SHARDED: reduce-scatter -> clip + Adam on this rank's 1/N shard -> all-gather
 *     (NEXT-2; rank r owns float4 units [Q*r/N, Q*(r+1)/N) of the flat vector, Q = P/4, the last
 *     rank also the P%4 tail).  NVLink volume 2(N-1)/N*4P per rank.  Parameters stay bit-identical
 *     on all ranks; Adam's m / v are only maintained on the owned shard (ZeRO-1).
 *   DDPPO_A8_ALLREAD: every rank reads all N gradients and runs the full Adam ((N-1)*4P bytes).
 * Both sum the N gradients in rank order 0..N-1 (identical per-element sums).  Any wait on a peer is
 * bounded (30 s of %globaltimer): on timeout the exchange leaves params / m / v untouched and
 * ddppo_check returns DDPPO_ERR_COMM (fatal).  Host-side setting, read when a learner step
 * is built (graphs are keyed by it). */
/*   DDPPO_A8_AUTO (default): the form with the lower modelled cost -- all-read moves (N-1)/N*4P more
 *     bytes per rank but has one cross-rank synchronisation instead of three; sharded is chosen when
 *     (N-1)(1-2/N)*4P / 770 GB/s + (1-1/N)*28P / 6.5 TB/s exceeds the two extra synchronisations
 *     (~20 us, measured): Depth at N >= 4, GPS at N = 8, never at N = 2. */
typedef enum { DDPPO_A8_SHARDED = 0, DDPPO_A8_ALLREAD = 1, DDPPO_A8_AUTO = 2 } ddppo_a8_mode;
ddppo_status ddppo_set_a8_mode(ddppo_ctx* ctx, int mode);

/* Engine of the visual encoders' implicit-GEMM convolutions (same arithmetic, host-side setting):
 *   DDPPO_CONV_TMA (default): TMA im2col / tiled boxes feeding a warp-specialised persistent tcgen05
 *     kernel (FPROP, stride-1 DGRAD, WGRAD of every convolution with a multiple of 32 input channels);
 *   DDPPO_CONV_CPASYNC: the cp.async-staged tcgen05 kernel (round 1; also the fallback for the
 *     stride-2 input gradients and the 8-channel RGB-D stem). */
typedef enum { DDPPO_CONV_CPASYNC = 0, DDPPO_CONV_TMA = 1 } ddppo_conv_engine;
ddppo_status ddppo_set_conv_engine(ddppo_ctx* ctx, int engine);
/* Operand precision of the visual encoders' forward convolutions on the TMA engine: 2 (default) =
 * bf16 hi / lo planes (x = hi + lo, hi*hi + hi*lo + lo*hi: ~16-bit mantissas -- the ReLU / max-pool
 * decisions the backward inherits are then within ~2^-16 of the fp32 ones); 1 = plain bf16. */
ddppo_status ddppo_set_fwd_planes(ddppo_ctx* ctx, int planes);

/* CUDA graphs for ddppo_learner_step (default on): the step is captured once per (configuration,
 * buffer addresses, minibatch shapes) -- after one eager run of a new configuration -- and
 * replayed; Adam's update count and the peer-barrier epoch are kept on the device so nothing
 * host-side is baked into the graph.  While per-family profiling is enabled the step runs eagerly. */
ddppo_status ddppo_set_graphs(ddppo_ctx* ctx, int enable);

/* params/m/v [P] updated in place; adv/ret [E][ld] outputs; stats_out (device float
 * [epochs*minibatches][8]) receives each minibatch's loss stats; host_cfg->adam.step is read,
 * *host_step_out receives the new update count. */
ddppo_status ddppo_learner_step(ddppo_ctx* ctx, const ddppo_model_desc* host_desc,
                                const ddppo_rollout* host_ro, const ddppo_learner_cfg* host_cfg,
                                float* params, float* m, float* v, float* adv, float* ret,
                                float* stats_out, void* ws, size_t ws_bytes,
                                int32_t* host_step_out, void* stream);

/* ------------------------------------------------------------------ measurement
 * Per-kernel-family device time (CUDA events recorded on the launching stream around every
 * launch of the family while profiling is enabled) and launch counts (always counted).
 * ddppo_profile_read is blocking (synchronises the recorded events); reset != 0 clears. */
typedef enum {
  DDPPO_K_GAE = 0, DDPPO_K_ADV_NORM, DDPPO_K_NET_FWD, DDPPO_K_HEAD, DDPPO_K_LOSS, DDPPO_K_NET_BWD,
  DDPPO_K_WGRAD, DDPPO_K_ALLREDUCE, DDPPO_K_ADAM, DDPPO_K_OTHER,
  /* sub-families, nested inside the ones above (their time is also counted there): the TMA
   * implicit-GEMM convolution kernel, the recurrence kernels (GRU / LSTM, fwd + BPTT), GroupNorm */
  DDPPO_K_CONV, DDPPO_K_RNN, DDPPO_K_GN, DDPPO_K_COUNT
} ddppo_kernel_family;

ddppo_status ddppo_profile_enable(ddppo_ctx* ctx, int enable);
ddppo_status ddppo_profile_read(ddppo_ctx* ctx, double* host_ms /* [DDPPO_K_COUNT] */,
                                int64_t* host_launches /* [DDPPO_K_COUNT] */, int reset);
/* Algorithmic work issued per family since the last reset (host-side accounting at launch: useful
 * dense-contraction FLOPs, 2*M*N*K with the bf16x3 forward counted once; counted while profiling
 * is enabled, i.e. for eager launches).  reset != 0 clears. */
ddppo_status ddppo_profile_flops(ddppo_ctx* ctx, double* host_flops /* [DDPPO_K_COUNT] */, int reset);
/* Shared-memory traffic of the TMA conv kernels per family since the last reset (same accounting
 * mode): per k-iteration the TMA's operand writes (A and B, every plane) plus the tcgen05.mma operand
 * reads (bf16x3: three products; SM100 MMA reads A and B from shared memory) -- the conv kernels'
 * binding resource for N <= 64.  reset != 0 clears. */
ddppo_status ddppo_profile_smem_bytes(ddppo_ctx* ctx, double* host_bytes /* [DDPPO_K_COUNT] */, int reset);

/* Diagnostic entry to the tcgen05 GEMM used inside the backward (stream-ordered):
 * C[m][n] = sum_k A[m*sam + k*sak] * B[n*sbn + k*sbk]; operands rounded to bf16, fp32 accumulate
 * in TMEM.  C is row-major with leading dimension ldc.  splits > 1 splits K over CTAs (needs
 * `partial`, splits*M*N floats; partials summed in split order).  prec = 1: bf16 operands;
 * prec = 3: each operand split x = hi + lo (both bf16) and C = hi*hi + hi*lo + lo*hi (~fp32
 * accuracy, used by the Depth encoder's forward).  Used by the tests. */
ddppo_status ddppo_debug_gemm_bf16(ddppo_ctx* ctx, const float* A, int64_t sam, int64_t sak,
                                   const float* B, int64_t sbn, int64_t sbk, float* C, int64_t ldc,
                                   int M, int N, int K, int splits, float* partial, int prec, void* stream);

/* Diagnostic entries to the Depth encoder's layers (stream-ordered; used by the tests).  All
 * activations NHWC fp32; conv weights PyTorch [Co][Ci][k][k].
 * conv2d: y[F][Ho][Wo][Co] = conv(x[F][H][W][Ci], w) (stride s, zero padding p; bf16 hi/lo
 *   operand planes) if y != NULL; if dy != NULL: dw = weight gradient, dx = input gradient (dx
 *   nullable), bf16 operands.  Ci == 1 (the stem: warp MMAs on bf16 hi/lo planes, fp32 SIMT off
 *   that grid; no dx) or Ci, Co multiples of 8.
 *   scratch == NULL: only *host_need (bytes) is written. */
ddppo_status ddppo_debug_conv2d(ddppo_ctx* ctx, const float* x, const float* w, int F, int H, int W,
                                int Ci, int Co, int k, int s, int p, float* y, const float* dy,
                                float* dx, float* dw, void* scratch, size_t scratch_bytes,
                                size_t* host_need, void* stream);
/* GroupNorm(16 groups, eps 1e-5) over y[F][HW][C]: z = (relu)(gamma*yhat + beta (+ residual)),
 * stats[F][16][2] = (mean, rstd); if dz != NULL: dy (rounded to bf16, the form the gradient GEMMs
 * consume), dgamma, dbeta (scratch: 4*F*HW*C + 64*F + 1024 floats). */
ddppo_status ddppo_debug_groupnorm(ddppo_ctx* ctx, const float* y, const float* gamma, const float* beta,
                                   const float* residual, int F, int HW, int C, int relu, float* z,
                                   float* stats, const float* dz, float* dy, float* dgamma,
                                   float* dbeta, float* scratch, void* stream);
/* The visual agents' (DEPTH / RGBD) forward discrete decisions, read from the workspace of the last
 * ddppo_policy_fwd on the same batch (bytes, NHWC): stem ReLU mask, max-pool argmax (window index
 * 0..8), then per residual block in order the ReLU masks of its branch convolutions (conv1[, conv2])
 * followed by the block-output ReLU mask, then the compression ReLU mask and the visual-FC ReLU
 * mask [F][512]; F = B*T_run.  out == NULL: only *host_n.  Lets a parity test hand the oracle's
 * backward the same decisions where a pre-activation sits within rounding of 0. */
ddppo_status ddppo_debug_depth_decisions(ddppo_ctx* ctx, const ddppo_model_desc* host_desc,
                                         const ddppo_batch* host_batch, void* ws, uint8_t* out, int64_t cap,
                                         int64_t* host_n, void* stream);
/* Single-device emulation of the peer-memory a8 over N in 1..8 ranks (tests): host_grads[r],
 * host_params[r], host_m[r], host_v[r], host_gsum[r] are device buffers of P floats for emulated rank
 * r; the exchange runs exactly the kernels of the multi-GPU path (barrier as N warps of one block,
 * then each phase rank by rank), with the flag areas and staged shards in `scratch`.
 * host_cfg->step = 1-based Adam step.  Outputs: params/m/v (m/v: owned shard only in SHARDED mode)
 * and gsum (rank-ordered gradient sum; SHARDED: the owned shard only).  scratch == NULL: *host_need. */
ddppo_status ddppo_debug_peer_a8(ddppo_ctx* ctx, int N, int mode, float* const* host_grads,
                                 float* const* host_params, float* const* host_m, float* const* host_v,
                                 int64_t P, const ddppo_adam_cfg* host_cfg, float* const* host_gsum,
                                 void* scratch, size_t scratch_bytes, size_t* host_need, void* stream);
/* Single-device emulation of the a10 peer counts exchange (the kernel of ddppo_allreduce_counts
 * once a learner is registered) over N ranks as N co-resident blocks (cooperative launch):
 * host_out[r*n + i] = sum over ranks (rank order) of host_vals[j*n + i].  Blocking. */
ddppo_status ddppo_debug_peer_counts(ddppo_ctx* ctx, int N, const int64_t* host_vals, int n,
                                     int64_t* host_out, void* scratch, size_t scratch_bytes,
                                     size_t* host_need);
/* 3x3 / stride 2 / pad 1 max pool (first maximum in window order; arg = window index 0..8).
   x [F][H][W][C] channels-last, C % 4 == 0 (else DDPPO_ERR_CONFIG); y / arg [F][Ho][Wo][C]. */
ddppo_status ddppo_debug_maxpool(ddppo_ctx* ctx, const float* x, int F, int H, int W, int C, float* y,
                                 uint8_t* arg, const float* dy, float* dx, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DDPPO_H_ */
