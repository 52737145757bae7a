/*
 * nj.h — C ABI of libnj: batched speculative-decoding verification on B200 (sm_100a)
 * and the Nightjar speculative-length bandit that drives it.
 *
 * Citation keys: P:n = PAPER.md line n (arXiv 2512.22420, LaTeX source);
 * S:n = SPEC.md line n; BJ = BASELINE.json north_star; "Leviathan" = the
 * speculative-sampling algorithm the paper cites at P:23 (leviathan2023fast).
 * DESIGN.md "Readings" R1..R14 resolve every place the paper is silent.
 *
 * ------------------------------------------------------------------------
 * Packed ragged batch (P:73 continuous batching; BJ "per-request variable-γ").
 *   B requests, request b carries gamma_b ∈ [0, gamma_max] drafts.
 *   N  = Σ_b (gamma_b + 1)  rows (verified positions),  G = Σ_b gamma_b drafts.
 *   row_off[b]   = Σ_{b'<b} (gamma_b' + 1)   (host exclusive scan, done inside)
 *   draft_off[b] = Σ_{b'<b} gamma_b'
 *   Row row_off[b]+j (j = 0..gamma_b) holds the target's final hidden state
 *   whose LM-head logits give p_j, the target distribution for position j;
 *   row j = gamma_b is the bonus position.  Draft i (i < gamma_b) of request b
 *   is draft_tokens[draft_off[b]+i] ~ q_i, with q_i = draft_probs row
 *   draft_off[b]+i.  Uniform slot row_off[b]+i (i < gamma_b) is the i-th
 *   acceptance test, slot row_off[b]+gamma_b is the final draw (R3).
 *
 * What nj_verify computes, per request b (Leviathan; BJ steps 1-3; R1):
 *   l_j(x)  = Σ_k W[x,k]·h_j[k]                (LM head, fp32 accumulate)
 *   p_j(x)  = exp(l_j(x) − lse_j), lse_j = log Σ_x exp l_j(x)  (online softmax)
 *   n_b     = first i < gamma_b with NOT(u_i·q_i(x_i) < p_i(x_i)), else gamma_b (R2)
 *   w(x)    = max(0, p_n(x) − q_n(x))  if n_b < gamma_b   (residual)
 *           = p_gamma(x)               otherwise          (bonus)
 *   W_b     = Σ_x w(x);  if W_b == 0 use w = p_n (R6)
 *   t_b     = min{x : Σ_{y≤x} w(y) > u_gamma·W_b}  ascending id (R5);
 *             on rounding overshoot the last x with w(x) > 0.
 *   accept_len[b] = n_b,  next_token[b] = t_b.
 * Accuracy contract (R12, R16):
 *   - Acceptance tests are certified (NJ_OPT_CERTIFY, default on): a test whose
 *     fp32 margin |u_i·q_i(x_i) − p_i(x_i)| is within the GEMM's measured error
 *     bound (2e-6..2e-5 relative, by path) sends the request to an fp64
 *     recomputation on the GPU (the plain definition), so every accept_len
 *     equals the fp64 definition.
 *   - Draws are NOT certified: at V = 152064 the CDF breakpoints are ~6.6e-6
 *     apart, so a band wide enough to cover the fp32 error would send most
 *     draws to fp64.  The LM-head GEMM restarts its TMEM accumulator often
 *     enough (and p = exp(l − lse) takes lse in fp64) that the residual /
 *     bonus CDF is accurate to well under 1e-6; next_token equals the fp64
 *     definition except when u_gamma lies within ~1e-6 of a boundary of the
 *     drawn token's CDF interval, where the neighbouring token may be returned
 *     (BJ's tie band; such requests are counted by the parity tests).
 *   - Zero residual mass (R6) is always redone in fp64 from p_n, certified or
 *     not (the fp64 fallback kernel runs on every call; it exits at once when
 *     nothing is queued).
 *
 * Conventions (all functions):
 *   - The caller owns every I/O buffer; nj_ctx owns its device workspace,
 *     sized at nj_create for max_batch and gamma_max.
 *   - Device functions are asynchronous on `stream` (a cudaStream_t passed as
 *     void*; NULL = legacy default stream); outputs are valid after the stream
 *     synchronises.  No device->host synchronisation happens inside nj_verify
 *     (gamma_per_req is a HOST array so every shape is known on the host), so
 *     it is CUDA-graph capturable.
 *   - One nj_ctx per stream; a ctx is not thread-safe.  The bandit is
 *     single-threaded.
 *   - Host-side shape and pointer checks return NJ_EINVAL / NJ_ESHAPE before
 *     any launch.  CUDA / NCCL failures return NJ_ECUDA / NJ_ENCCL; the
 *     message is available from nj_last_error.  Element values are not
 *     validated (u must be in [0,1), tokens in [0,V), q_i(x_i) > 0 expected).
 *   - bf16 tensors are passed as uint16_t bit patterns (IEEE bfloat16).
 *   - There is no CPU fallback: without a visible sm_100 device nj_create
 *     fails with NJ_ECUDA.
 */
#ifndef NJ_H
#define NJ_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    NJ_OK = 0,
    NJ_EINVAL = 1,        /* bad argument (NULL pointer, value out of range) */
    NJ_ESHAPE = 2,        /* inconsistent sizes / alignment */
    NJ_ECUDA = 3,         /* CUDA runtime / driver error */
    NJ_ENCCL = 4,         /* NCCL error */
    NJ_ENOMEM = 5,        /* allocation failed */
    NJ_EUNSUPPORTED = 6   /* configuration not supported by this build */
} nj_status;

typedef struct nj_ctx nj_ctx;
typedef struct nj_bandit nj_bandit;

/* ---------------------------------------------------------------- verify */

typedef struct {
    int32_t d;          /* hidden size; d % 8 == 0 (16-byte TMA row pitch)        */
    int32_t V;          /* GLOBAL vocabulary size, V >= 1                          */
    int32_t max_batch;  /* B_max, 1..1024                                   */
    int32_t gamma_max;  /* Γ_max, 0..15                                     */
    int32_t device;     /* CUDA device ordinal                                     */
    void*   nccl_comm;  /* NULL: unsharded.  Else an ncclComm_t (nj_nccl_comm_init): */
                        /* vocab-sharded LM head (BJ config 5, see below); this    */
                        /* rank owns W rows [v_begin,v_end) = nj_shard_range(...)  */
    int32_t v_begin;    /* shard start (global id); unsharded: 0                   */
    int32_t v_end;      /* shard end (exclusive);   unsharded: V                   */
} nj_config;

/* Optional per-call debug outputs (device buffers; any member may be NULL). */
typedef struct {
    float*   lse;      /* [N]  lse_j; NaN for rows the chosen path never evaluates  */
                       /*      (two-pass path: bonus row of a rejected request)     */
    float*   p_draft;  /* [G]  p_i(x_i), fp32                                       */
    double*  mass;     /* [B]  W_b of the distribution actually drawn from          */
    int32_t* flags;    /* [B]  NJ_FLAG_* bits                                       */
} nj_debug;

#define NJ_FLAG_FALLBACK  1  /* request recomputed by the fp64 certified fallback   */
#define NJ_FLAG_ZERO_MASS 2  /* residual mass 0 -> drew from p_n (R6)              */
#define NJ_FLAG_CLAMP     4  /* inverse-CDF overshoot -> clamped (R5)              */

/* Create a context on cfg->device.  Allocates the workspace for max_batch /
 * gamma_max.  Fails with NJ_ECUDA if the device is not sm_100. */
nj_status nj_create(const nj_config* cfg, nj_ctx** out);
void      nj_destroy(nj_ctx* ctx);
/* Last error message of ctx (static storage inside ctx; "" if none).  With
 * ctx == NULL returns the last nj_create failure message of this thread. */
const char* nj_last_error(const nj_ctx* ctx);

/* Verify one packed batch (see header comment).  Device pointers:
 *   hidden       [N, d]      bf16 row-major
 *   W_lm         [v_end - v_begin, d] bf16 row-major (nn.Linear weight layout)
 *   draft_tokens [G]         int32 global token ids
 *   draft_probs  [G, ldq]    fp32 full draft distributions q_i (ldq >= V);
 *                            sharded ranks read cols [v_begin,v_end)
 *   uniforms     [N]         fp32 in [0,1)
 *   accept_len   [B]         int32 out
 *   next_token   [B]         int32 out
 * Host pointer: gamma_per_req [B], each in [0, gamma_max].
 * B in [1, max_batch].  dbg may be NULL. */
nj_status nj_verify(nj_ctx* ctx, void* stream,
                    const uint16_t* hidden, const uint16_t* W_lm,
                    const int32_t* draft_tokens,
                    const float* draft_probs, int64_t ldq,
                    const int32_t* gamma_per_req, const float* uniforms,
                    int32_t B, int32_t* accept_len, int32_t* next_token,
                    const nj_debug* dbg);

/* End-to-end variant: every per-step input and output is a HOST pointer
 * (pinned memory recommended); W_lm stays a resident device pointer (model
 * weight).  Copies hidden / draft_tokens / uniforms into ctx staging buffers
 * on `stream`; draft_probs_h is read in place by the kernels when it is
 * pinned and mapped (UVA; NJ_OPT_Q_ZERO_COPY), else copied; runs nj_verify,
 * copies accept_len / next_token back and synchronises `stream` before
 * returning.  ldq as above (host row pitch). */
nj_status nj_verify_host(nj_ctx* ctx, void* stream,
                         const uint16_t* hidden_h, const uint16_t* W_lm,
                         const int32_t* draft_tokens_h,
                         const float* draft_probs_h, int64_t ldq,
                         const int32_t* gamma_per_req, const float* uniforms_h,
                         int32_t B, int32_t* accept_len_h, int32_t* next_token_h);

/* The draft rows g the last nj_verify_host call staged to the device before the
 * sampler (NJ_OPT_Q_STAGE_ROWS): *n_out = their count, the first max_rows of
 * them written to rows_out (may be NULL when max_rows = 0).  For byte
 * accounting of the host link (bench.py's e2e).  NJ_EINVAL on NULL ctx/n_out. */
nj_status nj_host_staged_rows(nj_ctx* ctx, int32_t* rows_out, int32_t max_rows, int32_t* n_out);

/* Execution path of nj_verify. */
typedef enum {
    NJ_PATH_AUTO = 0,    /* pick by size            */
    NJ_PATH_FUSED = 1,   /* one persistent kernel, logits resident in TMEM       */
    NJ_PATH_TWOPASS = 2, /* stats GEMM over drafts, accept, sample-row GEMM,     */
                         /* sampler kernels                                      */
    NJ_PATH_STAGED = 3   /* N <= 512: ONE GEMM pass over all N rows whose fp32   */
                         /* logits are staged in L2 (evict_last stores), accept, */
                         /* sampler kernels reading the B sample rows            */
} nj_path;

typedef enum {
    NJ_OPT_PATH = 1,          /* value: nj_path                                  */
    NJ_OPT_CERTIFY = 2,       /* 1 (default): acceptance tests within the error  */
                              /*    bound are recomputed in fp64; 0: off (zero-mass */
                              /*    draws R6 are redone in fp64 either way)          */
    NJ_OPT_FORCE_FALLBACK = 3,/* 1: recompute EVERY request in fp64 (tests)      */
    NJ_OPT_PROFILE = 4,       /* 1: bracket the dominant kernel of every nj_verify */
                              /*    with CUDA events (see nj_kernel_time)           */
    NJ_OPT_Q_ZERO_COPY = 5,   /* nj_verify_host: 1 (default) read a pinned, mapped */
                              /*    draft_probs_h in place over the host link (only */
                              /*    q_i(x_i) and rejected rows are touched); 0 copy */
                              /*    all G rows to the device first                  */
    NJ_OPT_Q_STAGE_ROWS = 6   /* nj_verify_host with in-place q, when the small-   */
                              /*    batch sampler runs (staged path, B <= 12): how  */
                              /*    many likely sample rows (first-rejection        */
                              /*    positions 0, 1, ... of every request) to copy   */
                              /*    to the device on a second stream while the GEMM */
                              /*    runs; -1 as many as the host link moves in the  */
                              /*    GEMM's time, 0 (default) none, else <= 256.     */
                              /*    Outputs are identical either way (same values). */
} nj_option;

nj_status nj_set_option(nj_ctx* ctx, nj_option opt, int64_t value);

/* Target temperature (verification variants; the paper
 * is silent on sampling settings, R1 reads it as T = 1): every
 * subsequent nj_verify of ctx uses p_j = softmax(l_j / T) as the target
 * distribution in place of softmax(l_j) -- acceptance u_i·q_i(x_i) < p_i(x_i),
 * residual max(0, p_n − q_n), bonus p_gamma -- and nj_propose draws from
 * softmax(l / T).  The kernels scale the accumulated fp32 logits by fp32(1/T)
 * before the softmax statistics (the fp64 fallback by 1/T in fp64); the
 * acceptance certificate widens by max(1, 1/T).  draft_probs are the draft's
 * own (already tempered) q.  temperature in (0, 1e6]; default 1.  T -> 0 is
 * nj_verify_greedy.  NJ_EINVAL otherwise.  Not applied by nj_lmhead_logits
 * (raw logits) or nj_sample_from_logits (given logits). */
nj_status nj_set_temperature(nj_ctx* ctx, double temperature);

/* Device time of the dominant kernel (fused verify kernel, or the stats GEMM
 * of the two-pass path) accumulated since the last reset, measured with CUDA
 * events recorded on the launch stream (NJ_OPT_PROFILE must be on).
 * Synchronises those events.  reset != 0 clears the accumulator. */
nj_status nj_kernel_time(nj_ctx* ctx, double* ms_total, int64_t* launches, int32_t reset);

/* Which path nj_verify would take for this batch and how many kernels it
 * launches (for bench accounting).  Host only. */
nj_status nj_plan(nj_ctx* ctx, const int32_t* gamma_per_req, int32_t B,
                  int32_t* path_out, int32_t* launches_out);

/* ---- test-only stage exports (used by tests/ for stage-isolated parity) ---- */

/* LM-head logits (BJ step 1) through the PRODUCTION GEMM kernel (k_lmhead, the
 * one the staged path, nj_propose and the sharded staged step launch; k_gemm_big,
 * the two-pass path's, when the context was created with NJ_LM=0):
 *   logits[r, x] = Σ_k W[x,k]·hidden[rows[r],k]   for x in [0, v_end-v_begin),
 * fp32, row-major with pitch ld_out (>= V_local).  rows: device int32
 * [n_rows], 1 <= n_rows <= min(max_batch·gamma_max, 1536).  ks: k-blocks (64
 * deep) per TMEM accumulator restart; 0 = the sample-row GEMM's
 * default (4, every group of k_lmhead included), 8 = the two-pass draft-row
 * GEMM's.  Test-only (element-wise
 * parity of the GEMM against the fp64 oracle). */
nj_status nj_lmhead_logits(nj_ctx* ctx, void* stream,
                           const uint16_t* hidden, const uint16_t* W_lm,
                           const int32_t* rows, int32_t n_rows,
                           float* logits, int64_t ld_out, int32_t ks);

/* Sampler stage (BJ step 3, residual / bonus draw) on given fp32 logits:
 *   logits   [B, ld_l] fp32 device, one row per request over the full vocab V
 *   residual [B] int32 device: 1 -> w = max(0, p − q_row), 0 -> w = p
 *   q        [B, ldq] fp32 device (read only for residual rows)
 *   u        [B] fp32 device final-draw uniforms
 *   out: next_token [B] int32, mass [B] double (W_b, may be NULL).
 * lse of each row is computed from the given logits.  Unsharded ctx only. */
nj_status nj_sample_from_logits(nj_ctx* ctx, void* stream,
                                const float* logits, int64_t ld_l,
                                const int32_t* residual,
                                const float* q, int64_t ldq,
                                const float* u, int32_t B,
                                int32_t* next_token, double* mass);

/* Draft-side proposal step (PAPER.md:23 — the draft
 * model proposes x_i ~ q_i, which the target then verifies): for B draft
 * positions with final hidden states h_b of the DRAFT model,
 *   l_b(x) = Σ_k W[x,k]·h_b[k]   (x < V; the draft LM head, e.g. d = 896,
 *                                 V = 151936 for a 0.5B-style draft)
 *   q_b(x) = exp(l_b(x) − lse_b),  lse_b = log Σ_x exp l_b(x)
 *   x_b    = min{x : Σ_{y≤x} q_b(y) > u_b·Σ_y q_b(y)}   (inverse CDF, R5)
 * Arguments (device pointers unless noted; the ctx is created with the draft's
 * d and V, unsharded):
 *   hidden  [B, d] bf16 row-major, 16-byte aligned
 *   W_lm    [V, d] bf16 row-major (the draft LM head)
 *   u       [B] fp32 in [0, 1): the draw's uniform per position
 *   tokens  [B] int32 out: x_b
 *   q_out   [B, ldq] fp32 out (ldq >= V): q_b, exactly the fp32 weights the
 *           draw summed (so q_b(x_b) > 0) — the draft_probs rows nj_verify takes
 * Same tcgen05 LM-head GEMM (accumulator restarted every 4 k-blocks, §6) and
 * sampler kernels as nj_verify's staged / two-pass paths.  The draw is not
 * certified (R16).  Errors: NJ_EINVAL (NULL), NJ_ESHAPE (B outside
 * [1, max_batch], ldq < V), NJ_EUNSUPPORTED (sharded ctx). */
nj_status nj_propose(nj_ctx* ctx, void* stream, const uint16_t* hidden, const uint16_t* W_lm,
                     const float* u, int32_t B, int32_t* tokens, float* q_out, int64_t ldq);

/* Greedy verification (the target distribution is
 * the argmax of its logits, temperature -> 0; the paper is silent on sampling
 * settings).  With p_i = one-hot at a_i = argmax_x l_i(x) (ties ->
 * lowest id), Leviathan's test u·q_i(x_i) < p_i(x_i) accepts
 * x_i iff x_i == a_i for any u in [0,1) and q_i(x_i) <= 1, and the residual
 * max(0, p_n − q_n) of the first rejected row is one-hot at a_n, so:
 *   accept_len[b] = first i < γ_b with draft x_i != a_i (else γ_b)
 *   next_token[b] = a_{n_b}  (the target's argmax at the first unmatched slot)
 * draft_probs and uniforms are not needed.  Layout of hidden / draft_tokens /
 * gamma_per_req as nj_verify.  Every row goes through the LM-head GEMM
 * (fp32 logits of <= 512 rows at a time) and a row argmax.  Errors as
 * nj_verify; NJ_EUNSUPPORTED on a vocab-sharded ctx. */
nj_status nj_verify_greedy(nj_ctx* ctx, void* stream, const uint16_t* hidden, const uint16_t* W_lm,
                           const int32_t* draft_tokens, const int32_t* gamma_per_req, int32_t B,
                           int32_t* accept_len, int32_t* next_token);

/* ------------------------------------------------------ vocab-sharded mode */
/* BJ config 5 / SURVEY §8a row a7, §8e: the LM head split along V over G
 * ranks (one process per GPU).  Rank r owns the contiguous, 128-row aligned
 * shard [v_begin, v_end) = nj_shard_range(V, G, r) (rank order = ascending
 * token id, which is the inverse-CDF order of R5).  Pass the communicator
 * (nj_nccl_comm_init) and the shard in nj_config; every rank then calls
 * nj_verify with the SAME hidden / draft / uniform / gamma inputs and its own
 * W shard (draft_probs rows are full-vocabulary rows; a rank reads only its
 * columns).  nj_verify runs in phases separated by three small exchanges on
 * `stream` (NCCL allgather of per-draft-row (lse_r, owned draft logit), of
 * per-request (lse, shard mass), and an allreduce-MAX of [token | flags]);
 * the certified fp64 fallback adds three more of the same kind; the sharded
 * driver always runs it (NJ_OPT_CERTIFY is ignored: the fallback also carries
 * the zero-mass draws R6, which no rank can redo alone).  Outputs
 * (accept_len, next_token, debug) are identical on every rank and equal the
 * unsharded definition (header comment) outside the 1e-6 tie band.
 * Error behaviour: NJ_ENCCL if libnccl.so.2 cannot be loaded or a collective
 * fails; NJ_ESHAPE if the shard is not nj_shard_range's.  The fused and
 * staged paths are unsharded-only (the sharded driver is the two-pass path). */

/* Shard of rank `rank` of `nranks`: [*v_begin, *v_end).  NJ_ESHAPE if V has
 * fewer 128-row tiles than ranks. */
nj_status nj_shard_range(int32_t V, int32_t nranks, int32_t rank, int32_t* v_begin, int32_t* v_end);

#define NJ_NCCL_ID_BYTES 128
/* NCCL bootstrap (libnccl.so.2 loaded at runtime): rank 0 creates the id,
 * the caller broadcasts the NJ_NCCL_ID_BYTES bytes (e.g. torch.distributed),
 * every rank calls nj_nccl_comm_init (collective; sets `device` current). */
nj_status nj_nccl_get_unique_id(void* id_out);
nj_status nj_nccl_comm_init(int32_t nranks, const void* id, int32_t rank, int32_t device, void** comm_out);
void      nj_nccl_comm_destroy(void* comm);

/* Single-process shard group: nshards contexts on cfg->device (cfg's shard
 * fields and nccl_comm are ignored; member r owns nj_shard_range(V, nshards,
 * r)) whose exchanges are device-to-device copies on `stream`.  Runs exactly
 * the per-rank kernels of the NCCL mode, so one GPU can check sharded parity.
 * nj_group_verify: W_shards is a HOST array of nshards device pointers (member
 * r's [v_end - v_begin, d] rows); other arguments as nj_verify.  dbg is filled
 * from member 0.  nj_group_member returns member r's context (options:
 * nj_set_option on every member), NULL if out of range. */
typedef struct nj_group nj_group;
nj_status nj_group_create(const nj_config* cfg, int32_t nshards, nj_group** out);
void      nj_group_destroy(nj_group* g);
nj_ctx*   nj_group_member(nj_group* g, int32_t r);
const char* nj_group_last_error(const nj_group* g);
nj_status nj_group_verify(nj_group* g, void* stream, const uint16_t* hidden, const uint16_t* const* W_shards,
                          const int32_t* draft_tokens, const float* draft_probs, int64_t ldq,
                          const int32_t* gamma_per_req, const float* uniforms, int32_t B,
                          int32_t* accept_len, int32_t* next_token, const nj_debug* dbg);

/* ---------------------------------------------------------------- bandit */
/* Nightjar arm selection (Algorithm 1) with the
 * c_prefill lookup (Table 1).  Host-only, no device code.
 * RNG: SplitMix64 over (seed, draw counter), draws consumed in the order
 * bin-type draw, then uniform-arm draw (R14). */

/* gamma_max >= 1, batch_max >= 1.  len_buckets[n_len],
 * batch_buckets[n_batch] strictly increasing; cost_ms[n_len*n_batch]
 * row-major by length bucket (NULL → c_prefill ≡ 0). */
nj_status nj_bandit_create(int32_t gamma_max, int32_t batch_max, uint64_t seed,
                           const int32_t* len_buckets, int32_t n_len,
                           const int32_t* batch_buckets, int32_t n_batch,
                           const double* cost_ms, nj_bandit** out);
void nj_bandit_destroy(nj_bandit* b);

/* γ_t for the current step (Algorithm 1).  batch_size in
 * 1..batch_max, l_max >= 0 the effective skip length.  Returns
 * γ >= 0, or -NJ_EINVAL on bad arguments. */
int32_t nj_select_gamma(nj_bandit* b, int32_t batch_size, int32_t l_max);

/* Reward feedback (Algorithm 1 line 190 + counters 191-200).  reward is the
 * realised goodput in tokens/s, >= 0. */
nj_status nj_observe(nj_bandit* b, int32_t batch_size, int32_t gamma,
                     double reward_tok_per_s);

/* Eq. 3 score of one candidate: 1/g̃ + 1(γ_prev=0 ∧ γ>0)·c_prefill/γ,
 * c_prefill in seconds.  Returns NaN for an unvisited arm. */
double nj_exploitation_score(const nj_bandit* b, int32_t batch_size,
                             int32_t gamma_prev, int32_t gamma, int32_t l_max);

/* c_prefill(L_max, B) in milliseconds: ceiling bucket with clamp; 0 if
 * L_max == 0. */
double nj_prefill_cost_ms(const nj_bandit* b, int32_t l_max, int32_t batch_size);

/* Inspection for tests: hierarchy counters of batch size B
 * (j_B, H_B, b_B, τ_B, bin type: -1 unset, 0 exploit, 1 explore) and
 * arm statistics (g̃_{B,γ}, visit count). */
nj_status nj_bandit_state(const nj_bandit* b, int32_t batch_size,
                          int32_t* j, int64_t* H, int64_t* bin, int64_t* tau,
                          int32_t* bin_type);
nj_status nj_bandit_arm(const nj_bandit* b, int32_t batch_size, int32_t gamma,
                        double* mean, int64_t* count);
int32_t   nj_bandit_last_gamma(const nj_bandit* b);

/* JSON snapshot.  Writes at most cap bytes (NUL-terminated),
 * *needed = full length + 1.  NJ_ESHAPE if cap is too small. */
nj_status nj_bandit_snapshot_json(const nj_bandit* b, char* buf, size_t cap,
                                  size_t* needed);

#ifdef __cplusplus
}
#endif
#endif /* NJ_H */
