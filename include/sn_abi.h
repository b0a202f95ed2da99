/*
 * sn_abi.h — C ABI of libsn100.so, the B200 (sm_100a) kernels behind the
 * Super Apriel per-layer mixer step (arXiv 2604.19877).
 *
 * Drop-in position: the reference's placement vocabulary
 * (R/pkg/src/placeopt/placements.py:19-105 — MixerCatalog / Placement with
 * codes A=FA, S=SWA, K=KDA, G=GDN) selects, per layer, which of these mixer
 * entry points the layer loop launches.  The reference ships no mixer code
 * (R/SPEC.md:8 scopes it out); each entry point below replaces the mixer the
 * paper describes (R/§6 R/PAPER.md:827-865) and that its
 * serving stack runs through vLLM/FLA/FlashInfer.
 *
 * Conventions (all functions):
 *   - plain device pointers + sizes; no allocation inside any call; every
 *     launch is enqueued on `stream` (a cudaStream_t passed as void*), so all
 *     of them are CUDA-graph capturable.  Lengths/positions are read from
 *     device arrays, never from the host.
 *   - `dtype` is the activation/weight I/O type (SN_BF16 or SN_F32).  Recurrent
 *     states, softmax statistics and the residual stream are always fp32.
 *   - return SN_OK or an error code; the message is in sn_last_error()
 *     (thread-local).  Nothing aborts or throws across the ABI.
 *   - stateless and reentrant; concurrency comes from streams / processes.
 *
 * Layouts (HBM):
 *   paged KV (FA):      k_cache/v_cache [num_pages][Hkv][page_size][D]   ("HND" pages:
 *                       one head's page is one contiguous page_size*D run, fed by
 *                       cp.async.bulk); block_table [B][max_blocks] int32.
 *   ring KV (SWA):      same page pool; a sequence owns window/page_size pages and
 *                       position p lives at ring slot p % window.
 *   recurrent state:    float [slots][Hv][D(v)][D(k)]  (each value column's key
 *                       vector contiguous: one coalesced 512 B row per column).
 *   conv ring:          T [slots][C][W]; the input at position p lives at slot p % W.
 */
#ifndef SN_ABI_H_
#define SN_ABI_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SN_ABI_VERSION 2

typedef enum { SN_OK = 0, SN_EINVAL = 1, SN_ECUDA = 2, SN_EUNSUPPORTED = 3 } sn_status;
typedef enum { SN_F32 = 0, SN_BF16 = 1 } sn_dtype;

/* Thread-local text of the last error (empty string if none). */
const char* sn_last_error(void);
int sn_abi_version(void);

/* ---------------------------------------------------------------- trunk
 * Shared trunk of every layer (R/PAPER.md:175-182, 855-856): embedding,
 * pre-norms, SiLU-gated FFN, final norm, greedy sampler.                  */

/* residual[r,:] = table[tokens[r],:] (fp32).  If seq_lens/positions are
 * non-NULL this is also the decode-step prologue: positions[b] = seq_lens[b];
 * seq_lens[b] += 1 for b < rows (so every later kernel of the step sees the
 * new token's position and the post-append length).  A negative token marks an
 * idle slot (continuous batching): positions[b] = -1, seq_lens[b] unchanged, a
 * zero residual row, and the KV append skips it.  rope_cs (optional, fp32
 * [rows][half][2]): the step's rotary (cos, sin) per pair at each row's position
 * (inv_freq [half]), read by the attention in-projection epilogue instead of
 * evaluating sincosf per head.                                              */
sn_status sn_embed(const int32_t* tokens, const void* table, float* residual,
                   int32_t* seq_lens, int32_t* positions, const float* inv_freq,
                   void* rope_cs, int half, int rows, int dim, int dtype, void* stream);

/* residual += delta (if non-NULL) + sum_{s<nsplit} partials[s] (the fp32 K-split slabs
 * [nsplit][rows][dim] of SN_GEMM_PARTIAL, added in slab order: deterministic);
 * out = rmsnorm(residual) * weight.                                          */
sn_status sn_add_rmsnorm(const void* delta, const float* partials, int nsplit,
                         float* residual, const void* weight, void* out, int rows,
                         int dim, float eps, int dtype, void* stream);

/* out[r, i] = silu(g) * u for the interleaved gate/up layout of GEMM mode
 * SN_GEMM_SWIGLU_IL (row of ceil(ffn/h) blocks of [h gate | h up] columns, row
 * stride ld); used on the prefill gate/up GEMM output.                       */
sn_status sn_swiglu_il(const void* gate_up, int ld, void* out, int rows, int ffn,
                       int h, int dtype, void* stream);

/* out_tokens[r] = argmax_v logits[r,v] (lowest index on ties); -1 for idle slots
 * (positions[r] < 0, positions may be NULL) so a token-feedback graph keeps them idle. */
sn_status sn_argmax(const void* logits, int rows, int vocab, int32_t* out_tokens,
                    const int32_t* positions, int dtype, void* stream);

/* ---------------------------------------------------------------- FA / SWA
 * R/PAPER.md:1540-1563 (GQA + RoPE; SWA = same weights shape, window mask
 * j in (t-w, t]).  Replaces the paged-KV attention backend the paper serves
 * with (FlashInfer in vLLM, R/PAPER.md:1793).                               */

/* Rotary embedding (rotate-half) on q and k of a fused qkv row
 * [q Hq*D | k Hkv*D | v Hkv*D] (pair_il != 0: the q / k columns of each head in the
 * rotary-pair interleaved order of sn_gemm_decode_attn_in), then append k,v at the row's
 * position into
 * the page pool (window==0: slot = pos; window>0: ring slot = pos % window,
 * rows older than seq_lens[seq]-window are not written).  q_out [rows][Hq][D];
 * k_out/v_out [rows][Hkv][D] optional (prefill attention input).                */
sn_status sn_rope_kv_append(const void* qkv, const int32_t* row_seq,
                            const int32_t* row_pos, const int32_t* seq_lens,
                            const float* inv_freq, void* q_out, void* k_out,
                            void* v_out, void* k_cache, void* v_cache,
                            const int32_t* block_table, int rows, int Hq, int Hkv,
                            int D, int page_size, int max_blocks, int window, int pair_il,
                            int dtype, void* stream);

/* Split-KV flash-decode over the page pool: one CTA per (split, kv head,
 * sequence); each split streams split_pages pages of one head through a
 * cp.async.bulk/mbarrier ring in shared memory; the GQA group of Hq/Hkv query
 * heads shares every K/V byte read.  The last CTA of a (seq, head) merges
 * the split partials (no second launch).  window==0 → FA over seq_lens[b]
 * keys; window>0 → SWA over min(seq_lens[b], window) ring slots.
 * workspace: sn_attn_decode_workspace_bytes(); counters: B*Hkv int32 zeroed
 * once at allocation (the kernel leaves them zero).                       */
size_t sn_attn_decode_workspace_bytes(int B, int Hq, int Hkv, int D, int max_splits);
sn_status sn_attn_decode(const void* q, const void* k_cache, const void* v_cache,
                         const int32_t* block_table, const int32_t* seq_lens,
                         void* out, float* workspace, int32_t* counters, int B,
                         int Hq, int Hkv, int D, int page_size, int max_blocks,
                         int window, int split_pages, int max_splits, float scale,
                         int dtype, void* stream);

/* Causal (window==0) or sliding-window prefill attention over packed sequences:
 * q [rows][Hq][D] (cu_seqlens).  Plain prefill (cu_k, q_off NULL): k/v are the
 * same rows [rows][Hkv][D].  Continuation: k/v [rows_k][Hkv][D] hold each
 * sequence's keys packed by cu_k, and query row r of sequence s attends as key
 * index cu_k[s] + (r - cu_seqlens[s]) + q_off[s] (q_off = position of the first
 * new token minus the position of the first packed key).                     */
sn_status sn_attn_prefill(const void* q, const void* k, const void* v,
                          const int32_t* cu_seqlens, const int32_t* cu_k,
                          const int32_t* q_off, void* out, int num_seqs, int rows,
                          int rows_k, int Hq, int Hkv, int D, int window,
                          float scale, int dtype, void* stream);

/* ---------------------------------------------------------------- GDN / KDA
 * R/PAPER.md:1565-1625.  Decode = the in-projection (sn_gemm_decode STORE) and one fused
 * kernel per layer: causal-conv update (+SiLU), L2-norm q,k, gates, delta-rule state update
 * in place, o = S^T q, gated RMSNorm.  State in HBM is touched exactly once (read + write),
 * in coalesced 512 B column rows.  Replaces FLA's fused_recurrent_gated_delta_rule /
 * fused_recurrent_kda decode path (3P-FLA/ops/gated_delta_rule/fused_recurrent.py:291-337)
 * behind the paper's GDN / KDA mixers.  conv_width must be 4.
 *
 * GDN proj row layout (one fused in-proj GEMM output, R/PAPER.md:1584-1587):
 *   [ q Hk*D | k Hk*D | v Hv*D | z Hv*D | b Hv | a Hv ]   conv channels = q|k|v
 *   g = -exp(A_log[h]) * softplus(a + dt_bias[h]),  beta = sigmoid(b),
 *   out = RMSNorm(o) * norm_w * silu(z)
 * proj is a [B][proj_stride] dtype matrix.                                        */
sn_status sn_gdn_decode(const void* proj, int proj_stride, void* conv_ring,
                        const void* conv_w, float* state, const int32_t* slot_idx,
                        const int32_t* positions, const float* A_log,
                        const float* dt_bias, const void* norm_w, void* out, int B,
                        int Hk, int Hv, int D, int conv_width, float scale,
                        float eps_l2, float eps_norm, int dtype, void* stream);

/* KDA proj row layout: [ q H*D | k H*D | v H*D | f1 R | g1 R | b H ]
 *   g[h,i] = -exp(A_log[h]) * softplus(f[h*D+i] + dt_bias[h*D+i]),  f = f1 @ f2_w^T
 *   out = RMSNorm(o) * norm_w * sigmoid(g1 @ g2_w^T + g2_b)
 * fg = [B][2*H*D] dtype: row b = [f1 @ f2_w^T | g1 @ g2_w^T], the second low-rank factors,
 * from one decode GEMM of the adjacent [f1 | g1] columns of proj against the block-diagonal
 * [f2_w 0; 0 g2_w] (R/PAPER.md:1614-1622).                                              */
sn_status sn_kda_decode(const void* proj, int proj_stride, const void* fg, void* conv_ring,
                        const void* conv_w, float* state, const int32_t* slot_idx,
                        const int32_t* positions, const float* A_log,
                        const float* dt_bias, const void* g2_b, const void* norm_w, void* out,
                        int B, int H, int D, int rank, int conv_width, float scale,
                        float eps_l2, float eps_norm, int dtype, void* stream);

/* Prefill building blocks (sequences packed by cu_seqlens).                */
/* y[t, c] = silu(sum_w conv_w[c,w] * x[t-(W-1)+w, c]) for c < channels (x
 * row stride x_stride); leaves the conv ring of slot_idx[s] in the decode
 * layout.  Continuation (appending to a live sequence): pos0[s] is the
 * absolute position of the first new token and ring_hist a copy of the rings
 * [num_seqs][channels][W] taken before the launch (inputs before pos0 come
 * from it); both NULL = start from an empty ring at position 0.            */
sn_status sn_conv_prefill(const void* x, int x_stride, void* y, const void* conv_w,
                          void* conv_ring, const void* ring_hist,
                          const int32_t* cu_seqlens, const int32_t* slot_idx,
                          const int32_t* pos0, int num_seqs, int rows, int channels,
                          int width, int dtype, void* stream);

/* Per-token gate prep: qn/kn = l2norm(q/k) (qn also * scale), fp32 [rows][Hk][D];
 * gexp = exp(g) fp32 ([rows][Hv] for GDN, [rows][Hv][D] for KDA);
 * beta fp32 [rows][Hv].  kind: 0 = GDN (a, b read from proj), 1 = KDA
 * (f = pre-softplus gate [rows][Hv*D] from the f2 GEMM, b from proj).       */
sn_status sn_delta_prep(int kind, const void* qkv_conv, const void* proj,
                        int proj_stride, int b_off, int a_off, const void* f,
                        const float* A_log, const float* dt_bias, void* qn,
                        void* kn, float* gexp, float* glog, float* beta, int rows,
                        int Hk, int Hv, int D, float scale, float eps_l2, int qk_dtype,
                        int dtype, void* stream);
/* (glog, optional, GDN only: the log decay g per [row][Hv], for the chunked prefill) */

/* Recurrent scan over each sequence: o[t] (fp32 [rows][Hv][D]) and the final
 * state written to state[slot_idx[s]] (read first if init_state != 0).      */
sn_status sn_delta_scan(int kind, const float* qn, const float* kn,
                        const void* qkv_conv, int v_off, int qkv_stride,
                        const float* gexp, const float* beta, float* o,
                        float* state, const int32_t* slot_idx,
                        const int32_t* cu_seqlens, int num_seqs, int Hk, int Hv,
                        int D, int init_state, int dtype, void* stream);

/* Two-phase chunked GDN prefill (long prompts): phase 1 computes every chunk's
 * local WY tiles in parallel (one CTA per (chunk, value head), TMA-fed tcgen05 /
 * TMEM products: K K^T, Q K^T, T diag(b e^G) K, T diag(b) V), phase 2 runs the
 * sequential state pass over precomputed bf16 tiles streamed through
 * double-buffered shared memory.  qn / kn: bf16 [rows][Hk][D] (sn_delta_prep with
 * qk_dtype SN_BF16); qkv_conv [rows][qkv_stride] bf16 (v_off a multiple of 64).  chunks: int32 [num_chunks][2] = (first token,
 * length <= 64) in sequence order; seq_chunk0: int32 [num_seqs+1] chunk offsets.
 * workspace: sn_gdn_chunk_workspace_bytes(num_chunks, Hv, D).                     */
size_t sn_gdn_chunk_workspace_bytes(int num_chunks, int Hv, int D);
sn_status sn_gdn_chunk_prefill2(const void* qn, const void* kn, const void* qkv_conv,
                                int v_off, int qkv_stride, int rows, const float* glog,
                                const float* beta, const int32_t* chunks,
                                const int32_t* seq_chunk0, int num_chunks, void* workspace,
                                float* o, float* state, const int32_t* slot_idx, int num_seqs,
                                int Hk, int Hv, int D, int init_state, int dtype, void* stream);

/* Two-phase chunked KDA prefill: the same WY chunk form with a per-key-channel
 * gate (FLA naive_chunk_kda, 3P-FLA/ops/kda/naive.py:69-166).  Hk = Hv = H;
 * glog: fp32 [rows][H][D] per-channel log gates (sn_delta_prep kind 1 with glog);
 * qn / kn: bf16 [rows][H][D] (TMA tiles; sn_delta_prep with qk_dtype SN_BF16);
 * workspace: sn_kda_chunk_workspace_bytes(num_chunks, H, D).  Replaces the
 * token-sequential sn_delta_scan(kind=1) for bf16 prompts.                      */
size_t sn_kda_chunk_workspace_bytes(int num_chunks, int H, int D);
sn_status sn_kda_chunk_prefill2(const void* qn, const void* kn, const void* qkv_conv,
                                int v_off, int qkv_stride, int rows, const float* glog,
                                const float* beta, const int32_t* chunks,
                                const int32_t* seq_chunk0, int num_chunks, void* workspace,
                                float* o, float* state, const int32_t* slot_idx,
                                int num_seqs, int H, int D, int init_state,
                                int dtype, void* stream);

/* out[r,h,:] = RMSNorm(o[r,h,:]) * norm_w * act(gate[r, h*D + :]),
 * act: 0 = silu (GDN), 1 = sigmoid (KDA).  gate row stride gate_stride.    */
sn_status sn_gated_rmsnorm(const float* o, const void* gate, int gate_stride,
                           const void* norm_w, void* out, int rows, int H, int D,
                           float eps, int act, int dtype, void* stream);

/* ---------------------------------------------------------------- head-parallel decode
 * Row-parallel projection all-reduce fused into the residual add + RMSNorm over peer
 * memory (NVLink P2P; csrc/sn_tp.cu).  Each rank's symmetric buffer (CUDA IPC, mapped in
 * every peer) holds an arrival counter and fp32 split-K slabs; the rank writes its partial
 * product there (sn_gemm_decode PARTIAL), bumps its counter (sn_tp_arrive), and
 * sn_tp_allreduce_add_rmsnorm waits for every peer's counter to reach its own, then sums all
 * ranks' slabs in rank order (bit-identical on every rank), adds the residual and normalises.
 * peer_slabs / peer_counters: device arrays of `world` addresses (this rank's included).
 * Replaces the NCCL all-reduce after the out-projection (north_star, config 5).          */
sn_status sn_tp_arrive(unsigned int* counter, void* stream);
sn_status sn_tp_allreduce_add_rmsnorm(const unsigned long long* peer_slabs,
                                      const unsigned long long* peer_counters, int world,
                                      int rank, int nsplit, float* residual,
                                      const void* weight, void* out, int rows, int dim,
                                      float eps, int dtype, void* stream);

/* ---------------------------------------------------------------- decode GEMM
 * Weight-streaming projection GEMM for decode batches: C[m][n] = sum_k X[m][k] W[n][k],
 * X [M][ldx], W [N][ldw] (nn.Linear layout), every projection of the decode step (the
 * trunk of R/PAPER.md:175-182 and each mixer's projections, R/PAPER.md:1540-1625).
 * bf16 (M <= 128): tcgen05/TMEM/TMA, the batch tile as the UMMA M operand and weight
 * blocks as N, (block, K split) items dealt to a persistent grid, block height / split
 * count chosen per shape to balance the SMs (sn_gemm_decode_plan), programmatic dependent
 * launch.  fp32 (numerics mode, any M): CUDA-core tiles with the same epilogues.
 *   SN_GEMM_STORE    : out T [M][ldo] = C
 *   SN_GEMM_RESID    : out fp32 [M][ldo] += C  (residual stream)
 *   SN_GEMM_PARTIAL  : out fp32 [S][M][ldo]: K split s writes slab s; S (1..8) is returned
 *                      in *splits_out; the consumer sums the slabs in order (sn_add_rmsnorm)
 *   SN_GEMM_SWIGLU_IL: W in blocks of h gate rows followed by the same h up rows
 *                      (h = sn_gemm_swiglu_block(N), last block zero-padded to 2h rows);
 *                      out T [M][ldo] = silu(C_gate) * C_up, N = FFN width
 *   SN_GEMM_ATTN_IN  : attention in-projection with RoPE + KV append fused
 *                      (sn_gemm_decode_attn_in)                                         */
typedef enum {
  SN_GEMM_STORE = 0,
  SN_GEMM_RESID = 2,
  SN_GEMM_PARTIAL = 3,
  SN_GEMM_SWIGLU_IL = 4,
  SN_GEMM_ATTN_IN = 6
} sn_gemm_mode;
int sn_gemm_swiglu_block(int N);
/* plan introspection: out[6] = {block rows, K splits, atoms per stage, blocks, grid, stages} */
int sn_gemm_decode_plan(int M, int N, int K, int mode, int* out);
/* tuning hook for benchmarks: force block rows (multiple of 16), atoms per stage, K splits
 * (PARTIAL) and a smaller grid for later launches in this process; zeros = the built-in plan */
void sn_gemm_decode_tune(int br, int ks, int splits, int grid);
sn_status sn_gemm_decode(const void* x, int M, int K, int ldx, const void* w, int N, int ldw,
                         void* out, int ldo, int mode, int* splits_out, int dtype, void* stream);
/* Attention in-projection.  W = [q Hq*D | k Hkv*D | v Hkv*D] rows with the q and k rows of
 * every head rotary-pair interleaved (sn_rope_pair_interleave order: row 2i = dim i, row 2i+1
 * = dim i + D/2; v rows as is).  q_out [M][Hq][D] gets RoPE(q) at positions[m]; RoPE(k) and
 * v are appended to the page pool at slot (window ? pos % window : pos) through block_table
 * [M][max_blocks] (the decode half of sn_rope_kv_append).  A slot past the block table is
 * not written and sets *err_flag = 1 (err_flag may be NULL).                           */
sn_status sn_gemm_decode_attn_in(const void* x, int M, int K, int ldx, const void* w, int ldw,
                                 const int32_t* positions, const float* inv_freq, void* q_out,
                                 void* k_cache, void* v_cache, const int32_t* block_table,
                                 int Hq, int Hkv, int D, int page_size, int max_blocks,
                                 int window, int32_t* err_flag, const void* rope_cs, int dtype,
                                 void* stream);

/* ---------------------------------------------------------------- fused decode chain
 * Everything between two mixer kernels of the decode step in ONE persistent launch
 * (R/PAPER.md:175-182 trunk + the mixers' projections, R/PAPER.md:1540-1625): e.g.
 * out-proj(l) -> add+RMSNorm -> FFN gate/up (SwiGLU) -> down -> add+RMSNorm -> in-proj(l+1)
 * [-> KDA gate factors].  GEMM phases are the decode GEMM above (same plans and epilogues);
 * NORM phases are sn_add_rmsnorm with split-K slabs, one batch row per CTA.  A grid-wide
 * barrier separates a phase from the one it depends on; the weights of the next GEMM phase
 * stream into shared memory while CTAs wait at it, so HBM never idles between projections.
 * One CTA per SM (grid <= #SMs, all co-resident).  bf16, M <= 128.
 * counter: one 64-bit device word per chain call site, zero-initialised once and never
 * reset (the barrier targets are taken modulo the per-launch arrival count).          */
typedef enum { SN_CHAIN_GEMM = 0, SN_CHAIN_NORM = 1 } sn_chain_kind;
typedef struct {
  int kind;      /* sn_chain_kind */
  int depends;   /* 1: reads what the phase before it wrote (a grid barrier separates them) */
  /* GEMM: out (+)= x[M][K] @ w[N][K]^T with the sn_gemm_mode epilogue `mode` */
  const void* x;
  int K, ldx;
  const void* w;
  int N, ldw;
  void* out;
  int ldo, mode;
  /* SN_GEMM_ATTN_IN epilogue (see sn_gemm_decode_attn_in) */
  const int32_t* positions;
  const float* inv_freq;
  void* q_out;
  void* k_cache;
  void* v_cache;
  const int32_t* block_table;
  int Hq, Hkv, D, page_size, max_blocks, window;
  int32_t* err_flag;
  const void* rope_cs;  /* optional (cos, sin) table from sn_embed */
  /* NORM: residual[M][dim] += sum of slabs partials[0..nsplit) (slab order; nsplit < 0: the K
   * splits of the latest PARTIAL GEMM phase before it); norm_out = rmsnorm(residual) * weight */
  const float* partials;
  int nsplit;
  float* residual;
  const void* weight;
  void* norm_out;
  int dim;
  float eps;
  /* GEMM SN_GEMM_RESID: optional [blocks][M] fp32 per-row sums of squares of the updated residual
   * over each weight block's columns; NORM: take the row's sum of squares from such a buffer
   * (n_ss blocks; n_ss < 0: the blocks of the latest RESID GEMM phase before it) */
  float* ss_out;
  const float* ss_in;
  int n_ss;
  int splits;    /* out: K splits the planner chose for a PARTIAL GEMM phase */
} sn_chain_phase;
sn_status sn_decode_chain(sn_chain_phase* phases, int n_phases, int M, unsigned long long* counter,
                          void* stream);
/* instrumentation: later launches write per-CTA %globaltimer stamps to buf ([grid][40] u64:
 * start, end, and per phase: inputs ready, outputs done, arrival, norm release); NULL = off */
void sn_decode_chain_trace(unsigned long long* buf);

/* ---------------------------------------------------------------- prefill GEMM
 * The projections of a prefill (every packed prompt row at once): C[m][n] = sum_k A[m][k]
 * W[n][k], A [M][lda] bf16, W [N][ldw] bf16 (nn.Linear layout), out [M][ldo].
 * tcgen05/TMEM/TMA, 2-CTA (cta_group::2) 256 x br output tiles on a persistent grid of CTA
 * pairs in L2-friendly bands.  mode SN_GEMM_STORE (out bf16), SN_GEMM_PARTIAL (out fp32: the
 * row-parallel projections whose partials a tensor-parallel prefill sums in fp32) or
 * SN_GEMM_SWIGLU_IL (W in blocks of swiglu_h gate rows then swiglu_h up rows, out bf16 =
 * silu(gate) * up, N = FFN width; swiglu_h a multiple of 16 <= 128).
 * Replaces the cuBLAS projections of the prefill (R/PAPER.md:845-848 dual path).          */
sn_status sn_gemm_prefill(const void* a, int M, int K, int lda, const void* w, int N, int ldw,
                          void* out, int ldo, int mode, int swiglu_h, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SN_ABI_H_ */
