/* qigen_b200.h — C ABI of libqigen_b200.so, the B200 (sm_100a) implementation
 * of QIGen's quantized-GEMV hot path (arXiv 2307.03738).
 *
 * Plain pointers and sizes only.  Every pointer argument is a DEVICE pointer
 * unless its name ends in `_host`.  `stream` is a cudaStream_t (NULL = legacy
 * default stream).  Every call is stream-ordered and returns a qigen_status;
 * on failure qigen_last_error() returns a message.  Status codes map onto the
 * reference's exception classes (config.py:34 ConfigError, packing.py:35
 * PackError, perfmodel.py:20 PlanError, all ValueError subclasses).
 *
 * Orientation follows the reference: W is n x m (n = K input
 * rows, m = N output columns), groups run along n per column, y = x W.
 *
 * Which reference interface each entry point replaces is cited on it; the
 * reference has no native FFI of its own — its seam is the runtime op
 * qgemv(pm, x, sums, threads) and the generated-kernel
 * calling convention (kernelgen.py:399-401).  INTEGRATION.md shows the
 * ctypes binding a maintainer of the reference would add.
 */
#ifndef QIGEN_B200_H_
#define QIGEN_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  QIGEN_OK = 0,
  QIGEN_ERR_CONFIG = 1,      /* ConfigError  (config.py:34)  */
  QIGEN_ERR_PACK = 2,        /* PackError    (packing.py:35) */
  QIGEN_ERR_PLAN = 3,        /* PlanError    (perfmodel.py:20) */
  QIGEN_ERR_CUDA = 4,        /* CUDA runtime failure          */
  QIGEN_ERR_ARG = 5,         /* null pointer / bad size       */
  QIGEN_ERR_UNSUPPORTED = 6  /* combination not implemented   */
} qigen_status;

typedef enum { QIGEN_ZERO_REAL32 = 0, QIGEN_ZERO_QUANTIZED = 1 } qigen_zero_mode; /* config.py:17-31 */
typedef enum { QIGEN_LAYOUT_ROW_SEQUENTIAL = 0, QIGEN_LAYOUT_ZCURVE = 1 } qigen_layout; /* packing.py:30-32 */
typedef enum { QIGEN_F32 = 0, QIGEN_F16 = 1, QIGEN_BF16 = 2 } qigen_dtype;

/* Flags for the `accumulate` argument of the GEMV entry points (bit set). */
#define QIGEN_GEMV_ACCUMULATE 1 /* y += x W instead of y = x W */
/* x is final before this launch (e.g. independent GEMVs back to back on inputs
 * prepared earlier): the GEMV reads and digitises x before its
 * programmatic-dependent-launch wait and waits only before writing y, so it
 * overlaps its predecessor completely; such a GEMV also lets ITS successor start
 * early.  So x must not be written by ANY kernel that may still be in flight
 * in the chain of early-starting launches before it, not just by the kernel
 * launched immediately before: G1 (writes h), G2 (X_READY, independent), G3
 * (X_READY, x = h) is wrong, because G3 can read h before G1 has written it.
 * Never set it when x is produced by a kernel of the same stream that was
 * launched after the last launch without this flag. */
#define QIGEN_GEMV_X_READY 2

int qigen_version(void);
const char* qigen_last_error(void);

/* ---- quantization (bit-exact with quant.py) ------------------------------- */

/* quant.py:119-127 quantize_matrix (+ _quantize_blocks :74-94).
 * w: f32 [n, m] row-major.  group_size 0 = FULL_COLUMN (config.py:12).
 * codes: u8 [n, m]; scales, zeros: f32 [G, m], G = n/group_size (1 for FC). */
int qigen_quantize(const float* w, int64_t n, int64_t m, int bits, int64_t group_size,
                   int zero_mode, uint8_t* codes, float* scales, float* zeros, void* stream);

/* quant.py:130-138 dequantize_matrix: out[n, m] = f32(s * (f32(code) - z)). */
int qigen_dequantize(const uint8_t* codes, const float* scales, const float* zeros,
                     int64_t n, int64_t m, int64_t group_size, float* out, void* stream);

/* ---- packing (bit-exact with packing.py) ---------------------------------- */

/* packing.py:204-214 _pack_matrix_rowseq: codes [n, m] -> n*m*bits/32 words,
 * word (r, k, c) at (r*Kw + k)*m + c (Kw = 3 for 3-bit, else 1). */
int qigen_pack_rowseq(const uint8_t* codes, int64_t n, int64_t m, int bits, uint32_t* words,
                      void* stream);
/* packing.py:229-242 extract_codes (ROW_SEQUENTIAL part): words -> codes [n, m]. */
int qigen_unpack_rowseq(const uint32_t* words, int64_t n, int64_t m, int bits, uint8_t* codes,
                        void* stream);
/* packing.py:175-201 _storage_permutation applied to words.  blk_rc holds the
 * (row_block, col_block) pairs in Morton storage order (packing.py:110-114),
 * int32 [nblk * 2], device memory.  to_zcurve=1: rowseq -> zcurve, 0: inverse. */
int qigen_permute_zcurve(const uint32_t* src, uint32_t* dst, int64_t n, int64_t m, int bits,
                         int64_t m_b, int64_t t_b, const int32_t* blk_rc, int64_t nblk,
                         int to_zcurve, void* stream);

/* ---- GPU panel layout --------------------------------------- */

/* Sizes of the panel layout: uint32 words of packed codes and float2 (s, z)
 * pairs.  K is padded to a multiple of 256 and m to a multiple of 16. */
int64_t qigen_panel_words(int64_t n, int64_t m, int bits);
int64_t qigen_panel_params(int64_t n, int64_t m, int64_t group_size);

/* Re-tile codes + scales/zeros into the panel layout (qw, qsz). */
int qigen_panels_from_codes(const uint8_t* codes, const float* scales, const float* zeros,
                            int64_t n, int64_t m, int bits, int64_t group_size, uint32_t* qw,
                            float* qsz, void* stream);
/* Inverse of the code part (round-trip tests). */
int qigen_panels_to_codes(const uint32_t* qw, int64_t n, int64_t m, int bits, uint8_t* codes,
                          void* stream);
/* Re-tile directly from reference ROW_SEQUENTIAL words (3-bit straddles of the
 * 96-bit stream, kernelgen.py:116-124, are resolved here). */
int qigen_panels_from_rowseq(const uint32_t* words, const float* scales, const float* zeros,
                             int64_t n, int64_t m, int bits, int64_t group_size, uint32_t* qw,
                             float* qsz, void* stream);

/* ---- the hot path ----------------------------------------------------------- */

/* Per-group input sums (Eq. 2): out[G] (FC: out[0] = total).
 * fp64 accumulation, rounded once to f32. */
int qigen_input_sums(const float* x, int64_t n, int64_t group_size, float* out, void* stream);

/* Replaces qgemv(pm, x, sums, threads) and the generated
 * kernel it drives (kernelgen.py:371-423).  x: `tokens` rows of n activations
 * (dtype x_dtype, row stride ldx elements); y: f32 [tokens, m] with row stride
 * ldy.  accumulate: 0 overwrites y, QIGEN_GEMV_ACCUMULATE adds to it, optionally
 * or-ed with QIGEN_GEMV_X_READY (see above).  k_splits=0 picks the K split
 * automatically.  Deterministic: results do not depend on the launch shape
 * beyond (n, m, bits, group_size, tokens, k_splits).  Input sums are fused. */
int qigen_gemv(const uint32_t* qw, const float* qsz, int64_t n, int64_t m, int bits,
               int64_t group_size, const void* x, int x_dtype, int64_t tokens, int64_t ldx,
               float* y, int64_t ldy, int accumulate, int k_splits, void* stream);

/* qigen_gemv with a fused activation prologue (the decode driver's glue):
 *   prologue 0: x as given;
 *   prologue 1: RMSNorm, x_k * rsqrt(mean_k(x^2) + eps) * prologue_w[k] (LLaMA RMSNorm);
 *   prologue 2: SwiGLU, silu(x[t, k]) * x[t, n + k] (x holds gate | up, ldx >= 2n);
 *   prologue 3: RMSNorm with its weight folded into W at quantization: y[t] =
 *     rsqrt(mean_k(x[t]^2) + eps) * (x[t] W), the 1/rms applied in the epilogue
 *     from the sums of squares of the x chunks (fixed reduction order).
 * workspace (device, >= qigen_gemv_workspace_size bytes, or NULL): scratch for the
 * activation digits when they are prepared once per call (long K chunks / many
 * tokens).  NULL allocates that scratch stream-ordered for this call
 * (cudaMallocFromPoolAsync / cudaFreeAsync on `stream`; a graph memory node
 * under capture), so concurrent calls on different streams never share it; the
 * stream-ordered free ends the programmatic-launch overlap with the next
 * kernel, so hot paths pass a workspace.  Every GEMV entry point is re-entrant
 * across streams and host threads: the only shared state is read-only
 * (weights) or caller-owned (x, y, workspace). */
int64_t qigen_gemv_workspace_size(int64_t n, int64_t tokens);
int qigen_gemv_ex(const uint32_t* qw, const float* qsz, int64_t n, int64_t m, int bits,
                  int64_t group_size, const void* x, int x_dtype, int64_t tokens, int64_t ldx,
                  float* y, int64_t ldy, int accumulate, int k_splits, int prologue,
                  const float* prologue_w, float eps, void* workspace, int64_t workspace_bytes,
                  void* stream);

/* Dependent GEMV chains of the decode driver without activation prep kernels.
 * A PRODUCER GEMV (y_digits set) writes its final output columns (after the
 * residual add) twice: as y, and as the prepared activation digits of the
 * consumer GEMV whose K is this m (times out_scale[col], e.g. the consumer's
 * RMSNorm weight), together with per-CTA sums of squares of y in
 * ss_out[t * qigen_gemv_ss_count(m) + cta].  The CONSUMER (x_digits set) reads
 * those digits instead of x (no prologue, no prep kernel) and, with ss_in,
 * applies the RMSNorm's 1 / rms = rsqrt(sum_c ss_in[t * ss_count + c] / n + eps)
 * in its epilogue (fixed summation order).  Digit buffers are
 * qigen_gemv_workspace_size(K, tokens) bytes, zero-filled once; producer and
 * consumer use the same token count.  Consumer group sizes 32..256 / FC. */
typedef struct {
  const void* x_digits;   /* consumer: prepared digits (or NULL: x as usual) */
  const float* ss_in;     /* consumer: producer's sums of squares (or NULL) */
  int ss_count;
  float eps;
  void* y_digits;         /* producer: consumer's digit buffer (or NULL) */
  const float* out_scale; /* producer: per-column multiplier (or NULL) */
  int64_t out_group;      /* producer: consumer's group size (0 = FC) */
  float* ss_out;          /* producer: sums of squares of y per CTA (or NULL) */
} qigen_gemv_chain_opts;
int64_t qigen_gemv_ss_count(int64_t m);
int qigen_gemv_chain(const uint32_t* qw, const float* qsz, int64_t n, int64_t m, int bits,
                     int64_t group_size, const void* x, int x_dtype, int64_t tokens, int64_t ldx,
                     float* y, int64_t ldy, int accumulate, int prologue, const float* prologue_w,
                     float eps, void* workspace, int64_t workspace_bytes,
                     const qigen_gemv_chain_opts* opts, void* stream);

/* ---- grouped GEMV: many independent GEMVs in one persistent launch ----------
 * Replaces a sequence of independent qgemv(pm_i, x_i) calls of the reference
 * runtime (e.g. its bench over a sweep of matrices,
 * SPEC.md:418-426) by one schedule over all of them: one CTA per SM streams
 * (GEMV, 128 columns, full K) work items back to back, so no per-GEMV launch
 * latency or split-K reduction sits between them.  Each descriptor has the
 * meaning of the qigen_gemv arguments (panel-layout weights, 1..2 activation
 * rows).  Pointers are captured at create time; run() may be graph-captured.
 * x and y may point into page-locked host memory (device-accessible under UVA):
 * the activation prep then reads x over PCIe instead of needing an H2D copy;
 * pageable host memory is rejected (QIGEN_ERR_ARG).  A plan's activation
 * records and schedule counter belong to the plan: run one plan on one stream
 * at a time (different plans run concurrently).
 * Results equal qigen_gemv's to f32 rounding (full-K reduction per column,
 * deterministic). */
typedef struct {
  const uint32_t* qw;
  const float* qsz;
  int64_t n, m;
  int bits;
  int64_t group_size;
  const void* x;
  int x_dtype;
  int64_t tokens, ldx;
  float* y;
  int64_t ldy;
} qigen_gemv_desc;
typedef struct qigen_gemv_group qigen_gemv_group;
int qigen_gemv_group_create(int count, const qigen_gemv_desc* descs, qigen_gemv_group** out);
int qigen_gemv_group_run(const qigen_gemv_group* group, void* stream);
int qigen_gemv_group_destroy(qigen_gemv_group* group);
/* run() with every y pointer moved by (y_base - y_plan_base) bytes: the same
 * plan writes a fresh output block per call (e.g. page-locked host memory, the
 * zero-copy qgemv_batch result: GEMVs whose y is host memory are never K-split,
 * so their outputs are plain 32-byte coalesced stores).  QIGEN_ERR_ARG when
 * y_base is pageable host memory, or host memory while the plan (created with
 * device y) K-splits some GEMV. */
int qigen_gemv_group_run_rebased(const qigen_gemv_group* group, const void* y_plan_base,
                                 void* y_base, void* stream);
/* Host-buffer form of a group run, the blocking qgemv_batch round trip
 * (SPEC.md:349-357 returns host results): x_bytes from pinned host x_host to
 * x_dev (the device block the group's descriptors point into), the run, y_bytes
 * from y_dev back to pinned host y_host, then a stream synchronize. */
int qigen_gemv_group_run_host(const qigen_gemv_group* group, const void* x_host, void* x_dev,
                              size_t x_bytes, const void* y_dev, void* y_host, size_t y_bytes,
                              void* stream);

/* ---- decode-step glue (LLaMA driver) ----------------------------------------- */

/* RoPE on q and k of a fused QKV output qkv f32 [B, 3, H, hd] at position pos
 * (cos/sin: [hd/2] for that position); q -> f16 [B, H, hd]; k, v appended (f16)
 * to the layer's caches [B, H, ctx, hd] at pos. */
int qigen_rope_kv(const float* qkv, int64_t batch, int64_t heads, int64_t head_dim,
                  const float* cos_pos, const float* sin_pos, void* q_out, void* k_cache,
                  void* v_cache, int64_t ctx, int64_t pos, void* stream);
/* out f16 [rows, d] = h * rsqrt(mean(h^2) + eps) * w. */
int qigen_rmsnorm_f16(const float* h, const float* w, int64_t rows, int64_t d, float eps,
                      void* out, void* stream);

/* Fused decode attention for one new token per sequence (flash-decoding split
 * over positions): RoPE on q and the new k at `pos` (cos_pos/sin_pos: [hd/2]),
 * append of k and v to the f16 caches [batch, heads, ctx, hd], softmax(q K^T *
 * scale) V over positions 0..pos, out f32 [batch, heads * hd].  head_dim 64 or
 * 128.  workspace: >= qigen_attn_decode_workspace_size bytes, zero-filled once
 * before first use (the kernel leaves it reusable).  Launched with programmatic
 * dependent launch: the cached K/V rows stream before the wait on the kernel
 * that produced qkv.  Replaces the torch SDPA + RoPE glue of the decode driver
 * (no reference counterpart: SPEC.md:13,384). */
int64_t qigen_attn_decode_workspace_size(int64_t batch, int64_t heads, int64_t head_dim,
                                         int64_t ctx);
int qigen_attn_decode(const float* qkv, int64_t batch, int64_t heads, int64_t head_dim,
                      const float* cos_pos, const float* sin_pos, void* k_cache, void* v_cache,
                      int64_t ctx, int64_t pos, float scale, float* out, void* workspace,
                      int64_t workspace_bytes, void* stream);

/* ---- tensor-parallel one-shot all-reduce (decode driver)
 * Row-parallel layers push their partial outputs from the GEMV epilogue
 * straight into every rank's inbox over NVLink (peer-mapped device memory) and
 * count the columns they delivered; each rank then adds the partials to its
 * residual in rank order.  No NCCL call on the data path; results bit-identical
 * on every rank.  Protocol and layout: csrc/tp.cuh, DESIGN.md §7.  Replaces the
 * torch.distributed/NCCL all-reduce the driver issues after o_proj and
 * down_proj (no reference counterpart: the reference is single-process,
 * SPEC.md:376). */
typedef struct qigen_tp_comm qigen_tp_comm;
/* Bytes of each rank's buffer (header + 2 slots x world x max_tokens x d f32). */
int64_t qigen_tp_buffer_size(int world, int64_t d, int64_t max_tokens);
/* cudaMalloc + zero a buffer; ipc_handle_out (64 bytes, or NULL) receives its
 * cudaIpcMemHandle for the peers. */
int qigen_tp_alloc(int64_t bytes, void** ptr, void* ipc_handle_out);
int qigen_tp_free(void* ptr);
/* Map a peer's buffer (cudaIpcOpenMemHandle, lazy peer access). */
int qigen_tp_open_peer(const void* ipc_handle, void** ptr);
int qigen_tp_close_peer(void* ptr);
/* bases[q] = rank q's buffer as addressable from this process (bases[rank] is
 * this rank's own).  Ranks emulated on one GPU pass each other's plain device
 * pointers.  `layers` = uses of each slot per decode step. */
int qigen_tp_create(int rank, int world, int64_t d, int64_t max_tokens, int layers,
                    void* const* bases, qigen_tp_comm** out);
int qigen_tp_destroy(qigen_tp_comm* comm);
/* Start of a decode step on this rank (advances the epoch the reduces wait for). */
int qigen_tp_step_begin(const qigen_tp_comm* comm, void* stream);
/* Row-parallel qigen_gemv_ex (accumulate 0, automatic K split) whose epilogue
 * stores the partial into slot `slot` of every rank instead of a local y. */
int qigen_gemv_tp_push(const qigen_tp_comm* comm, int slot, const uint32_t* qw, const float* qsz,
                       int64_t n, int64_t m, int bits, int64_t group_size, const void* x,
                       int x_dtype, int64_t tokens, int64_t ldx, int prologue,
                       const float* prologue_w, float eps, void* workspace,
                       int64_t workspace_bytes, void* stream);
/* h[tokens, d] += sum of the ranks' partials of slot `slot`, use `layer` of the
 * current step, in rank order (waits for every rank's columns; a wait longer
 * than 4 s sets the error flag instead of hanging). */
int qigen_tp_reduce(const qigen_tp_comm* comm, int slot, int layer, float* h, int64_t tokens,
                    void* stream);
/* 1 if a reduce on this rank timed out since the last call (then cleared). */
int qigen_tp_error(const qigen_tp_comm* comm, int* out);

/* Vocab-parallel LM head with the greedy argmax fused: for each
 * of `batch` (1..8) tokens, xn = fp16(h * rsqrt(mean(h^2) + eps) * norm_w),
 * logits[b, v] = xn . W[v] (W fp16 [vocab, d] row-major, f32 accumulation,
 * written when `logits` is non-NULL), out_max[b] / out_idx[b] = the maximum and
 * vocab_offset + its row (lowest row on ties).  A rank of a vocab-parallel
 * group reduces (out_max, out_idx) across ranks instead of gathering logits.
 * workspace >= qigen_lm_head_workspace_size bytes, zero-filled once before
 * first use (the kernel leaves it zeroed).  Deterministic for any grid.
 * Replaces the decode driver's cuBLAS GEMV + argmax (no reference counterpart,
 * SPEC.md:13). */
int64_t qigen_lm_head_workspace_size(int64_t vocab, int64_t d, int64_t batch);
int qigen_lm_head(const float* h, const float* norm_w, float eps, const void* w_f16,
                  int64_t vocab, int64_t d, int64_t batch, int64_t vocab_offset, float* logits,
                  float* out_max, int64_t* out_idx, void* workspace, int64_t workspace_bytes,
                  void* stream);

/* qigen_attn_decode whose heads also write their outputs as the o_proj GEMV's
 * prepared activation digits (qigen_gemv_chain_opts.x_digits of a GEMV with K
 * = heads * head_dim, `batch` tokens, group size o_group >= 64): the o_proj
 * GEMV then needs no prologue.  head_dim 128. */
int qigen_attn_decode_chain(const float* qkv, int64_t batch, int64_t heads, int64_t head_dim,
                            const float* cos_pos, const float* sin_pos, void* k_cache,
                            void* v_cache, int64_t ctx, int64_t pos, float scale, float* out,
                            void* workspace, int64_t workspace_bytes, void* o_digits,
                            int64_t o_group, void* stream);

/* Small-batch quantized GEMM on the tcgen05 tensor cores (north_star (c)):
 * weights dequantized to fp16 (w = s (c - z)) in shared memory, activations
 * converted to fp16, f32 accumulation in TMEM.  4-bit, group 32..256 (dividing
 * 256), 1..256 tokens (meant for tokens >= 16).  workspace >=
 * qigen_gemm_tc_workspace_size bytes (the fp16 activation tiles). */
int64_t qigen_gemm_tc_workspace_size(int64_t n, int64_t tokens);
int qigen_gemm_tc(const uint32_t* qw, const float* qsz, int64_t n, int64_t m, int bits,
                  int64_t group_size, const void* x, int x_dtype, int64_t tokens, int64_t ldx,
                  float* y, int64_t ldy, int accumulate, int k_splits, void* workspace,
                  int64_t workspace_bytes, void* stream);

/* ---- tuning / debugging aids ------------------------------------------------
 * Not part of the product API: measurement knobs for tools/ and tests.  Each
 * knob is PER CALLING HOST THREAD (thread-local): setting it changes only the
 * launches that thread makes, never another thread's.  Defaults are the
 * product settings. */

/* Debugging aid: when buf is non-NULL every later qigen_gemv launch writes
 * %globaltimer stamps (entry, after the PDL wait, after the activation
 * prologue, after the main loop, exit, ...) to buf[(cta_y*grid_x + cta_x)*16 + i]. */
int qigen_debug_trace(void* buf);
/* Debugging aid: same points as qigen_debug_trace, SM clock64 values. */
int qigen_debug_trace_clk(void* buf);
/* Tuning aid: weight stages per warp issued before griddepcontrol.wait
 * (-1 = the whole first ring fill, the default). */
int qigen_debug_prefetch(int stages_before_wait);
/* Tuning aid: 1 = always digitise activations in the separate prep kernel. */
int qigen_debug_force_prep(int on);
/* Tuning aid: cap the automatic K split (thread-block cluster size) of the GEMV. */
int qigen_debug_max_split(int s);
/* Tuning aid: 1 (default) = GEMVs with the RMSNorm prologue digitise through the
 * one-CTA-per-token prep kernel. */
int qigen_debug_norm_prep(int on);
/* Tuning aid: L2 evict_first on weight copies, warps per CTA (8/16), ring KB per CTA, grid cap. */
int qigen_debug_gemv_tuning(int policy, int wpc, int ring_kb, int max_ctas);
/* Tuning aid: 1 = trigger the dependent launch (PDL) at GEMV kernel entry. */
int qigen_debug_early_trigger(int on);
/* Tuning aid for the tensor-core path: 1 = skip A-tile stores, 2 = skip MMAs. */
int qigen_debug_tc_mode(int mode);
/* Tuning aid for the grouped GEMV: 1 = stream weights and activations only. */
int qigen_debug_group_mode(int mode);
/* Debugging aid: per-CTA %globaltimer stamps of the decode attention kernel
 * (entry, after the PDL wait, before the combine, exit) at buf[cta * 4 + i]. */
int qigen_debug_attn_trace(void* buf);
/* Tuning aid: cap on the position splits (cluster size, <= 16) per head of the decode attention. */
int qigen_debug_attn_splits(int n);

/* ---- persistent decode stack (csrc/decode_stack.cu) --------------------------- */

/* All layers of a batch-1 LLaMA-architecture decode step on one GPU as ONE
 * persistent launch (one CTA per SM; the layers' quantized linears and the
 * attention are phases separated by grid barriers, weights stream through
 * per-warp rings that never drain between phases).  Consumer of the quantized
 * GEMV; no reference counterpart (the reference has no model path),
 * the arithmetic of each linear is that of qigen_gemv (kernelgen.py:227-240).
 * Per layer: RMSNorm -> fused QKV -> RoPE + KV append + attention over
 * positions 0..pos -> o_proj + residual -> RMSNorm -> fused gate|up -> SwiGLU ->
 * down_proj + residual.  Deterministic. */
typedef struct qigen_stack_layer {
  const void* qw[4];    /* panel words of W_qkv [d, 3d] (q | k | v heads), W_o [d, d],
                           W_gate|up [d, 2 ffn], W_down [ffn, d] */
  const void* qsz[4];   /* their (s, z) */
  const float* norm1;   /* RMSNorm weight before QKV [d] */
  const float* norm2;   /* RMSNorm weight before gate|up [d] */
  void* k_cache;        /* f16 [heads][ctx][128]; row `pos` is appended by the step */
  void* v_cache;
} qigen_stack_layer;
typedef struct qigen_stack_desc {
  int32_t layers, d_model, heads, head_dim, ffn, bits;
  int64_t group_size;   /* 32, 64 or 128 */
  int64_t ctx;          /* rows of the KV caches */
  float eps;            /* RMSNorm epsilon */
} qigen_stack_desc;
typedef struct qigen_decode_stack qigen_decode_stack;
/* QIGEN_ERR_UNSUPPORTED for shapes outside the kernel's limits (head_dim != 128,
 * other group sizes, ...): callers fall back to the per-op chain. */
int qigen_decode_stack_create(const qigen_stack_desc* desc, const qigen_stack_layer* layers,
                              qigen_decode_stack** out);
/* h_in: the embedded token f32 [d]; h_out: the residual after the last layer
 * f32 [d] (input of the final RMSNorm + LM head); cosv / sinv: RoPE factors of
 * `pos` f32 [64]; scale: 1 / sqrt(head_dim).  Stream-ordered, graph-capturable.
 * One run at a time per handle. */
int qigen_decode_stack_run(const qigen_decode_stack* s, const float* h_in, float* h_out,
                           const float* cosv, const float* sinv, int64_t pos, float scale,
                           void* stream);
/* Synchronous: non-zero *out if a wait inside the last runs timed out (bit 0: grid
 * barrier, bit 1: weight stage); re-arms the handle. */
int qigen_decode_stack_error(const qigen_decode_stack* s, int* out);
/* grid: CTAs; shape: ring stages * 100000 + supersteps per stage * 10000 + the K
 * slabs of the four GEMV phases as digits (qkv, o, gate|up, down). */
int qigen_decode_stack_info(const qigen_decode_stack* s, int* grid, int* shape, int* smem_bytes);
int qigen_decode_stack_destroy(qigen_decode_stack* s);
/* Tuning aid (per calling thread, read at create): supersteps per weight stage
 * (1 or 2), the cap on ring stages per warp and the K slabs (1, 2 or 4) wanted for
 * the qkv, o, gate|up and down phases as four digits (default 2424). */
int qigen_debug_stack_tuning(int sss, int depth, int ksl);
/* Tuning aid (per calling thread): bits 0-1, read at run: 1 = stream the weights
 * through the rings without the math (results are meaningless): the data-movement
 * floor; bits 2-4, read at create: cap on the position chunks (CTAs) per head of
 * the attention phase (0 = default 4); bits 8+, read at create: (MB + 1) of L2
 * prefetch per phase hand-off. */
int qigen_debug_stack_mode(int mode);

/* ---- owning handle (for C callers; the Python host uses the calls above) ---- */

typedef struct qigen_weights qigen_weights;

/* Build a device-resident weight handle from reference-format device buffers:
 * packed words in `layout` (ZCURVE needs blk_rc/nblk/m_b/t_b, else pass 0),
 * scales/zeros f32 [G, m]. */
int qigen_weights_create(const uint32_t* words, int layout, int64_t n, int64_t m, int bits,
                         int64_t group_size, int64_t m_b, int64_t t_b, const int32_t* blk_rc,
                         int64_t nblk, const float* scales, const float* zeros, void* stream,
                         qigen_weights** out);
int qigen_weights_destroy(qigen_weights* w);
/* qgemv on device buffers through the handle. */
int qigen_weights_gemv(const qigen_weights* w, const void* x, int x_dtype, int64_t tokens,
                       float* y, int accumulate, void* stream);
/* End-to-end call with HOST buffers: copies x_host in, runs the GEMV, copies
 * y_host out and synchronises `stream` (the reference-facing blocking call,
 * SPEC.md:349-357).  Device staging is stream-ordered scratch, so one handle may
 * serve several threads / streams concurrently. */
int qigen_weights_gemv_host(const qigen_weights* w, const float* x_host, int64_t tokens,
                            float* y_host, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* QIGEN_B200_H_ */
