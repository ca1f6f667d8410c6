/* sparsewire_b200 — C ABI of the B200-native structural-plasticity hot path.
 *
 * Every entry point takes plain device pointers and sizes (no torch types),
 * enqueues work on the given CUDA stream (cudaStream_t passed as void*) and
 * returns an sw_status (0 = OK).  Nothing here allocates device memory:
 * persistent buffers are caller-owned (torch tensors in the Python host
 * layer), scratch comes from caller-provided workspace pointers.
 *
 * Each function names the reference interface it replaces
 * (paths relative to /root/reference/pkg/src/sparsewire/).
 */
#ifndef SPARSEWIRE_B200_H
#define SPARSEWIRE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define SW_API __attribute__((visibility("default")))
#else
#define SW_API
#endif

#define SW_ABI_VERSION 1
#define SW_MAX_PLANES 8

/* Status codes; the Python layer maps them onto the reference exception
 * taxonomy of errors.py:4-37. */
typedef enum {
  SW_OK = 0,
  SW_ERR_ROW_FULL = 1,          /* errors.RowFull        */
  SW_ERR_DUPLICATE_EDGE = 2,    /* errors.DuplicateEdge  */
  SW_ERR_SLOT_OUT_OF_RANGE = 3, /* errors.SlotOutOfRange */
  SW_ERR_K_TOO_LARGE = 4,       /* errors.KTooLarge      */
  SW_ERR_STALE_TRANSPOSE = 5,   /* errors.StaleTranspose */
  SW_ERR_INVALID_ARG = 6,       /* ValueError            */
  SW_ERR_CUDA = 7               /* launch / runtime failure */
} sw_status;

/* Padded ragged matrix + slot-aligned variable planes.
 * Replaces RaggedMatrix (connectivity.py:24-62) + SynVarMatrix (:65-88).
 * row_length[num_pre] int32; target[num_pre, stride] int32 (stride =
 * max(max_row_length, 1), connectivity.py:35); planes[p] is
 * [num_pre, stride] with plane_bytes[p] in {4, 8}. */
typedef struct sw_ragged {
  int32_t num_pre;
  int32_t num_post;
  int32_t max_row_length;
  int32_t stride;
  int32_t* row_length;
  int32_t* target;
  int32_t n_planes;
  int32_t plane_bytes[SW_MAX_PLANES];
  void* planes[SW_MAX_PLANES];
} sw_ragged_t;

/* Packed per-(pre, post) bits, LSB-first, tail bits zero.
 * Replaces Bitfield (bitfield.py:19-96). words[num_pre, words_per_row]. */
typedef struct sw_bitfield {
  uint64_t* words;
  int32_t num_pre;
  int32_t num_post;
  int32_t words_per_row;
} sw_bitfield_t;

/* ---- library ---------------------------------------------------------- */
SW_API int sw_abi_version(void);
SW_API const char* sw_last_error(void);
/* Number of kernels this library has enqueued so far (graph capture counts once). */
SW_API long long sw_launch_count(void);
/* Device self-test of the SplitMix64 golden vectors (test_rng.py:118-123);
 * writes mix64(0), mix64(1), mix64(G) into out[3] (device pointer). */
SW_API int sw_rng_selftest(uint64_t* out3, void* stream);

/* ---- counter RNG (rng.py:64-153) --------------------------------------- */
/* out[i] = draw #(counter0 + i) of stream `key`   (CounterRng.u64_array, rng.py:93-96) */
SW_API int sw_rng_u64(uint64_t key, uint64_t counter0, int64_t n, uint64_t* out, void* stream);
/* out[i] = uniform01 of draw #(counter0 + i)       (CounterRng.uniform01_array, rng.py:102-104) */
SW_API int sw_rng_uniform01(uint64_t key, uint64_t counter0, int64_t n, double* out, void* stream);
/* `count` sequential uniform_int(n) draws with exact rejection (rng.py:106-114);
 * out[count] receives the final counter.  Single-stream, for tests. */
SW_API int sw_rng_uniform_int_seq(uint64_t key, uint64_t n, int64_t count, uint64_t* out, void* stream);
/* Per-row child keys: out[r] = child_key(key, r)   (CounterRng.child_key, rng.py:84-86) */
SW_API int sw_rng_child_keys(uint64_t key, int64_t n, uint64_t* out, void* stream);

/* ---- bitfields ----------------------------------------------------------- */
/* Bitfield.randomize (bitfield.py:92-96): word w of row i = draw #(i*W + w). */
SW_API int sw_bitfield_randomize(const sw_bitfield_t* bf, uint64_t key, void* stream);

/* ---- ragged primitives (connectivity.py:91-136) ------------------------- */
/* Remove the marked slots of every row with the exact chained
 * swap-with-last order of remove_slots (connectivity.py:130-136).
 * marked[num_pre, stride] uint8 (nonzero = remove). removed[num_pre] int64
 * receives the per-row count (may be NULL). */
SW_API int sw_ragged_remove_marked(const sw_ragged_t* m, const uint8_t* marked,
                            int64_t* removed, void* stream);

/* Column slice for post-sharded propagation (SURVEY 8e M-prop; no
 * reference counterpart -- the reference propagates over whole rows,
 * connectivity.py:139-148).  dst row i = the synapses of src row i with
 * lo <= target < hi, in src slot order, target - lo, every plane copied;
 * dst->num_post = hi - lo, same num_pre and plane types.  Rows longer than
 * dst->stride are truncated; *max_len (device int32, optional, caller
 * zeroed) gets the longest slice row so the caller can check. */
SW_API int sw_ragged_column_slice(const sw_ragged_t* src, int32_t lo, int32_t hi, const sw_ragged_t* dst,
                                  int32_t* max_len, void* stream);
/* add_synapse (connectivity.py:91-112) on one row: RowFull, DuplicateEdge
 * (when multapse_free), else append post with every plane zeroed and
 * values[p] stored where set_mask[p] != 0.  status (device int32[1]) gets
 * the new slot, or -SW_ERR_ROW_FULL / -SW_ERR_DUPLICATE_EDGE. */
SW_API int sw_ragged_add_synapse(const sw_ragged_t* m, int32_t pre, int32_t post,
                                 const double* values, const uint8_t* set_mask,
                                 int32_t multapse_free, int32_t* status, void* stream);
/* remove_slots / remove_synapse (connectivity.py:115-136) on one row, the
 * reference's descending chained swap-with-last order.  slots[k] (device);
 * status (device int32[2]): [0] = 0 or -SW_ERR_SLOT_OUT_OF_RANGE. */
SW_API int sw_ragged_remove_row_slots(const sw_ragged_t* m, int32_t pre, const int32_t* slots,
                                      int32_t k, int32_t* status, void* stream);

/* Pairwise-Bernoulli initialisation (init_pairwise_bernoulli, connectivity.py:212-245):
 * pair (i, j) uses uniform01 draw #(counter0 + i*num_post + j) of `key` and
 * connects iff u < p.  mode 0: p = density; mode 1: density with p(i,i) = 0;
 * mode 2: p = lut[((xj-xi) mod side) + side*((yj-yi) mod side)] on a
 * side x side torus (topomap.py:376-388).  Count pass then fill pass
 * (capacity is chosen on the host from *max_len, as the reference does). */
SW_API int sw_init_bernoulli_count(int64_t num_pre, int32_t num_post, uint64_t key,
                                   uint64_t counter0, int32_t mode, double density,
                                   const double* lut, int32_t side, int32_t* row_length,
                                   int32_t* max_len, void* stream);
SW_API int sw_init_bernoulli_fill(int64_t num_pre, int32_t num_post, uint64_t key,
                                  uint64_t counter0, int32_t mode, double density,
                                  const double* lut, int32_t side, int32_t* row_length,
                                  int32_t* target, int32_t stride, void* stream);

/* ---- DEEP R (deep_r.py:23-177) ------------------------------------------ */
/* DeepR.init_bitfields (deep_r.py:50-64). */
SW_API int sw_deepr_init_bitfields(const sw_ragged_t* m, int32_t weight_plane,
                            const sw_bitfield_t* sign, const sw_bitfield_t* conn,
                            uint64_t sign_key, void* stream);
/* DeepR.l1_step (deep_r.py:68-77): grad += sign ? +l1 : -l1 on valid slots. */
SW_API int sw_deepr_l1(const sw_ragged_t* m, int32_t grad_plane, const sw_bitfield_t* sign,
                const uint32_t* sign_slot, double l1, void* stream);
/* Slot-aligned sign cache: sign_slot[num_pre, ceil(stride/32)] uint32, bit s
 * of row i = sign bit of (i, target[i, s]).  Derived state (invisible to
 * parity): eliminate / form / l1 keep it in step with every slot move and
 * placement so the eliminate scan reads 1 bit per synapse instead of
 * gathering 64-bit words from the num_post-wide sign row.  NULL = gather. */
SW_API int sw_deepr_sign_cache_build(const sw_ragged_t* m, const sw_bitfield_t* sign,
                                     uint32_t* sign_slot, void* stream);
/* Eliminate rule host+row phases (deep_r.py:81-99): removes sign-mismatched
 * synapses with the exact remove_slots order, clears their conn bits,
 * dormant[i] = count (int64).  With sign_slot and mark_scratch (same shape
 * as sign_slot, caller scratch) it runs as a streaming scan kernel plus a
 * removal kernel over the rows with removals; without mark_scratch, one
 * warp-per-row kernel does both. */
SW_API int sw_deepr_eliminate(const sw_ragged_t* m, int32_t weight_plane,
                       const sw_bitfield_t* sign, const sw_bitfield_t* conn,
                       int64_t* dormant, uint32_t* sign_slot, uint32_t* mark_scratch,
                       void* stream);
/* One pass of the form rule (deep_r.py:110-145).
 *   pending_src[num_pre] int64: dormant (pass 0) or unplaced of the previous
 *     pass; summed on device into counters[0] (= D, the number of host draws).
 *   host_key  = fold_key(seed,"host",rule_id,update,pass)   (updates.py:346-349)
 *   row_base  = fold_key(seed,"row", rule_id,update,pass)   (updates.py:313-314)
 *   activations[num_pre] int32 scratch, unplaced[num_pre] int64 out,
 *   counters[4] int64 device: [0]=D, [1]=sum(unplaced), [2]=rejected host draws,
 *   [3] reserved.  pending_src may alias unplaced (it is consumed first). */
SW_API int sw_deepr_form_pass(const sw_ragged_t* m, const sw_bitfield_t* conn,
                       int32_t exclude_diagonal, const int64_t* pending_src,
                       uint64_t host_key, uint64_t row_base,
                       int32_t* activations, int64_t* unplaced,
                       int64_t* counters, const sw_bitfield_t* sign, uint32_t* sign_slot,
                       void* stream);

/* Row-sharded form pass (SURVEY 8e M-update; replaces the single-process
 * _form_host / _form_row phases of deep_r.py:110-145 when rows are split
 * over ranks).  Each rank owns rows [row0, row0 + m->num_pre) of a
 * num_pre_global-row matrix.  Order per pass, with the host collectives
 * between (integer sums, so the result is bit-exact with sw_deepr_form_pass):
 *   sw_deepr_form_pending     counters[0..3] = 0; counters[0] = local sum of
 *                             pending_src                 -> all-reduce counters[0]
 *   sw_deepr_form_hist_chunk  act_full[num_pre_global] = histogram of host
 *                             draws [D*rank/world, D*(rank+1)/world); rejected
 *                             draws into counters[2]      -> all-reduce counters[2]
 *   sw_deepr_form_hist_fix    (one rank only) the draws that replace the
 *                             rejected ones, from counter D -> reduce-scatter
 *                             act_full by row owner into activations[num_pre]
 *   sw_deepr_form_rows_shard  placement of the local rows with the global
 *                             row's stream key child(row_base, row0 + i); the
 *                             local unplaced sum into counters[1]
 *                                                         -> all-reduce counters[1] */
SW_API int sw_deepr_form_pending(const int64_t* pending_src, int64_t num_rows, int64_t* counters,
                                 void* stream);
SW_API int sw_deepr_form_hist_chunk(int64_t* counters, uint64_t host_key, int64_t num_pre_global,
                                    int32_t rank, int32_t world, int32_t* act_full, void* stream);
SW_API int sw_deepr_form_hist_fix(int64_t* counters, uint64_t host_key, int64_t num_pre_global,
                                  int32_t* act_full, void* stream);
SW_API int sw_deepr_form_rows_shard(const sw_ragged_t* m, const sw_bitfield_t* conn,
                                    int32_t exclude_diagonal, uint64_t row_base, int64_t row0,
                                    const int32_t* activations, int64_t* unplaced, int64_t* counters,
                                    const sw_bitfield_t* sign, uint32_t* sign_slot, void* stream);

/* Microbenchmark sign-flip injection: valid slot (i, s) negates plane value
 * when uniform01 draw #(i*stride + s) of key < prob (SURVEY 8(d) M-update). */
SW_API int sw_flip_signs(const sw_ragged_t* m, int32_t plane, uint64_t key, double prob, void* stream);

/* ---- Adam (plasticity.py:198-227) ---------------------------------------- */
/* p -= lr*(m/c1)/(sqrt(v/c2)+eps) after the moment updates; g := 0.
 * All float64, n elements, exact reference op order. */
SW_API int sw_adam_f64(double* p, double* g, double* m, double* v, int64_t n,
                double b1, double one_minus_b1, double b2, double one_minus_b2,
                double c1, double c2, double lr, double eps, void* stream);

/* ---- e-prop (_kernels.py:15-39) ------------------------------------------- */
/* Drop-in for eprop_accumulate_batch: reference layout eps/ebar [B,P,S] f32,
 * grad [P,S] f64, pre_trace [B,P], psi/lsig [B,num_post]; thread per
 * synapse, replicas ascending, float32 ops separately rounded (bit-exact). */
SW_API int sw_eprop_accumulate_batch(const int32_t* targets, const int32_t* row_length,
                                     int32_t num_pre, int32_t stride, const float* pre_trace,
                                     const float* psi, const float* lsig, int32_t batch,
                                     int32_t num_post, float* eps, float* ebar, double* grad,
                                     float beta, float rho, float alpha, void* stream);
/* Per-batch compact synapse order for the fused step: synapses bucketed by
 * (target >> shift, pre, slot).  scratch: 2*n + ceil(n/4096) + 1 int32
 * with n = G*num_pre, G = ((num_post-1) >> shift) + 1.  out_* have e_pad entries (multiple of
 * 32); entries past *total are padding (out_off = -1). */
SW_API int sw_eprop_plan(const int32_t* row_length, const int32_t* target, int32_t num_pre,
                         int32_t stride, int32_t num_post, int32_t shift, int32_t* scratch,
                         int32_t* out_pre, int32_t* out_post, int32_t* out_off,
                         int32_t e_pad, int32_t* total, void* stream);
/* out[e] = plane[off[e]] (0 for off < 0) / plane[off[e]] = in[e] */
SW_API int sw_gather_f64(const double* plane, const int32_t* off, int32_t n, double* out, void* stream);
SW_API int sw_scatter_f64(double* plane, const int32_t* off, int32_t n, const double* in, void* stream);

/* One projection onto the hidden layer in compact plan order. */
typedef struct sw_eprop_seg {
  const int32_t* pre;       /* [e_pad] presynaptic index   */
  const int32_t* post;      /* [e_pad] postsynaptic index  */
  const float* pre_trace;   /* [B, num_pre] xbar or zbar   */
  float* eps;               /* [e_pad/32, B, 32] tile-major */
  float* ebar;              /* [e_pad/32, B, 32]            */
  double* grad;             /* [e_pad] compact gradient    */
  int32_t num_pre;
  int32_t e_pad;            /* multiple of 32              */
} sw_eprop_seg_t;

/* Fused hot-path step: both projections' eligibility recursion and
 * gradient accumulation (bit-identical to eprop_accumulate_batch on the
 * same synapses) plus, when d != NULL, the readout gradients
 * g_w_out[C,H] += d^T zbar and g_b_out[C] += sum_b d (classifier.py:221-222).
 * workspace: 2 uint32 zeroed once by the caller (tile tickets; the kernel
 * leaves them zeroed, so the launch can be captured in a CUDA graph).
 * max_blocks_per_sm: 0 = as many tile workers as fit; a smaller value leaves
 * room on every SM for a concurrently running kernel (the next timestep's
 * forward pass, see EpropClassifierTrainer). */
SW_API int sw_eprop_fused_step(const sw_eprop_seg_t* segs, int32_t n_segs, const float* psi,
                               const float* lsig, int32_t batch, int32_t hidden, float beta,
                               float rho, float alpha, const double* d, const float* zbar,
                               double* g_w_out, double* g_b_out, int32_t num_classes,
                               int32_t max_blocks_per_sm, uint32_t* workspace, void* stream);

#define SW_EPROP_MAX_BLOCK 16
/* k consecutive timesteps (1 <= k <= SW_EPROP_MAX_BLOCK) of the fused step in one pass over
 * the eligibility state (temporal blocking: the forward pass of the k steps
 * runs first, it never reads eps/ebar/grad).  Per step s < k: psi[s],
 * lsig[s] [B,H]; pre_trace[seg][s] [B, num_pre]; d[s] [B,C] and zbar[s]
 * [B,H] for the readout gradients (d[0] == NULL: no readout).  The segment's
 * own pre_trace field is ignored.  eps/ebar are bit-identical to k calls of
 * sw_eprop_fused_step; the gradient too for k = 1, and for k > 1 up to the
 * float64 rounding of adding k per-step partial sums (each in ascending
 * replica order). */
typedef struct sw_eprop_block {
  int32_t k;
  const float* psi[SW_EPROP_MAX_BLOCK];
  const float* lsig[SW_EPROP_MAX_BLOCK];
  const float* pre_trace[2][SW_EPROP_MAX_BLOCK];
  const double* d[SW_EPROP_MAX_BLOCK];
  const float* zbar[SW_EPROP_MAX_BLOCK];
  /* optional split readout: ro_scratch of sw_eprop_readout_scratch_bytes(
   * hidden, num_classes, ro_splits) bytes, ZEROED once by the caller (the
   * kernel leaves its counters zeroed again); NULL = one block per class and
   * 32 hidden units.  Both are deterministic. */
  double* ro_scratch;
  int32_t ro_splits;
} sw_eprop_block_t;
SW_API int64_t sw_eprop_readout_scratch_bytes(int32_t hidden, int32_t num_classes, int32_t splits);
SW_API int sw_eprop_fused_block(const sw_eprop_seg_t* segs, int32_t n_segs, const sw_eprop_block_t* blk,
                                int32_t batch, int32_t hidden, float beta, float rho, float alpha,
                                double* g_w_out, double* g_b_out, int32_t num_classes,
                                uint32_t* workspace, void* stream);

/* ---- replica-minor e-prop pass (the trainer's hot path) ----------------------
 * The forward pass writes its per-step vectors replica-major ([B, n]).
 * sw_eprop_prep makes replica-minor copies of a group of k steps --
 * xbar_t[k][num_inputs][ldb], zbar_t/psi_t[k][hidden][ldb] -- and the learning
 * signal lsig_t[k][hidden][ldb] = f32(sum_c d[b][c] * w_out[c][h]) (classes
 * ascending: classifier.py:223).  Columns b in [batch, ldb) are zero.
 * sw_eprop_pass runs k recursion steps of _kernels.py:15-39 over both
 * projections on those copies: eps/ebar in [e_pad/SPW][ldb/32][32][SPW]
 * order (SPW-synapse tile, 32-replica chunk, lane = (32/SPW)*synapse +
 * replica group, SPW replicas), ldb a multiple of 32, bit-identical to the
 * reference's; the float64 gradient terms are summed per synapse in
 * 64-replica splits and the splits added in order (within float64 rounding
 * of the reference's replica-ordered sum).  scratch:
 * sw_eprop_pass_scratch_bytes(total e_pad, ldb) bytes, zeroed once (the kernel
 * leaves its counters zero). */
typedef struct sw_eprop_prep {
  int32_t k, batch, ldb, num_inputs, hidden, num_classes;
  const float* xbar[SW_EPROP_MAX_BLOCK];   /* [batch, num_inputs] per step */
  const float* zbar[SW_EPROP_MAX_BLOCK];   /* [batch, hidden] */
  const float* psi[SW_EPROP_MAX_BLOCK];    /* [batch, hidden] */
  const double* d[SW_EPROP_MAX_BLOCK];     /* [batch, num_classes] */
  const double* w_out;                     /* [num_classes, hidden] */
  float* xbar_t; float* zbar_t; float* psi_t; float* lsig_t;
  /* optional readout gradients (classifier.py:221-222) over the group:
   * g_w_out[C, H] += sum d^T zbar, g_b_out[C] += sum d, through ro_partial
   * (sw_eprop_prep_scratch_bytes); g_w_out NULL = none */
  double* g_w_out; double* g_b_out; double* ro_partial;
  /* defer_reduce != 0: the readout partials accumulate in ro_partial over
   * the batch's groups (zeroed before the first, e.g. by the previous
   * sw_eprop_prep_reduce) and sw_eprop_prep_reduce adds them once */
  int32_t defer_reduce;
  /* psl_t != NULL: psi and lsig are written interleaved instead of to
   * psi_t / lsig_t: psl_t[k][h][ldb/4][8] holds, per group of 4 replicas,
   * their 4 psi then their 4 lsig values (the pass reads both with one
   * 32-byte load; sw_eprop_tpass_t.psl) */
  float* psl_t;
} sw_eprop_prep_t;
SW_API int sw_eprop_prep_reduce(const sw_eprop_prep_t* p, void* stream);
SW_API int64_t sw_eprop_prep_scratch_bytes(int32_t k, int32_t batch, int32_t hidden, int32_t num_classes);
SW_API int sw_eprop_prep(const sw_eprop_prep_t* p, void* stream);

typedef struct sw_eprop_tseg {
  const int32_t* pre;                        /* [e_pad] plan order */
  const int32_t* post;
  const float* trace_t[SW_EPROP_MAX_BLOCK];  /* [num_pre, ldb] per step */
  float* eps; float* ebar;                   /* [e_pad/SPW][ldb/32][32][SPW] */
  double* grad;                              /* [e_pad] compact gradient */
  int32_t e_pad;
} sw_eprop_tseg_t;
typedef struct sw_eprop_tpass {
  int32_t k;
  const float* psi_t[SW_EPROP_MAX_BLOCK];    /* [hidden, ldb] per step */
  const float* lsig_t[SW_EPROP_MAX_BLOCK];
  void* scratch;
  /* defer_reduce != 0: the split partials accumulate in scratch over the
   * batch's passes (zeroed before the first) and sw_eprop_pass_reduce adds
   * them to the gradients once (zeroing them again) */
  int32_t defer_reduce;
  /* state_zero != 0: eps and ebar start from zero (the first pass of a
   * batch): they are written, not read */
  int32_t state_zero;
  /* psl != 0: psi_t[k] is the interleaved psi/lsig array of
   * sw_eprop_prep_t.psl_t (step k), lsig_t ignored */
  int32_t psl;
} sw_eprop_tpass_t;
SW_API int sw_eprop_pass_reduce(const sw_eprop_tseg_t* segs, int32_t n_segs, int32_t ldb, void* scratch,
                                void* stream);
/* synapses per warp tile of sw_eprop_pass (SPW): eps/ebar are laid out
 * [e_pad/SPW][ldb/32][32 lanes][SPW replicas], lane = (32/SPW)*synapse + group */
#ifndef SW_EPROP_PASS_SPW
#define SW_EPROP_PASS_SPW 4
#endif
SW_API int32_t sw_eprop_pass_synapses_per_warp(void);
SW_API int64_t sw_eprop_pass_scratch_bytes(int32_t e_pad_total, int32_t ldb);
SW_API int sw_eprop_pass(const sw_eprop_tseg_t* segs, int32_t n_segs, const sw_eprop_tpass_t* p,
                           int32_t ldb, float beta, float rho, float alpha, void* stream);

/* ---- neurons (neurons.py) --------------------------------------------------- */
/* AlifLayer.step (neurons.py:60-67), float32, n = batch*hidden elements. */
SW_API int sw_alif_step(float* v, float* a, float* z, const float* rec, const float* ext,
                        int64_t n, float alpha, float rho, float beta, float v_thr, void* stream);
/* AlifLayer.surrogate (neurons.py:69-73). */
SW_API int sw_alif_surrogate(const float* v, const float* a, float* psi, int64_t n, float beta,
                             float v_thr, void* stream);
/* LifCondLayer.step (neurons.py:137-148); spike_bits[ceil(n/32)] (LSB = lowest id). */
SW_API int sw_lif_cond_step(double* V, double* g, int64_t* ref_until, const double* incoming,
                            int32_t n, int64_t step_index, double decay_s, double g_leak,
                            double v_rest, double e_exc, double v_theta, double v_reset,
                            double h, double tau_m, int64_t ref_steps, uint32_t* spike_bits,
                            void* stream);
/* PoissonSource.poisson_step (neurons.py:189-195): u = uniform01 #(counter0 + node) < p. */
SW_API int sw_poisson_step(uint64_t key, int64_t counter0, const double* p, int32_t n,
                           uint32_t* spike_bits, void* stream);

/* Correlated Poisson rates and per-step probabilities on the device
 * (neurons.py:175-193); centers[2*n_centers] (x, y) device array.  CUDA
 * exp/hypot (a few ulp from numpy): an option for large grids. */
SW_API int sw_poisson_rates(int32_t side, const double* centers, int32_t n_centers, double f_base,
                            double f_peak, double sigma, double h, double* rates, double* p,
                            void* stream);

/* ---- classifier timestep (classifier.py:188-234) ----------------------------- */
typedef struct sw_clf_step {
  const int32_t* in_row_length;  const int32_t* in_target;  const float* in_w32;
  int32_t in_stride;  int32_t num_inputs;
  const int32_t* rec_row_length; const int32_t* rec_target; const float* rec_w32;
  int32_t rec_stride; int32_t hidden;
  const double* w_out; const double* b_out; int32_t num_classes;
  const double* p_in;      /* [B, num_inputs] per-example spike probability  */
  const uint64_t* ex_key;  /* [B] fold_key(seed,"task","example",e)          */
  const int32_t* labels;   /* [B]                                            */
  int32_t t;               /* timestep                                       */
  int32_t batch;
  float* v; float* a; float* z; float* zbar; float* xbar;     /* [B,H] / [B,NI] */
  double* y; double* pi_sum; double* loss; double* d;         /* [B,C] / [B]    */
  float* psi; float* lsig;                                    /* [B,H]          */
  float alpha; float rho; float beta; float v_thr; double alpha64;
  /* previous-step traces (NULL = update xbar/zbar in place): with separate
   * in/out trace buffers the next step's forward pass can run while the
   * e-prop update still reads this step's traces */
  const float* zbar_in; const float* xbar_in;
  /* n_steps >= 1: one launch runs timesteps t .. t+n_steps-1 (block per
   * replica, steps back to back).  zbar/xbar/psi/lsig/d are then the bases of
   * slot_count contiguous per-step slots [slot][batch][width]; step t writes
   * slot t % slot_count and reads the traces of slot (t-1) % slot_count
   * (zbar_in/xbar_in ignored).  n_steps = 0: one step, fields as above. */
  int32_t n_steps; int32_t slot_count;
  /* packed (target, f32 weight) rows, [num_pre][tw_stride] int32 pairs with
   * an even tw_stride (sw_clf_pack_rows): read entry by entry by the
   * grouped forward (in_bits), staged with one bulk copy per spiking row by
   * the single-step register-resident forward.  NULL: k_clf_step. */
  const int32_t* in_tw; const int32_t* rec_tw;
  int32_t in_tw_stride; int32_t rec_tw_stride;
  /* precomputed input spikes (sw_clf_inputs), grouped launches only:
   * in_bits[t][batch][in_words]; NULL = the kernel draws them itself */
  const uint32_t* in_bits; int32_t in_words;
  /* with in_bits: [n_steps][batch][ceil(hidden/32)] scratch for the hidden
   * spike words of the launch's steps; the readout / softmax of those steps
   * then runs as a second launch (k_clf_readout) over all of them at once */
  uint32_t* z_bits;
} sw_clf_step_t;
/* The trial's input side at once (classifier.py:63-67, 210-213): every input
 * spike of steps 0..steps-1 from the examples' counter streams, as words
 * in_bits[t][batch][words] (words = ceil(num_inputs/32)), and the input
 * traces xbar_t[t][num_inputs][ldb] (replica-minor, zero past the batch).
 * num_inputs <= 25600. */
typedef struct sw_clf_inputs {
  int32_t steps, batch, ldb, num_inputs, words;
  const double* p_in;        /* [batch, num_inputs] */
  const uint64_t* ex_key;    /* [batch] */
  float alpha;
  float* xbar_t;
  uint32_t* in_bits;
} sw_clf_inputs_t;
SW_API int sw_clf_inputs(const sw_clf_inputs_t* p, void* stream);
/* tw[i][s] = (target[i][s], f32(w[i][s])) for s < row_length[i], (0, 0)
 * after; tw_stride >= stride, even. */
SW_API int sw_clf_pack_rows(const int32_t* row_length, const int32_t* target, const double* w,
                            int32_t num_pre, int32_t stride, int32_t tw_stride, int32_t* tw, void* stream);
/* Fused forward timestep(s) for all replicas (block per replica). */
SW_API int sw_clf_step(const sw_clf_step_t* params, void* stream);
/* out2[0] = sum of per-replica cross-entropy, out2[1] = #correct (argmax pi_sum). */
SW_API int sw_clf_batch_stats(const double* loss, const double* pi_sum, const int32_t* labels,
                              int32_t batch, int32_t num_classes, double* out2, void* stream);
SW_API int sw_f64_to_f32(const double* in, float* out, int64_t n, void* stream);
/* zero n <= 16 device ranges (bytes[i] bytes at ptrs[i]) in one launch: the
 * per-batch state resets of the trainer */
#define SW_ZERO_MAX_RANGES 16
SW_API int sw_zero_ranges(void* const* ptrs, const int64_t* bytes, int32_t n, void* stream);
SW_API int sw_scale_f64(double* x, int64_t n, double s, void* stream);

/* ---- transpose (connectivity.py:151-203) ----------------------------------- */
/* TransposeMap.rebuild in CSR form with slack: for post j, (pre, slot) of
 * its incoming synapses in [col_ptr[j], col_ptr[j] + col_length[j]) ordered
 * by (pre, slot) (the reference's lexsort order); column j has room for
 * col_ptr[j+1] - col_ptr[j] = col_length[j] + slack entries (slack >= 0;
 * room for sw_transpose_patch).  col_length[N], col_ptr[N+1],
 * src_pre/src_slot[>= edges + N*slack], cursor[N] scratch, *max_len =
 * widest column.  changed: device flag (NULL = always); when it reads 0
 * nothing is rebuilt (remap-only-if-changed, updates.py:367-369). */
SW_API int sw_transpose_rebuild(const sw_ragged_t* m, int32_t* col_length, int32_t* col_ptr,
                                int32_t* src_pre, int32_t* src_slot, int32_t* cursor,
                                int32_t* max_len, const int32_t* changed, int32_t slack, void* stream);
/* The same rebuild as one cooperative launch (grid barriers between the
 * count / scan / scatter / sort phases; a single launch that exits at once
 * when *changed reads 0).  block_scratch: >= 2048 int32 (device). */
SW_API int sw_transpose_rebuild_coop(const sw_ragged_t* m, int32_t* col_length, int32_t* col_ptr,
                                     int32_t* src_pre, int32_t* src_slot, int32_t* cursor,
                                     int32_t* max_len, const int32_t* changed,
                                     int32_t* block_scratch, int32_t slack, void* stream);
/* sw_transpose_rebuild_coop gated by a flag the call also resets
 * (clear_changed != 0): the patch path's "overflowed, rebuild" flag. */
SW_API int sw_transpose_rebuild_gated(const sw_ragged_t* m, int32_t* col_length, int32_t* col_ptr,
                                      int32_t* src_pre, int32_t* src_slot, int32_t* cursor,
                                      int32_t* max_len, int32_t* changed, int32_t* block_scratch,
                                      int32_t slack, int32_t clear_changed, void* stream);
/* Incremental remap (connectivity.py:173-192 applied to one update's
 * changes instead of the whole matrix).  patch_log (device int32, written by
 * the mutating kernel, e.g. sw_rewire_update with prm->patch_log):
 *   [0] = rows whose structure changed, [1] = removed (pre, post) pairs,
 *   [2] = overflow flag, [3] reserved, then cap row ids, then cap pairs.
 * For every column touched by those rows (their current targets and their
 * removed targets) the entries of the changed rows are dropped and the rows'
 * current synapses merged back in (pre, slot) order, in place.  A column
 * that outgrows its slack, or a log that overflowed, sets *rebuild = 1 (the
 * caller's gated sw_transpose_rebuild_coop then rebuilds everything; the
 * result is identical either way).  The log counters are reset for the next
 * update.  scratch: sw_transpose_patch_scratch_bytes(num_pre, num_post). */
SW_API int64_t sw_transpose_patch_scratch_bytes(int32_t num_pre, int32_t num_post);
SW_API int sw_transpose_patch(const sw_ragged_t* m, int32_t* col_length, const int32_t* col_ptr,
                              int32_t* src_pre, int32_t* src_slot, int32_t* patch_log, int32_t cap,
                              int32_t* rebuild, void* scratch, void* stream);

/* ---- spike propagation (connectivity.py:139-148) ---------------------------- */
/* Event-driven atomic mode: out[target] += w over the rows in
 * spikes[*n_spikes] (device count; max_spikes bounds the grid).
 * Few spiking rows: warp per row, float64 RED into L2.  Many rows,
 * num_post <= 65536 and a workspace of >= sw_propagate_workspace_bytes():
 * one CTA per SM accumulates one 16384-post slab in shared memory over its
 * group's rows, then the per-group slabs are reduced (ascending group order)
 * into out after a grid barrier.  Summation order across rows is not
 * deterministic in either form (shared-memory / L2 atomics). */
SW_API int sw_propagate_atomic(const int32_t* row_length, const int32_t* target, const double* w,
                               int32_t num_pre, int32_t num_post, int32_t stride,
                               const int32_t* spikes, const int32_t* n_spikes, int32_t max_spikes,
                               double* out, void* workspace, int64_t workspace_bytes,
                               void* stream);
/* Workspace bytes the slab form of sw_propagate_atomic needs on the current device. */
SW_API int64_t sw_propagate_workspace_bytes(void);

/* Post-slab bucketed rows (a derived copy for propagate_spikes over a matrix
 * whose connectivity and weights stay fixed across many steps; SURVEY §8e
 * "column slices of every row").  G = sw_prop_bucket_slabs(num_post) slabs of
 * 16384 posts (num_post <= 131072).  Arrays, caller-allocated:
 *   bt, bslot uint16 [num_pre*stride], bw float64 [num_pre*stride],
 *   soff uint16 [num_pre*(G+1)].
 * Row i's synapses, grouped by slab and in slot order within a slab, sit in
 * the row's own padded slot range; soff[i*(G+1)+j] is slab j's first entry.
 * Rebuild after a structural change (like TransposeMap, connectivity.py:173);
 * after a weight-only change sw_prop_buckets_refresh re-gathers bw. */
SW_API int32_t sw_prop_bucket_slabs(int32_t num_post);
SW_API int sw_prop_buckets_build(const int32_t* row_length, const int32_t* target, const double* w,
                                 int32_t num_pre, int32_t num_post, int32_t stride, uint16_t* bt,
                                 uint16_t* bslot, double* bw, uint16_t* soff, void* stream);
SW_API int sw_prop_buckets_refresh(const int32_t* row_length, const double* w, int32_t num_pre,
                                   int32_t stride, const uint16_t* bslot, double* bw, void* stream);
/* propagate_spikes (connectivity.py:139-148), atomic-mode semantics (float64,
 * summation order not fixed: shared-memory atomics per slab, then the groups'
 * partial slabs summed in ascending group order): out[j] += sum over the
 * spiking rows.  One cooperative launch; workspace >=
 * sw_prop_bucketed_workspace_bytes(num_post). */
SW_API int64_t sw_prop_bucketed_workspace_bytes(int32_t num_post);
SW_API int sw_propagate_bucketed(const uint16_t* soff, const uint16_t* bt, const double* bw, int32_t num_post,
                                 int32_t stride, const int32_t* spikes, const int32_t* n_spikes,
                                 int32_t max_spikes, double* out, void* workspace, int64_t workspace_bytes,
                                 void* stream);
/* Same contract over the same bucketed copy (its weight snapshot), one warp
 * per spiking row with float64 L2 atomics: for few spiking rows, where the
 * slab pass's fixed cost dominates. */
SW_API int sw_propagate_bucketed_atomic(const uint16_t* soff, const uint16_t* bt, const double* bw,
                                        int32_t num_post, int32_t stride, const int32_t* spikes,
                                        const int32_t* n_spikes, int32_t max_spikes, double* out,
                                        void* stream);
typedef struct sw_prop_proj {
  const int32_t* col_ptr;    /* transpose CSR of the projection (column j: col_ptr[j], col_length[j]) */
  const int32_t* col_length;
  const int32_t* src_pre;
  const int32_t* src_slot;
  const double* weights;     /* [num_pre, stride] */
  const uint32_t* spike_bits;/* presynaptic spikes, bit i of word i/32 */
  int32_t stride;
} sw_prop_proj_t;
/* Bit-exact with np.add.at in ascending spike order: out[j] = (accumulate ?
 * out[j] : 0) + contributions of projection 0 (ascending pre) then 1. */
SW_API int sw_propagate_ordered(const sw_prop_proj_t* projs, int32_t n_proj, int32_t num_post,
                                double* out, int32_t accumulate, void* stream);
/* Ascending id list of the set bits (single block). */
SW_API int sw_spike_bits_to_list(const uint32_t* bits, int32_t n, int32_t* list, int32_t* count,
                                 void* stream);

/* ---- trace STDP (plasticity.py:42-95) --------------------------------------- */
SW_API int sw_stdp_decay(double* x, int32_t nx, double dx, double* y, int32_t ny, double dy,
                         void* stream);
/* on_pre_spikes: w = clip(w - a_minus*y[post]) on spiking rows, then x[pre] += 1 */
SW_API int sw_stdp_pre(const int32_t* row_length, const int32_t* target, double* w, int32_t stride,
                       int32_t num_pre, const uint32_t* pre_bits, const double* y, double* x,
                       double a_minus, double w_min, double w_max, void* stream);
/* on_post_spikes through the transpose: w = clip(w + a_plus*x[pre]), then y[post] += 1 */
SW_API int sw_stdp_post(const int32_t* col_ptr, const int32_t* col_length, const int32_t* src_pre, const int32_t* src_slot,
                        double* w, int32_t stride, int32_t num_post, const uint32_t* post_bits,
                        const double* x, double* y, double a_plus, double w_min, double w_max,
                        void* stream);

/* ---- topographic-map rewiring (topomap.py:70-223) --------------------------- */
typedef struct sw_rewire_params {
  uint64_t host_prefix;      /* fold_key(seed, "host") */
  uint64_t row_prefix;       /* fold_key(seed, "row")  */
  int32_t rule_id;
  int32_t side;              /* torus side length (num_post = side*side) */
  int64_t total_attempts;    /* n_attempts * scale^2 (topomap.py:360) */
  const double* form_lut;    /* [num_post] formation probability by torus offset */
  const double* dist_lut;    /* [num_post] toroidal distance by torus offset */
  double g_theta, p_dep, p_pot, g_init;
  void* scratch;             /* sw_rewire_scratch_bytes(num_post, total_attempts) bytes for rows with
                                more than 64 attempts (processed serially, exact); NULL: such rows
                                count as errors (totals[7]) */
  int32_t* patch_log;        /* optional sw_transpose_patch log (rows changed, removed pairs) */
  int32_t patch_cap;
} sw_rewire_params_t;
SW_API int64_t sw_rewire_scratch_bytes(int32_t num_post, int64_t total_attempts);
/* One RewiringRule update (host + row phases), no host round trip.
 * attempts[num_pre] int32 (input when forced_attempts != 0), update_count
 * (device int64, read then incremented), keys[2] scratch, totals[16] int64
 * out ([0] removed [1] kept [2] formed [3] form_missed [4] form_full
 * [5] attempts [7] error count (a row with more attempts than num_post);
 * [8], [9] internal), changed (device flag for the remap),
 * rej scratch int64; ev_off/ev_kind/ev_d (may be NULL): per-attempt event
 * records in row order (kind 1 = elimination, 2 = formation, distance). */
SW_API int sw_rewire_update(const sw_ragged_t* m, int32_t weight_plane, const sw_rewire_params_t* prm,
                            int32_t* attempts, int64_t* update_count, uint64_t* keys,
                            int64_t* totals, int32_t* changed, int64_t* rej, int32_t* ev_off,
                            int8_t* ev_kind, double* ev_d, int32_t forced_attempts, void* stream);

/* Per-update structural-change log of the two projections (RunRecord
 * rewires_per_update; topomap.py:457-458 collect()):
 * log[u] = {removed_a, formed_a, removed_b, formed_b}, u = *update_count - 1
 * clamped to [0, cap). */
SW_API int sw_topomap_log(const int64_t* update_count, const int64_t* totals_a,
                          const int64_t* totals_b, int64_t* log, int64_t cap, void* stream);

/* ---- topographic-map step (topomap.py:419-452) ------------------------------ */
typedef struct sw_topomap_step {
  int32_t n;                      /* nodes per sheet (num_pre = num_post) */
  int64_t* step;                  /* device step index, incremented per step */
  uint64_t poisson_key;           /* fold_key(seed, "poisson"); counter = step*n + node */
  const double* p_src;            /* [n] 1 - exp(-rate*h*1e-3) (host numpy) */
  uint32_t* src_bits;             /* [ceil(n/32)] source spikes of this step */
  uint32_t* tgt_bits;             /* [ceil(n/32)] target spikes of this step */
  double* V; double* g_tot; int64_t* ref_until; double* pending;
  double decay_s, g_leak, v_rest, e_exc, v_theta, v_reset, h, tau_m;
  int64_t ref_steps;
  const int32_t* ff_row_length; const int32_t* ff_target; double* ff_g; int32_t ff_stride;
  const int32_t* ff_col_ptr; const int32_t* ff_col_len; const int32_t* ff_src_pre; const int32_t* ff_src_slot;
  const int32_t* lat_row_length; const int32_t* lat_target; double* lat_g; int32_t lat_stride;
  const int32_t* lat_col_ptr; const int32_t* lat_col_len; const int32_t* lat_src_pre; const int32_t* lat_src_slot;
  double* ff_x; double* ff_y; double* lat_x; double* lat_y;
  double decay_x, decay_y, a_plus, a_minus, w_min, w_max;
  /* postsynaptic shard [post_lo, post_hi) of this rank (0, n when unsharded):
   * the LIF update and the propagation into `pending` cover these posts only;
   * bounds on 32-post spike-word boundaries.  Source spikes, trace decays,
   * STDP and the step counter cover the whole sheet. */
  int32_t post_lo, post_hi;
} sw_topomap_step_t;
/* neurons -> ordered propagation + trace decay -> STDP pre -> STDP post ->
 * step += 1; spike_counts[2] (device, may be NULL) accumulate spikes. */
SW_API int sw_topomap_step(const sw_topomap_step_t* s, int64_t* spike_counts, void* stream);
/* The same step split around the target-spike exchange of the sharded
 * model (topomap.py:426-450 with postsynaptic sharding):
 * sw_topomap_neurons = Poisson sources (all nodes) + LIF (owned posts),
 * writing src_bits fully and tgt_bits for the owned words; the caller then
 * all-gathers tgt_bits; sw_topomap_synapses = the rest of the step. */
SW_API int sw_topomap_neurons(const sw_topomap_step_t* s, void* stream);
/* n_steps whole steps (unsharded sheet) in one persistent cooperative launch:
 * the phases of a step are separated by grid-wide barriers instead of kernel
 * boundaries.  barrier_words: 2 zeroed uint32 (device), left consistent for
 * the next launch.  Same results as n_steps calls of sw_topomap_step. */
SW_API int sw_topomap_run_steps(const sw_topomap_step_t* s, int32_t n_steps, int64_t* spike_counts,
                                uint32_t* barrier_words, void* stream);
SW_API int sw_topomap_synapses(const sw_topomap_step_t* s, int64_t* spike_counts, void* stream);
/* n_steps whole steps (unsharded sheet) as 2 launches per step: the
 * propagation of step t, then step t's STDP pre and post phases together
 * with step t+1's neuron phase (trace increments deferred to the next
 * propagation; synapses whose pre and post both spiked updated once, in
 * order, by the pre phase); the spike words alternate between s->src_bits /
 * s->tgt_bits and src_bits_alt / tgt_bits_alt (same sizes) and the last
 * step's words end in s's buffers.  Same results as n_steps calls of
 * sw_topomap_step. */
SW_API int sw_topomap_steps_fused(const sw_topomap_step_t* s, uint32_t* src_bits_alt, uint32_t* tgt_bits_alt,
                                  int32_t n_steps, int64_t* spike_counts, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SPARSEWIRE_B200_H */
