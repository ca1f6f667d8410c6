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
                double l1, void* stream);
/* Eliminate rule host+row phases (deep_r.py:81-99): warp per row; removes
 * sign-mismatched synapses with the exact remove_slots order, clears their
 * conn bits, dormant[i] = count (int64). */
SW_API int sw_deepr_eliminate(const sw_ragged_t* m, int32_t weight_plane,
                       const sw_bitfield_t* sign, const sw_bitfield_t* conn,
                       int64_t* dormant, void* stream);
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
                       int64_t* counters, void* stream);

/* ---- Adam (plasticity.py:198-227) ---------------------------------------- */
/* p -= lr*(m/c1)/(sqrt(v/c2)+eps) after the moment updates; g := 0.
 * All float64, n elements, exact reference op order. */
SW_API int sw_adam_f64(double* p, double* g, double* m, double* v, int64_t n,
                double b1, double one_minus_b1, double b2, double one_minus_b2,
                double c1, double c2, double lr, double eps, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SPARSEWIRE_B200_H */
