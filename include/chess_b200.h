/*
 * chess_b200.h — C-ABI of the B200-native CHESS decode hot path.
 *
 * The reference (`pagesel`, /root/reference/pkg/src/pagesel) is pure Python +
 * NumPy and has no FFI; its drop-in surface is the public Python API listed in
 * pagesel/__init__.py:43-86.  Every entry point below replaces one function
 * group of that API (cited per function) and is what a ctypes binding in the
 * reference package would call.
 *
 * Conventions
 *  - Plain C: device pointers are `void*`/typed pointers, sizes are int32/int64,
 *    streams are `void*` (a cudaStream_t).  No torch types.
 *  - The caller owns every device buffer (allocated by torch in the Python
 *    host layer).  Kernels never allocate; scratch comes from the
 *    `workspace` pointer sized by chess_workspace_bytes().
 *  - Entry points validate host-side and launch asynchronously; they never
 *    synchronise the stream.  Status codes map 1:1 to pagesel exceptions
 *    (SURVEY.md §8b "Errors").
 *  - Numerics: per-sequence state vectors (page vectors, chunk/grid sums,
 *    running key sums, anchor) are float64 and follow the reference's f64
 *    operation order bit-for-bit; the large scanned summary matrices may be
 *    stored as float32 mirrors (summary_dtype 0) or scanned in float64
 *    (summary_dtype 1).  Scores are always accumulated in float64.
 */
#ifndef CHESS_B200_H
#define CHESS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CHESS_ABI_VERSION 5

/* Status codes.  Python shim maps them to the pagesel exception classes
 * (pagesel/errors.py:4-21 and the ValueError/IndexError sites listed). */
enum ChessStatus {
  CHESS_OK = 0,
  CHESS_ERR_CONFIG = 1,        /* ConfigurationError  (config.py:36-48, kv_store.py:111) */
  CHESS_ERR_OUT_OF_PAGES = 2,  /* OutOfPagesError     (kv_store.py:129-132)            */
  CHESS_ERR_EMPTY_CONTEXT = 3, /* EmptyContextError   (selection.py:55-56)             */
  CHESS_ERR_SHAPE = 4,         /* ValueError dim mismatch (selection.py:68-72)         */
  CHESS_ERR_INDEX = 5,         /* IndexError          (kv_store.py:161-164)            */
  CHESS_ERR_ORDER = 6,         /* ValueError unsealed/out-of-order (hierarchy.py:108-114) */
  CHESS_ERR_VALUE = 7,         /* ValueError bad distribution (uncertainty.py:25-29)   */
  CHESS_ERR_CUDA = 8,          /* CUDA launch/runtime error                            */
  CHESS_ERR_UNSUPPORTED = 9    /* shape with no compiled kernel instance               */
};

/* Element dtypes for function-level entry points. */
enum ChessDtype { CHESS_F32 = 0, CHESS_F64 = 1, CHESS_BF16 = 2 };

/* Trigger policies (simulate.py:78-91, 163-170).  EVERY_STEP is a bench-only
 * policy that forces selection on every decode token (worst case). */
enum ChessPolicy {
  CHESS_POLICY_NEVER = 0,
  CHESS_POLICY_ALWAYS = 1,
  CHESS_POLICY_FIXED = 2,
  CHESS_POLICY_DYNAMIC = 3,
  CHESS_POLICY_EVERY_STEP = 4
};

/* Working-set provenance tags (selection.py:126-140: sink > window > semantic). */
enum ChessProvenance { CHESS_PROV_NONE = 0, CHESS_PROV_SEMANTIC = 1, CHESS_PROV_WINDOW = 2, CHESS_PROV_SINK = 3 };

/* Shape of a batched decode state.  Mirrors SelectionConfig (config.py:16-52)
 * plus the model shape; D = layers*kv_heads*head_dim is the flattened key
 * dimension of the reference (kv_store.py:35). */
typedef struct ChessDims {
  int32_t batch;           /* sequence slots                                   */
  int32_t layers;          /* L                                                */
  int32_t kv_heads;        /* H_kv                                             */
  int32_t q_heads;         /* H_q (multiple of H_kv)                           */
  int32_t head_dim;        /* d                                                */
  int32_t page_size;       /* B   (config.py:27)                               */
  int32_t pages_per_chunk; /* N_c (config.py:28)                               */
  int32_t chunks_per_grid; /* N_g (config.py:29)                               */
  int32_t max_pages;       /* per-sequence page-table / index capacity         */
  int32_t window_pages;    /* W   (config.py:33)                               */
  int32_t max_ws;          /* block-table row capacity (>= max_pages)          */
  int32_t summary_dtype;   /* 0: scan float32 mirrors, 1: scan float64,
                            * 2: scan bf16 mirrors (held in the *_vec32 buffers) */
  int64_t dim;             /* D                                                */
  int64_t ld;              /* summary row stride in elements (>= D, % 4 == 0)  */
  int64_t n_phys;          /* physical pages in the KV pool                    */
} ChessDims;

/* Device-resident batched decode state.  Every pointer is a device pointer
 * owned by the caller.  Layouts ([..] = row-major):
 *   k_pool, v_pool : bf16 [layers][n_phys][kv_heads][page_size][head_dim]
 *   page_table     : i32  [batch][max_pages]          (kv_store.py:94-100)
 *   page_vec64     : f64  [batch][max_pages][ld]       (hierarchy.py:37, :115)
 *   chunk_sum64    : f64  [batch][max_chunks][ld]      (hierarchy.py:38)
 *   grid_sum64     : f64  [batch][max_grids][ld]       (hierarchy.py:40)
 *   chunk_vec64/grid_vec64 : f64 centroids sum/count   (hierarchy.py:78-92)
 *   *_vec32        : f32 mirrors of the three centroid matrices (scan copies)
 *   key_sum        : f64  [batch][ld]  running sum of the open page's keys
 *   anchor         : f64  [batch][ld]  Eq.3 anchor (selection.py:44-59)
 *   semantic       : i32  [batch][max_pages] sorted selected pages
 *   ws_logical/block_table/ws_prov : [batch][max_ws]
 *   ent_ring       : f64  [batch][page_size] per-token entropies of the open page
 * max_chunks = ceil(max_pages/N_c), max_grids = ceil(max_chunks/N_g). */
typedef struct ChessState {
  ChessDims d;
  void* k_pool;
  void* v_pool;
  int32_t* page_table;
  int32_t* num_pages;    /* [batch] page-table entries in use (incl. open tail) */
  int32_t* tail_fill;    /* [batch] rows written in the last page (0..B)        */
  int64_t* token_count;  /* [batch]                                             */
  int32_t* sink_count;   /* [batch] (kv_store.py:122-125)                       */
  uint8_t* sealed;       /* [batch] tail sealed by the last append              */
  int32_t* num_sealed;   /* [batch] pages folded into the index                 */
  double* page_vec64;
  double* chunk_sum64;
  double* grid_sum64;
  double* chunk_vec64;
  double* grid_vec64;
  float* page_vec32;
  float* chunk_vec32;
  float* grid_vec32;
  double* key_sum;
  double* anchor;
  int32_t* semantic;
  int32_t* n_semantic;
  int32_t* sel_stats;    /* [batch][8]: G, C, P, A_c, A_p, k_g, k_c, k_p of the last pass */
  int32_t* ws_logical;
  int32_t* block_table;
  int8_t* ws_prov;
  int32_t* ws_len;
  double* ent_ring;
  int32_t* ent_count;    /* [batch] entropies recorded for the open page         */
  int32_t* gen_pages;    /* [batch] generated pages completed                    */
  double* page_stats;    /* [batch][2] (mean_entropy, varentropy) of last page   */
  uint8_t* fire;         /* [batch] selection gate                               */
  uint32_t* trigger_count; /* [batch] sealed pages whose policy decision fired a
                          * reselection (backtracking events); may be NULL     */
  /* Optional device page pool: PagedKvStore's free list (kv_store.py:103-136)
   * on the device, so generation never returns to the host for a page.
   * pool_free == NULL: the caller fills page_table (host-managed).  A slot's
   * pool pages are the run page_table[s][pool_base[s] .. pool_end[s]). */
  int32_t* pool_free;    /* [n_phys] free physical page ids (a stack)            */
  int32_t* pool_top;     /* [1] ids on the stack                                 */
  int32_t* pool_base;    /* [batch] first page-table entry owned by the pool     */
  int32_t* pool_end;     /* [batch] one past the last entry holding a pool page  */
  uint8_t* pool_oom;     /* [batch] an allocation found the pool empty (sticky)  */
  void* workspace;
  size_t workspace_bytes;
} ChessState;

/* Selection knobs (config.py:27-34).  full_scan = 1 scores every row as in
 * Alg. 1 literally; 0 (default) scores only children of kept parents, which
 * is output-identical (masked top-k never keeps a child of a pruned parent). */
typedef struct ChessSelectCfg {
  double rho_grid;
  double rho_chunk;
  double rho_page;
  int32_t full_scan;
  int32_t force_all;     /* ignore fire[] and select for every slot */
  int32_t defer_ws;      /* 1: write the semantic sets but leave working sets and
                          * block tables untouched (marked pending) until
                          * chess_flush_working_sets, so the pass can run
                          * concurrently with sparse_decode reading them */
  int32_t pad_;
} ChessSelectCfg;

/* Trigger knobs (uncertainty.py:86-98, simulate.py:163-170). */
typedef struct ChessTriggerCfg {
  int32_t policy;        /* enum ChessPolicy */
  int32_t interval;      /* fixed(N) */
  int32_t mode;          /* 0 joint, 1 any */
  int32_t pad_;
  double tau_entropy;
  double tau_varentropy;
} ChessTriggerCfg;

/* ---- library / ABI ---------------------------------------------------- */
int chess_abi_version(void);
size_t chess_dims_sizeof(void);
size_t chess_state_sizeof(void);
/* Last error message of the calling thread (NUL-terminated, truncated). */
int chess_last_error(char* buf, size_t n);
/* Validates a shape (ConfigurationError on failure). */
int chess_validate_dims(const ChessDims* d);
/* Scratch needed by the batched entry points for this shape. */
size_t chess_workspace_bytes(const ChessDims* d);

/* ---- batched decode path (one stream; capturable in a CUDA graph) ------ */

/* Zero all per-slot counters/state of the slots with mask[s] != 0 (or all
 * slots if mask == NULL).  create_sequence (kv_store.py:122-125). */
int chess_reset_slots(const ChessState* st, const uint8_t* mask, void* stream);

/* Append one token's K/V row per active slot (kv_store.py:141-154).
 * k_rows/v_rows: bf16 [batch][row_stride] (one stride for both), flattened
 * (layer, kv_head, d).
 * Opens the pre-reserved page page_table[s][num_pages[s]] when the tail is
 * sealed (allocation is host-side, kv_store.py:127-136), accumulates the f64
 * running key sum, sets sealed[s], and rebuilds the block table when a page
 * was opened (working set depends on len(page_table), selection.py:131).
 * active == NULL appends to every slot. */
int chess_append_kv(const ChessState* st, const void* k_rows, const void* v_rows,
                    int64_t row_stride, const uint8_t* active, void* stream);

/* The same append (kv_store.py:141-154) one layer range at a time, for a
 * model that produces a layer's K/V only after the previous layer's
 * attention.  k_rows/v_rows: bf16 [batch][row_stride] (one stride for both)
 * holding the columns of layers [layer_begin, layer_end) only.  The call with layer_begin == 0 is the token's first: it
 * opens the page and publishes the counters / block table exactly as
 * chess_append_kv (so layer 0's decode already sees the token); calls with
 * layer_begin > 0 write the same row of the same page.  Every layer must be
 * appended once, in increasing order, before chess_summary_seal. */
int chess_append_kv_layers(const ChessState* st, int32_t layer_begin, int32_t layer_end, const void* k_rows,
                           const void* v_rows, int64_t row_stride, const uint8_t* active, void* stream);

/* K1: fold every just-sealed tail page (sealed[s]) into the index
 * (HierarchyIndex.finalize_page, hierarchy.py:102-136) from the running key
 * sum, refresh the Eq.3 anchor (selection.py:44-59) and clear sealed[s]. */
int chess_summary_seal(const ChessState* st, void* stream);

/* K1b: bulk-build the index of each slot from the first n_pages[s] pages of
 * its page table, reading the K pool (prefill path; equals finalize_page in
 * logical order, hierarchy.py:165-174).  n_pages is a device pointer. */
int chess_summary_build(const ChessState* st, const int32_t* n_pages, void* stream);

/* K1c: build slot `seq`'s index from given f64 page vectors
 * (HierarchyIndex.from_page_vectors, hierarchy.py:43-58). rows: device f64
 * [n][row_stride]. */
int chess_summary_from_vectors(const ChessState* st, int32_t seq, const double* rows,
                               int32_t n, int64_t row_stride, void* stream);

/* K1d: fold one page given its key rows (device, dtype, [n_rows][row_stride])
 * into slot `seq`'s index at logical index num_sealed[seq]: Eq.1 mean in the
 * reference's row order, then finalize_page's chunk/grid update
 * (hierarchy.py:102-136).  Used by the function-level HierarchyIndex API. */
int chess_summary_fold(const ChessState* st, int32_t seq, const void* rows, int32_t dtype,
                       int32_t n_rows, int64_t row_stride, void* stream);

/* ---- device page pool (kv_store.py:103-136: _allocate / OutOfPagesError) --
 * chess_pool_init: the stack := ids[0..n) (device ids, n <= n_phys).
 * chess_pool_reserve: slot s takes counts[s] pages (device i32 [batch]) into
 *   page_table[s][pool_end ..) — all or none; none sets pool_oom[s].  Call it
 *   with 1 at admission; afterwards chess_summary_seal reserves the next page
 *   of every slot whose tail sealed, and chess_append_kv refuses to open a
 *   page that was not reserved (pool_oom[s] = 1, the token is not written).
 *   The caller maps a set pool_oom[s] to OutOfPagesError.
 * chess_pool_release: slots with mask[s] (NULL: all) push their pool pages
 *   back and clear pool_base/pool_end/pool_oom; call before chess_reset_slots. */
int chess_pool_init(const ChessState* st, const int32_t* ids, int32_t n, void* stream);
int chess_pool_reserve(const ChessState* st, const int32_t* counts, void* stream);
int chess_pool_release(const ChessState* st, const uint8_t* mask, void* stream);

/* K2+K3: anchor scoring + masked top-k cascade + working set + block table
 * (compute_anchor/score_all/hierarchical_prune/reconstruct_working_set/
 * gather_pages, selection.py:44-140, kv_store.py:156-166) for every slot
 * with fire[s] != 0 (or all slots if cfg->force_all). */
int chess_select(const ChessState* st, const ChessSelectCfg* cfg, void* stream);

/* KV-head-sharded selection (score_all's GEMV is a sum over the
 * (layer, head) column slices, selection.py:62-74).  Rank r holds kv heads
 * [r*H/n, (r+1)*H/n) of every layer, so its state's summary rows give
 * PARTIAL Eq.4 scores.  One cascade level = partial -> caller's all-gather
 * (NCCL) of `partial` -> combine.  Levels 0, 1, 2 (grids, chunks of kept
 * grids, pages of kept chunks) for the conditional scan; level 3 alone for
 * cfg->full_scan.
 *   partial  : f64 [batch][ld_partial]  this rank's partial scores, in the
 *              level's candidate order (written for slots that fired)
 *   gathered : f64 [world][batch][ld_partial]  every rank's `partial`,
 *              rank-major; summed in rank order, so all ranks select
 *              identically
 * ld_partial >= the level's row capacity (max_grids, max_chunks, max_pages,
 * or their sum for level 3).  Combine at level 2 (or 3) writes the semantic
 * set, working set and block table exactly as chess_select. */
int chess_select_partial(const ChessState* st, const ChessSelectCfg* cfg, int32_t level,
                         double* partial, int64_t ld_partial, void* stream);
int chess_select_combine(const ChessState* st, const ChessSelectCfg* cfg, int32_t level,
                         const double* gathered, int32_t world, int64_t ld_partial, void* stream);

/* The same exchange over peer memory instead of a library all-gather: the
 * partial scan's tail stores its rows straight into every rank's receive
 * buffer (NVLink stores through peer-mapped pointers) and release-stores a
 * per-(slot, source) flag; pull waits for the flags (acquire, system scope),
 * adds the rows in rank order and finishes the level like
 * chess_select_combine.  No host round trip and no collective launch per
 * level; CUDA-graph capturable (generations live on the device).
 * Per level, on every rank:
 *   recv[p]  : DEVICE array of world pointers; recv[p] is rank p's receive
 *              buffer, f64 [2][world][batch][ld] (double-buffered by gen & 1)
 *   flags[p] : DEVICE array of world pointers; rank p's u32 [batch][world]
 *   my_recv, my_flags : this rank's own entries (recv[rank], flags[rank])
 *   gen      : this rank's u32 [batch] exchanges completed per slot
 *   err      : this rank's i32 [1], set to 1 by a pull wait > 10 s
 * recv/flags/gen/err zeroed before the first exchange; every rank calls
 * push(level) then pull(level) in the same level order.  chess_p2p_* give
 * IPC-shareable device memory for the buffers (cudaMalloc + IPC handles). */
typedef struct ChessPeerExchange {
  int32_t world, rank;
  int64_t ld;
  double* const* recv;
  uint32_t* const* flags;
  double* my_recv;
  uint32_t* my_flags;
  uint32_t* gen;
  int32_t* err;
} ChessPeerExchange;
int chess_select_push(const ChessState* st, const ChessSelectCfg* cfg, int32_t level,
                      const ChessPeerExchange* px, void* stream);
int chess_select_pull(const ChessState* st, const ChessSelectCfg* cfg, int32_t level,
                      const ChessPeerExchange* px, void* stream);
/* Per-layer output gather of the KV-head shard over peer memory: K4 stores
 * every output row of this rank's query heads into its own `out` block and
 * into its block of EVERY other rank's output region (NVLink stores from the
 * epilogue), so no all-gather follows the layer; chess_gather_finish ends the
 * step: a two-phase barrier on per-source flags (system scope: "written",
 * then "copied out") around the copy of the peers' blocks of this rank's
 * region into `out`, so no rank's next step overwrites a region before every
 * rank copied it.
 *   regions[p] : HOST array of world pointers (this process's mappings);
 *                rank p's region, bf16 [layers][world][batch][q_heads*head_dim],
 *                16-byte aligned
 *   flags[p]   : DEVICE array of world pointers; rank p's u32 [world]
 *   my_flags   : this rank's flags (flags[rank])
 *   gen        : this rank's u32 [2] {steps finished, CTA counter}, zeroed
 *   err        : this rank's i32 [1], set by a wait > 10 s
 * Every rank runs chess_sparse_decode_gather for each layer (out = its
 * [layer][rank] block of the step's output, out_stride = q_heads*head_dim)
 * and then chess_gather_finish once per step with the whole output, bf16
 * [layers][world][batch][q_heads*head_dim]. */
typedef struct ChessPeerOutputs {
  int32_t world, rank;
  void* const* regions;
  uint32_t* const* flags;
  uint32_t* my_flags;
  uint32_t* gen;
  int32_t* err;
} ChessPeerOutputs;
int chess_sparse_decode_gather(const ChessState* st, int32_t layer, const void* q, int64_t q_stride,
                               void* out, int64_t out_stride, float* lse, float softmax_scale,
                               uint32_t flags, const ChessPeerOutputs* po, void* stream);
int chess_gather_finish(const ChessState* st, const ChessPeerOutputs* po, void* out, void* stream);
#define CHESS_IPC_HANDLE_BYTES 64
int chess_p2p_alloc(int64_t bytes, void** ptr);           /* zeroed device memory */
int chess_p2p_free(void* ptr);
int chess_p2p_export(void* ptr, uint8_t* handle);         /* handle: CHESS_IPC_HANDLE_BYTES */
int chess_p2p_open(const uint8_t* handle, void** ptr);    /* peer's allocation in this process */
int chess_p2p_close(void* ptr);

/* K3 epilogue alone: rebuild working set + block table from the cached
 * semantic set for all slots (selection.py:126-140). */
int chess_build_working_set(const ChessState* st, void* stream);

/* ... for the slots a defer_ws selection pass marked pending only. */
int chess_flush_working_sets(const ChessState* st, void* stream);

/* K4: sparse paged decode attention for one layer over the block table.
 * q: bf16 [batch][q_heads][head_dim] with batch stride q_stride (elements);
 * out: bf16 [batch][q_heads][head_dim] (out_stride); lse: f32 [batch][q_heads]
 * natural-log LSE (may be NULL).  Not in the reference (simulate.py:186 only
 * counts attention ops); oracle restated in oracle/attention.py. */
int chess_sparse_decode(const ChessState* st, int32_t layer, const void* q, int64_t q_stride,
                        void* out, int64_t out_stride, float* lse, float softmax_scale,
                        void* stream);

/* Launch-ordering flags of chess_sparse_decode_ex / _gather.  K4 is launched
 * with programmatic dependent launch.  CHESS_ATTN_AFTER_DECODE promises that
 * the kernel before it on the stream is another chess_sparse_decode (which
 * writes only out/lse), so K4 may read the block table, ws_len, tail_fill and
 * the first K/V pages before griddepcontrol.wait and overlap that kernel's
 * tail.  Without it (chess_sparse_decode, flags 0) K4 waits for the previous
 * kernel's writes before reading any state — required after chess_append_kv*,
 * which writes the token's K/V row, tail_fill and (page open) the block table. */
#define CHESS_ATTN_AFTER_DECODE 1u
int chess_sparse_decode_ex(const ChessState* st, int32_t layer, const void* q, int64_t q_stride,
                           void* out, int64_t out_stride, float* lse, float softmax_scale,
                           uint32_t flags, void* stream);

/* K5: entropy of each slot's next-token distribution from fp32 logits
 * (entropy of softmax, uncertainty.py:22-31), appended to the open page's
 * entropy ring; when the tail just sealed, page statistics
 * (uncertainty.py:41-48, NumPy summation order), trigger (uncertainty.py:86-98)
 * and policy (simulate.py:163-170) set fire[s].  logits: [batch][ld]. */
int chess_entropy_trigger(const ChessState* st, const float* logits, int64_t vocab,
                          int64_t ld, const ChessTriggerCfg* cfg, double* entropy_out,
                          void* stream);

/* K5b: append given per-slot entropies (f64 [batch]) to the entropy rings of
 * the active slots and run page statistics / trigger / policy at seal (same
 * epilogue as chess_entropy_trigger; used when the caller already holds
 * probabilities, simulate.py:160-170). */
int chess_record_entropy(const ChessState* st, const double* entropy, const uint8_t* active,
                         const ChessTriggerCfg* cfg, void* stream);

/* ---- function-level kernels (mirror pagesel free functions) ------------ */

/* score_all: scores[i] = sum_k anchor[k]*rows[i][k] in f64 (selection.py:62-74). */
int chess_score_rows(const void* rows, int32_t dtype, int64_t n_rows, int64_t dim, int64_t ld,
                     const double* anchor, double* scores, void* stream);

/* Row mean in the reference's order (page pooling hierarchy.py:115 and the
 * anchor window mean selection.py:59): out[k] = (sum_i rows[i][k]) / n. */
int chess_mean_rows(const void* rows, int32_t dtype, int64_t n_rows, int64_t dim, int64_t ld,
                    double* out, void* stream);

/* hierarchical_prune with arbitrary parent maps (selection.py:91-111).
 * Writes the kept pages in increasing order to out_pages and their count to
 * out_count[0]; out_count[1..2] = kept grids, kept chunks.  workspace >=
 * chess_prune_workspace_bytes(G, C, P) = 16*(G + C + P) + 4*(G + C) bytes. */
size_t chess_prune_workspace_bytes(int32_t G, int32_t C, int32_t P);
int chess_prune(const double* s_g, int32_t G, const double* s_c, int32_t C, const double* s_p,
                int32_t P, const int64_t* page_to_chunk, const int64_t* chunk_to_grid,
                double rho_grid, double rho_chunk, double rho_page, int32_t* out_pages,
                int32_t* out_count, void* workspace, void* stream);

/* Masked top-k with ties to the lower index (selection.py:77-88 and
 * oracle_flat_topk :114-123).  active may be NULL.  sorted != 0 returns the
 * kept indices in increasing order; otherwise in descending score order
 * (argsort(-s, stable) order).  workspace >= 16*n bytes. */
int chess_topk(const double* scores, int32_t n, int32_t k, const uint8_t* active,
               int32_t* out_idx, int32_t* out_count, int32_t sorted, void* workspace,
               void* stream);

/* reconstruct_working_set + gather_pages (selection.py:126-140,
 * kv_store.py:156-166).  selected may be unsorted / contain duplicates. */
int chess_working_set(const int32_t* selected, int32_t n_sel, int32_t n_pages, int32_t window,
                      int32_t sinks, const int32_t* page_table, int32_t* out_pages,
                      int8_t* out_prov, int32_t* out_phys, int32_t* out_len, void* stream);

/* gather_pages: out[i] = page_table[idx[i]]; err[0] = first bad position+1. */
int chess_gather_pages(const int32_t* page_table, int32_t n_pages, const int64_t* idx,
                       int32_t n, int32_t* out, int32_t* err, void* stream);

/* entropy over probability rows (uncertainty.py:22-31); flags[r] bit0 =
 * negative entry, bit1 = |sum-1| > 1e-9. */
int chess_entropy_probs(const double* probs, int64_t rows, int64_t n, int64_t ld, double* out,
                        int32_t* flags, void* stream);

/* entropy of softmax(logits) per row, fp32 logits, f64 result.  workspace
 * >= chess_entropy_workspace_bytes(rows), zero-initialised once. */
size_t chess_entropy_workspace_bytes(int64_t rows);
int chess_entropy_logits(const float* logits, int64_t rows, int64_t vocab, int64_t ld,
                         double* out, void* workspace, void* stream);

/* page_uncertainty (uncertainty.py:41-48): out = {mean, population var} in
 * NumPy pairwise summation order. */
int chess_page_uncertainty(const double* ent, int32_t n, double* out, void* stream);

/* calibrate (uncertainty.py:59-83) on the device: page_uncertainty of every
 * page's per-token entropies (entropies [n_pages][ld] f64, counts[p] >= 1
 * entries in row p, device), then the nearest-rank percentile
 * (rank = ceil(percentile * n_pages), uncertainty.py:59-61) of the page means
 * and, independently, of the variances.  out = {tau_H, tau_V} (device f64).
 * workspace >= chess_calibrate_workspace_bytes(n_pages). */
size_t chess_calibrate_workspace_bytes(int32_t n_pages);
int chess_calibrate(const double* entropies, const int32_t* counts, int32_t n_pages, int64_t ld,
                    double percentile, double* out, void* workspace, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* CHESS_B200_H */
