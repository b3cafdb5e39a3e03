// capi.cu — extern "C" entry points of libchess_b200.so (include/chess_b200.h).
//
// Host-side validation mirrors the reference's error sites (config.py:36-48,
// selection.py:55-56/68-72, hierarchy.py:108-114, kv_store.py:161-164); every
// check happens before launch, no entry point synchronises its stream.
#include <cstdarg>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "common.cuh"
#include <nvtx3/nvToolsExt.h>

// One NVTX range per C-ABI call (SURVEY.md §5 "Tracing / profiling"): host-side
// push/pop around the launch, so an nsys timeline names each kernel's entry
// point.  Header-only NVTX v3: without an attached tool a push is one
// predicted-not-taken branch.
namespace {
struct NvtxScope {
  explicit NvtxScope(const char* name) { nvtxRangePushA(name); }
  ~NvtxScope() { nvtxRangePop(); }
};
}  // namespace
#define CHESS_NVTX(name) NvtxScope chess_nvtx_scope_(name)

namespace chess {

int launch_reset(const ChessState&, const uint8_t*, cudaStream_t);
int launch_append(const ChessState&, const Workspace&, const void*, const void*, int64_t,
                  const uint8_t*, cudaStream_t, int64_t col0 = 0, int64_t ncols = -1, int post = 0);
int launch_seal(const ChessState&, const Workspace&, cudaStream_t);
int launch_select_tc_level(const ChessState&, const Workspace&, const SelParams&, int, cudaStream_t);
int launch_build(const ChessState&, const int32_t*, cudaStream_t);
int launch_from_vectors(const ChessState&, int, const double*, int, int64_t, const int32_t*,
                        cudaStream_t);
int launch_mean_rows(const void*, int, int64_t, int64_t, int64_t, double*, cudaStream_t);
int launch_select(const ChessState&, const Workspace&, const SelParams&, int, cudaStream_t);
int launch_flush_ws(const ChessState&, const Workspace&, cudaStream_t);
size_t calibrate_workspace_bytes(int n);
int launch_calibrate(const double*, const int32_t*, int, int64_t, int, double*, void*, cudaStream_t);
int launch_pool_init(const ChessState&, const int32_t*, int, cudaStream_t);
int launch_pool_reserve(const ChessState&, const int32_t*, cudaStream_t);
int launch_pool_release(const ChessState&, const uint8_t*, cudaStream_t);
int launch_select_partial(const ChessState&, const Workspace&, const SelParams&, int, cudaStream_t);
int launch_select_pull(const ChessState&, const Workspace&, const SelParams&, int, const double*,
                       const uint32_t*, uint32_t*, int32_t*, cudaStream_t);
int launch_select_combine(const ChessState&, const Workspace&, const SelParams&, int,
                          const double*, int, cudaStream_t);
int launch_build_ws_all(const ChessState&, cudaStream_t);
int launch_score_rows(const void*, int, int64_t, int64_t, int64_t, const double*, double*,
                      cudaStream_t);
int launch_prune(const double*, int, const double*, int, const double*, int, const int64_t*,
                 const int64_t*, double, double, double, int32_t*, int32_t*, void*, cudaStream_t);
int launch_topk(const double*, int, int, const uint8_t*, int32_t*, int32_t*, int, void*,
                cudaStream_t);
int launch_working_set(const int32_t*, int, int, int, int, const int32_t*, int32_t*, int8_t*,
                       int32_t*, int32_t*, cudaStream_t);
int launch_gather_pages(const int32_t*, int, const int64_t*, int, int32_t*, int32_t*,
                        cudaStream_t);
int launch_sparse_decode(const ChessState&, const Workspace&, int, const void*, int64_t, void*,
                         int64_t, float*, float, uint32_t, cudaStream_t, const PeerOut* = nullptr);
int launch_gather_finish(uint32_t* const*, uint32_t*, int, int, uint32_t*, int32_t*, const void*, int64_t,
                         int64_t, void*, cudaStream_t);
int launch_entropy_trigger(const ChessState&, const Workspace&, const float*, int64_t, int64_t,
                           const ChessTriggerCfg&, double*, cudaStream_t);
int launch_entropy_logits(const Workspace&, const float*, int64_t, int64_t, int64_t, double*,
                          cudaStream_t);
int launch_entropy_probs(const double*, int64_t, int64_t, int64_t, double*, int32_t*,
                         cudaStream_t);
int launch_page_uncertainty(const double*, int, double*, cudaStream_t);
int launch_fold(const ChessState&, const Workspace&, int, const void*, int, int, int64_t,
                cudaStream_t);
int launch_record_entropy(const ChessState&, const double*, const uint8_t*,
                          const ChessTriggerCfg&, cudaStream_t);
int attn_ctas_for(const ChessDims&);

static thread_local char g_err[512] = {0};

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(CHESS_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return CHESS_OK;
}

int num_sms() {
  static int cached = 0;
  if (cached == 0) {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && n > 0)
      cached = n;
    else {
      cudaGetLastError();
      cached = 148;
    }
  }
  return cached;
}

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

size_t workspace_layout(const ChessDims& d, void* base, Workspace* ws) {
  const int64_t b = d.batch;
  const int64_t mr = max_rows(d);
  const int64_t nsl = (d.ld + scan_slice(d.summary_dtype) - 1) / scan_slice(d.summary_dtype);
  const int64_t gq = d.kv_heads > 0 ? d.q_heads / d.kv_heads : 1;
  const int64_t attn_slots = b * d.kv_heads + kAttnWarpsMax;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off = align_up(off + bytes, 256);
    return o;
  };
  const size_t o_sel_done = take(b * 4);
  const size_t o_ws_pending = take(b * 4);
  const size_t o_flow = take((1 + 4 * b) * 4);
  const size_t o_cand = take(b * 3 * mr * 4);
  const size_t o_cand_n = take(b * 4 * 4);
  const size_t o_scores = take(b * mr * 8);
  const size_t o_keys = take(b * mr * 8);
  const size_t o_part = take(b * mr * nsl * 8);
  const size_t o_kept = take(b * mr * 4);
  const size_t o_plist = take(b * mr * 4);
  const size_t o_attn_done = take(b * d.kv_heads * 4);
  const size_t o_attn_part = take(attn_slots * gq * (d.head_dim + 4) * 4);
  const size_t o_ent_done = take(b * 4);
  const size_t o_ent_part = take(b * kEntSplit * 3 * 8);
  const size_t o_app = take(b * 4);
  const size_t o_seal = take(b * 4);
  // tensor-core scan state (summary_dtype 3 only)
  const bool tcs = d.summary_dtype == kSummaryTc;
  const int64_t nkb_pad = tcs ? (d.ld / 64 + kTcKbs - 1) / kTcKbs * kTcKbs : 0;
  const size_t o_mpend = take(b * 4);
  const size_t o_atile = take(tcs ? b * nkb_pad * 1024 : 0);
  const size_t o_astats = take(tcs ? b * nsl * 4 * 8 : 0);
  const size_t o_aexp = take(tcs ? b * nsl * 4 : 0);
  const size_t o_cls = take(tcs ? b * mr * 4 : 0);
  const size_t o_unc = take(tcs ? b * mr * 4 : 0);
  const size_t o_umeta = take(b * 4 * 4);
  if (ws && base) {
    uint8_t* p = reinterpret_cast<uint8_t*>(base);
    ws->sel_done = reinterpret_cast<int32_t*>(p + o_sel_done);
    ws->ws_pending = reinterpret_cast<int32_t*>(p + o_ws_pending);
    ws->flow = reinterpret_cast<int32_t*>(p + o_flow);
    ws->cand = reinterpret_cast<int32_t*>(p + o_cand);
    ws->cand_n = reinterpret_cast<int32_t*>(p + o_cand_n);
    ws->scores = reinterpret_cast<double*>(p + o_scores);
    ws->keys = reinterpret_cast<uint64_t*>(p + o_keys);
    ws->part = reinterpret_cast<double*>(p + o_part);
    ws->kept = reinterpret_cast<int32_t*>(p + o_kept);
    ws->plist = reinterpret_cast<int32_t*>(p + o_plist);
    ws->attn_done = reinterpret_cast<int32_t*>(p + o_attn_done);
    ws->attn_part = reinterpret_cast<float*>(p + o_attn_part);
    ws->ent_done = reinterpret_cast<int32_t*>(p + o_ent_done);
    ws->ent_part = reinterpret_cast<double*>(p + o_ent_part);
    ws->append_done = reinterpret_cast<int32_t*>(p + o_app);
    ws->seal_done = reinterpret_cast<int32_t*>(p + o_seal);
    ws->mirror_pend = reinterpret_cast<int32_t*>(p + o_mpend);
    ws->anc_tile = tcs ? p + o_atile : nullptr;
    ws->anc_stats = tcs ? reinterpret_cast<double*>(p + o_astats) : nullptr;
    ws->anc_exp = tcs ? reinterpret_cast<int32_t*>(p + o_aexp) : nullptr;
    ws->cls = tcs ? reinterpret_cast<int32_t*>(p + o_cls) : nullptr;
    ws->unc = tcs ? reinterpret_cast<int32_t*>(p + o_unc) : nullptr;
    ws->unc_meta = reinterpret_cast<int32_t*>(p + o_umeta);
    ws->nkb_pad = (int32_t)nkb_pad;
    ws->n_slices = (int32_t)nsl;
    ws->attn_ctas = std::min(attn_ctas_for(d), kAttnCtasMax);
  }
  return off;
}

static int validate(const ChessDims& d) {
  if (d.batch < 1 || d.batch > kMaxBatch) return fail(CHESS_ERR_CONFIG, "batch must be in [1, %d]", kMaxBatch);
  if (d.page_size < 1) return fail(CHESS_ERR_CONFIG, "page_size must be >= 1, got %d", d.page_size);
  if (d.page_size > 256) return fail(CHESS_ERR_UNSUPPORTED, "page_size must be <= 256");
  if (d.pages_per_chunk < 1 || d.chunks_per_grid < 1) return fail(CHESS_ERR_CONFIG, "hierarchy fan-outs must be >= 1");
  if (d.window_pages < 1) return fail(CHESS_ERR_CONFIG, "window_pages must be >= 1");
  if (d.layers < 1 || d.kv_heads < 1 || d.head_dim < 1 || d.q_heads < d.kv_heads || d.q_heads % d.kv_heads)
    return fail(CHESS_ERR_CONFIG, "bad model shape");
  if (d.dim != (int64_t)d.layers * d.kv_heads * d.head_dim)
    return fail(CHESS_ERR_CONFIG, "dim must equal layers*kv_heads*head_dim");
  if (d.ld < d.dim || d.ld % 4) return fail(CHESS_ERR_CONFIG, "ld must be >= dim and a multiple of 4");
  if (d.summary_dtype == 2 && d.ld % 8)
    return fail(CHESS_ERR_CONFIG, "bf16 summary mirrors need ld %% 8 == 0 (16-byte rows for the bulk copies)");
  if (d.max_pages < 1 || d.max_ws < 1) return fail(CHESS_ERR_CONFIG, "max_pages/max_ws must be >= 1");
  // a working set can hold every page of the table (policy 'never' keeps all
  // sealed pages, plus the open tail); a shorter block-table row would cut
  // the window / tail entries K4 relies on
  if (d.max_ws < d.max_pages)
    return fail(CHESS_ERR_CONFIG, "max_ws (%d) must be >= max_pages (%d): a working set may hold every page",
                d.max_ws, d.max_pages);
  if (d.n_phys < 1) return fail(CHESS_ERR_CONFIG, "store capacity must be >= 1 page");
  if (d.summary_dtype < 0 || d.summary_dtype > 3)
    return fail(CHESS_ERR_CONFIG, "summary_dtype must be 0 (f32), 1 (f64), 2 (bf16) or 3 (fp16 tensor-core scan)");
  if (d.summary_dtype == kSummaryTc) {
    // row groups of 8 consecutive children = one TMA box / MMA row block
    if (d.pages_per_chunk % 8 || d.chunks_per_grid % 8)
      return fail(CHESS_ERR_UNSUPPORTED, "summary_dtype 3 needs hierarchy fan-outs that are multiples of 8");
    if (d.ld % 64) return fail(CHESS_ERR_CONFIG, "summary_dtype 3 needs ld %% 64 == 0 (64-element K blocks)");
  }
  return CHESS_OK;
}

static int state_ws(const ChessState* st, Workspace* ws) {
  if (!st) return fail(CHESS_ERR_CONFIG, "null state");
  int rc = validate(st->d);
  if (rc) return rc;
  const size_t need = workspace_layout(st->d, nullptr, nullptr);
  if (!st->workspace || st->workspace_bytes < need)
    return fail(CHESS_ERR_CONFIG, "workspace too small: need %zu bytes", need);
  workspace_layout(st->d, st->workspace, ws);
  return CHESS_OK;
}

}  // namespace chess

using namespace chess;

extern "C" {

int chess_abi_version(void) { return CHESS_ABI_VERSION; }
size_t chess_dims_sizeof(void) { return sizeof(ChessDims); }
size_t chess_state_sizeof(void) { return sizeof(ChessState); }

int chess_last_error(char* buf, size_t n) {
  if (buf && n) {
    strncpy(buf, g_err, n - 1);
    buf[n - 1] = 0;
  }
  return (int)strlen(g_err);
}

int chess_validate_dims(const ChessDims* d) {
  if (!d) return fail(CHESS_ERR_CONFIG, "null dims");
  return validate(*d);
}

size_t chess_workspace_bytes(const ChessDims* d) {
  if (!d || validate(*d)) return 0;
  return workspace_layout(*d, nullptr, nullptr);
}

int chess_reset_slots(const ChessState* st, const uint8_t* mask, void* stream) {
  CHESS_NVTX("chess_reset_slots");
  Workspace ws;
  int rc = state_ws(st, &ws);
  if (rc) return rc;
  return launch_reset(*st, mask, (cudaStream_t)stream);
}

int chess_append_kv(const ChessState* st, const void* k_rows, const void* v_rows,
                    int64_t row_stride, const uint8_t* active, void* stream) {
  CHESS_NVTX("chess_append_kv");
  Workspace ws;
  int rc = state_ws(st, &ws);
  if (rc) return rc;
  if (!k_rows || !v_rows || row_stride < st->d.dim) return fail(CHESS_ERR_SHAPE, "append: bad rows");
  return launch_append(*st, ws, k_rows, v_rows, row_stride, active, (cudaStream_t)stream);
}

int chess_append_kv_layers(const ChessState* st, int32_t layer_begin, int32_t layer_end, const void* k_rows,
                           const void* v_rows, int64_t row_stride, const uint8_t* active, void* stream) {
  CHESS_NVTX("chess_append_kv_layers");
  Workspace ws;
  int rc = state_ws(st, &ws);
  if (rc) return rc;
  const ChessDims& d = st->d;
  if (layer_begin < 0 || layer_end > d.layers || layer_begin >= layer_end)
    return fail(CHESS_ERR_INDEX, "append_kv_layers: layer range [%d, %d) invalid for %d layers", layer_begin,
                layer_end, d.layers);
  const int64_t per_layer = (int64_t)d.kv_heads * d.head_dim;
  const int64_t ncols = (layer_end - layer_begin) * per_layer;
  if (!k_rows || !v_rows || row_stride < ncols) return fail(CHESS_ERR_SHAPE, "append_kv_layers: bad rows");
  return launch_append(*st, ws, k_rows, v_rows, row_stride, active, (cudaStream_t)stream,
                       layer_begin * per_layer, ncols, layer_begin > 0 ? 1 : 0);
}

int chess_summary_seal(const ChessState* st, void* stream) {
  CHESS_NVTX("chess_summary_seal");
  Workspace ws;
  int rc = state_ws(st, &ws);
  if (rc) return rc;
  return launch_seal(*st, ws, (cudaStream_t)stream);
}

int chess_summary_build(const ChessState* st, const int32_t* n_pages, void* stream) {
  CHESS_NVTX("chess_summary_build");
  Workspace ws;
  int rc = state_ws(st, &ws);
  if (rc) return rc;
  if (!n_pages) return fail(CHESS_ERR_CONFIG, "summary_build: null n_pages");
  return launch_build(*st, n_pages, (cudaStream_t)stream);
}

int chess_summary_from_vectors(const ChessState* st, int32_t seq, const double* rows, int32_t n,
                               int64_t row_stride, void* stream) {
  CHESS_NVTX("chess_summary_from_vectors");
  Workspace ws;
  int rc = state_ws(st, &ws);
  if (rc) return rc;
  if (seq < 0 || seq >= st->d.batch) return fail(CHESS_ERR_INDEX, "slot %d out of range", seq);
  if (n < 0 || n > st->d.max_pages) return fail(CHESS_ERR_CONFIG, "from_vectors: %d rows exceed capacity", n);
  if (n > 0 && (!rows || row_stride < st->d.dim)) return fail(CHESS_ERR_SHAPE, "from_vectors: bad rows");
  // device copy of n for the epilogue: reuse the slot's sel_done counter cell? no —
  // use the append counter of `seq` temporarily is unsafe; write into cand_n.
  int32_t* n_dev = ws.cand_n + 4 * seq + 3;
  cudaMemcpyAsync(n_dev, &n, sizeof(int32_t), cudaMemcpyHostToDevice, (cudaStream_t)stream);
  return launch_from_vectors(*st, seq, rows, n, row_stride, n_dev, (cudaStream_t)stream);
}

int chess_summary_fold(const ChessState* st, int32_t seq, const void* rows, int32_t dtype,
                       int32_t n_rows, int64_t row_stride, void* stream) {
  CHESS_NVTX("chess_summary_fold");
  Workspace ws;
  int rc = state_ws(st, &ws);
  if (rc) return rc;
  if (seq < 0 || seq >= st->d.batch) return fail(CHESS_ERR_INDEX, "slot %d out of range", seq);
  if (n_rows < 1) return fail(CHESS_ERR_ORDER, "only sealed pages can be finalized");
  if (!rows || row_stride < st->d.dim) return fail(CHESS_ERR_SHAPE, "fold: bad rows");
  if (dtype < 0 || dtype > 2) return fail(CHESS_ERR_CONFIG, "bad dtype");
  return launch_fold(*st, ws, seq, rows, dtype, n_rows, row_stride, (cudaStream_t)stream);
}

int chess_record_entropy(const ChessState* st, const double* entropy, const uint8_t* active,
                         const ChessTriggerCfg* cfg, void* stream) {
  CHESS_NVTX("chess_record_entropy");
  Workspace ws;
  int rc = state_ws(st, &ws);
  if (rc) return rc;
  if (!cfg || !entropy) return fail(CHESS_ERR_CONFIG, "record_entropy: null argument");
  if (cfg->policy < 0 || cfg->policy > 4) return fail(CHESS_ERR_CONFIG, "unknown policy %d", cfg->policy);
  if (cfg->policy == CHESS_POLICY_FIXED && cfg->interval < 1) return fail(CHESS_ERR_CONFIG, "fixed interval must be >= 1 page");
  if (cfg->mode != 0 && cfg->mode != 1) return fail(CHESS_ERR_VALUE, "unknown trigger mode %d", cfg->mode);
  return launch_record_entropy(*st, entropy, active, *cfg, (cudaStream_t)stream);
}

static int select_params(const ChessSelectCfg* cfg, SelParams* out) {
  if (!cfg) return fail(CHESS_ERR_CONFIG, "null select cfg");
  const double r[3] = {cfg->rho_grid, cfg->rho_chunk, cfg->rho_page};
  for (int i = 0; i < 3; ++i)
    if (!(r[i] > 0.0 && r[i] <= 1.0)) return fail(CHESS_ERR_CONFIG, "ratios must be in (0, 1]");
  SelParams prm = {};
  prm.rho[0] = r[0];
  prm.rho[1] = r[1];
  prm.rho[2] = r[2];
  prm.full_scan = cfg->full_scan;
  static const int dbg_mode = getenv("CHESS_SELECT_MODE") ? atoi(getenv("CHESS_SELECT_MODE")) : 0;
  prm.mode = dbg_mode;
  prm.force_all = cfg->force_all;
  prm.defer_ws = cfg->defer_ws;
  *out = prm;
  return CHESS_OK;
}

int chess_select(const ChessState* st, const ChessSelectCfg* cfg, void* stream) {
  CHESS_NVTX("chess_select");
  Workspace ws;
  int rc = state_ws(st, &ws);
  if (rc) return rc;
  SelParams prm;
  if ((rc = select_params(cfg, &prm))) return rc;
  return launch_select(*st, ws, prm, 0, (cudaStream_t)stream);
}

// ---- debug / test entries (not in include/chess_b200.h) -------------------

// summary_dtype 3: anchor split + tensor-core scan of one level (conditional
// cascade), stopping before the exact rescoring launch
extern "C" int chess_debug_select_tc_level(const ChessState* st, const ChessSelectCfg* cfg, int32_t level,
                                           void* stream) {
  Workspace ws;
  int rc = state_ws(st, &ws);
  if (rc) return rc;
  if (st->d.summary_dtype != kSummaryTc) return fail(CHESS_ERR_CONFIG, "summary_dtype 3 only");
  if (level < 0 || level > 2) return fail(CHESS_ERR_VALUE, "level %d", level);
  SelParams prm;
  if ((rc = select_params(cfg, &prm))) return rc;
  return launch_select_tc_level(*st, ws, prm, level, (cudaStream_t)stream);
}

// Copy slot `slot`'s certified intervals of the last tensor-core level tail
// (lo in ws.scores, hi in the first slice partial), classes, the
// {uncertain, seats left, candidates, cumulative rescored} counters and the
// level's candidate ids (level > 0) to host buffers (synchronous; any pointer
// may be NULL).
extern "C" int chess_debug_tc_read(const ChessState* st, int32_t slot, int32_t level, int32_t n, double* lo,
                                   double* hi, int32_t* cls, int32_t* meta, int32_t* cand) {
  Workspace ws;
  int rc = state_ws(st, &ws);
  if (rc) return rc;
  if (st->d.summary_dtype != kSummaryTc) return fail(CHESS_ERR_CONFIG, "summary_dtype 3 only");
  const int64_t mr = max_rows(st->d);
  if (slot < 0 || slot >= st->d.batch || n < 0 || n > mr) return fail(CHESS_ERR_INDEX, "slot/n out of range");
  cudaDeviceSynchronize();
  if (lo) cudaMemcpy(lo, ws.scores + slot * mr, n * sizeof(double), cudaMemcpyDeviceToHost);
  if (hi)
    cudaMemcpy2D(hi, sizeof(double), ws.part + slot * mr * ws.n_slices, ws.n_slices * sizeof(double),
                 sizeof(double), n, cudaMemcpyDeviceToHost);
  if (cls) cudaMemcpy(cls, ws.cls + slot * mr, n * sizeof(int32_t), cudaMemcpyDeviceToHost);
  if (meta) cudaMemcpy(meta, ws.unc_meta + 4 * slot, 4 * sizeof(int32_t), cudaMemcpyDeviceToHost);
  if (cand && level > 0)
    cudaMemcpy(cand, ws.cand + (slot * 3 + level) * mr, n * sizeof(int32_t), cudaMemcpyDeviceToHost);
  return check_launch("debug_tc_read");
}

// rows a level can have for one slot: its exchange row stride must hold them
static int64_t level_capacity(const ChessDims& d, int level) {
  const int64_t mc = (d.max_pages + d.pages_per_chunk - 1) / d.pages_per_chunk;
  const int64_t mg = (mc + d.chunks_per_grid - 1) / d.chunks_per_grid;
  return level == 0 ? mg : level == 1 ? mc : level == 2 ? (int64_t)d.max_pages : mg + mc + d.max_pages;
}

static int check_level(const ChessState* st, const ChessSelectCfg* cfg, int32_t level, int64_t ld) {
  if (cfg->full_scan ? level != 3 : (level < 0 || level > 2))
    return fail(CHESS_ERR_VALUE, "select level %d invalid (conditional scan: 0..2, full scan: 3)", level);
  if (ld < level_capacity(st->d, level))
    return fail(CHESS_ERR_SHAPE, "exchange stride %lld < level %d capacity %lld", (long long)ld, level,
                (long long)level_capacity(st->d, level));
  return CHESS_OK;
}

int chess_select_partial(const ChessState* st, const ChessSelectCfg* cfg, int32_t level,
                         double* partial, int64_t ld_partial, void* stream) {
  CHESS_NVTX("chess_select_partial");
  Workspace ws;
  int rc = state_ws(st, &ws);
  if (rc) return rc;
  SelParams prm;
  if ((rc = select_params(cfg, &prm))) return rc;
  if ((rc = check_level(st, cfg, level, ld_partial))) return rc;
  if (!partial) return fail(CHESS_ERR_SHAPE, "select_partial: null partial buffer");
  prm.xout = partial;
  prm.xld = ld_partial;
  return launch_select_partial(*st, ws, prm, level, (cudaStream_t)stream);
}

int chess_select_combine(const ChessState* st, const ChessSelectCfg* cfg, int32_t level,
                         const double* gathered, int32_t world, int64_t ld_partial, void* stream) {
  CHESS_NVTX("chess_select_combine");
  Workspace ws;
  int rc = state_ws(st, &ws);
  if (rc) return rc;
  SelParams prm;
  if ((rc = select_params(cfg, &prm))) return rc;
  if ((rc = check_level(st, cfg, level, ld_partial))) return rc;
  if (!gathered || world < 1) return fail(CHESS_ERR_SHAPE, "select_combine: bad gathered buffer / world");
  prm.xld = ld_partial;
  return launch_select_combine(*st, ws, prm, level, gathered, world, (cudaStream_t)stream);
}

static int peer_params(const ChessState* st, const ChessSelectCfg* cfg, int32_t level,
                       const ChessPeerExchange* px, SelParams* prm) {
  int rc;
  if ((rc = select_params(cfg, prm))) return rc;
  if (!px) return fail(CHESS_ERR_CONFIG, "null peer exchange");
  if ((rc = check_level(st, cfg, level, px->ld))) return rc;
  if (px->world < 1 || px->world > kMaxPeers || px->rank < 0 || px->rank >= px->world)
    return fail(CHESS_ERR_CONFIG, "peer exchange rank %d / world %d invalid (world <= %d)", px->rank, px->world,
                kMaxPeers);
  if (!px->recv || !px->flags || !px->gen || !px->err)
    return fail(CHESS_ERR_CONFIG, "peer exchange: null recv/flags/gen/err");
  prm->xpeer = px->recv;
  prm->xflag = px->flags;
  prm->xgen = px->gen;
  prm->xrank = px->rank;
  prm->xworld = px->world;
  prm->xld = px->ld;
  return CHESS_OK;
}

int chess_select_push(const ChessState* st, const ChessSelectCfg* cfg, int32_t level,
                      const ChessPeerExchange* px, void* stream) {
  CHESS_NVTX("chess_select_push");
  Workspace ws;
  int rc = state_ws(st, &ws);
  if (rc) return rc;
  SelParams prm;
  if ((rc = peer_params(st, cfg, level, px, &prm))) return rc;
  return launch_select_partial(*st, ws, prm, level, (cudaStream_t)stream);
}

int chess_select_pull(const ChessState* st, const ChessSelectCfg* cfg, int32_t level,
                      const ChessPeerExchange* px, void* stream) {
  CHESS_NVTX("chess_select_pull");
  Workspace ws;
  int rc = state_ws(st, &ws);
  if (rc) return rc;
  SelParams prm;
  if ((rc = peer_params(st, cfg, level, px, &prm))) return rc;
  if (!px->my_recv || !px->my_flags) return fail(CHESS_ERR_CONFIG, "select_pull: null my_recv/my_flags");
  return launch_select_pull(*st, ws, prm, level, px->my_recv, px->my_flags, px->gen, px->err, (cudaStream_t)stream);
}

int chess_p2p_alloc(int64_t bytes, void** ptr) {
  if (!ptr || bytes <= 0) return fail(CHESS_ERR_CONFIG, "p2p_alloc: bad arguments");
  if (cudaMalloc(ptr, (size_t)bytes) != cudaSuccess) return fail(CHESS_ERR_CUDA, "p2p_alloc: cudaMalloc");
  if (cudaMemset(*ptr, 0, (size_t)bytes) != cudaSuccess) return fail(CHESS_ERR_CUDA, "p2p_alloc: memset");
  return CHESS_OK;
}
int chess_p2p_free(void* ptr) {
  return cudaFree(ptr) == cudaSuccess ? CHESS_OK : fail(CHESS_ERR_CUDA, "p2p_free");
}
int chess_p2p_export(void* ptr, uint8_t* handle) {
  static_assert(sizeof(cudaIpcMemHandle_t) == CHESS_IPC_HANDLE_BYTES, "ipc handle size");
  cudaIpcMemHandle_t h;
  if (!ptr || !handle || cudaIpcGetMemHandle(&h, ptr) != cudaSuccess)
    return fail(CHESS_ERR_CUDA, "p2p_export: cudaIpcGetMemHandle");
  memcpy(handle, &h, sizeof(h));
  return CHESS_OK;
}
int chess_p2p_open(const uint8_t* handle, void** ptr) {
  cudaIpcMemHandle_t h;
  if (!handle || !ptr) return fail(CHESS_ERR_CONFIG, "p2p_open: null argument");
  memcpy(&h, handle, sizeof(h));
  if (cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
    return fail(CHESS_ERR_CUDA, "p2p_open: cudaIpcOpenMemHandle");
  return CHESS_OK;
}
int chess_p2p_close(void* ptr) {
  return cudaIpcCloseMemHandle(ptr) == cudaSuccess ? CHESS_OK : fail(CHESS_ERR_CUDA, "p2p_close");
}

static int pool_state(const ChessState* st) {
  if (!st) return fail(CHESS_ERR_CONFIG, "null state");
  if (!st->pool_free || !st->pool_top || !st->pool_base || !st->pool_end || !st->pool_oom)
    return fail(CHESS_ERR_CONFIG, "state has no device page pool (pool_* pointers unset)");
  return CHESS_OK;
}

int chess_pool_init(const ChessState* st, const int32_t* ids, int32_t n, void* stream) {
  CHESS_NVTX("chess_pool_init");
  int rc = pool_state(st);
  if (rc) return rc;
  if (n < 0 || n > st->d.n_phys) return fail(CHESS_ERR_CONFIG, "pool of %d pages > n_phys %lld", n, (long long)st->d.n_phys);
  if (n > 0 && !ids) return fail(CHESS_ERR_SHAPE, "pool_init: null ids");
  return launch_pool_init(*st, ids, n, (cudaStream_t)stream);
}

int chess_pool_reserve(const ChessState* st, const int32_t* counts, void* stream) {
  CHESS_NVTX("chess_pool_reserve");
  int rc = pool_state(st);
  if (rc) return rc;
  if (!counts) return fail(CHESS_ERR_SHAPE, "pool_reserve: null counts");
  return launch_pool_reserve(*st, counts, (cudaStream_t)stream);
}

int chess_pool_release(const ChessState* st, const uint8_t* mask, void* stream) {
  CHESS_NVTX("chess_pool_release");
  int rc = pool_state(st);
  if (rc) return rc;
  return launch_pool_release(*st, mask, (cudaStream_t)stream);
}

int chess_flush_working_sets(const ChessState* st, void* stream) {
  CHESS_NVTX("chess_flush_working_sets");
  Workspace ws;
  int rc = state_ws(st, &ws);
  if (rc) return rc;
  return launch_flush_ws(*st, ws, (cudaStream_t)stream);
}

int chess_build_working_set(const ChessState* st, void* stream) {
  CHESS_NVTX("chess_build_working_set");
  Workspace ws;
  int rc = state_ws(st, &ws);
  if (rc) return rc;
  return launch_build_ws_all(*st, (cudaStream_t)stream);
}

int chess_sparse_decode(const ChessState* st, int32_t layer, const void* q, int64_t q_stride,
                        void* out, int64_t out_stride, float* lse, float softmax_scale,
                        void* stream) {
  return chess_sparse_decode_ex(st, layer, q, q_stride, out, out_stride, lse, softmax_scale, 0u, stream);
}

int chess_sparse_decode_ex(const ChessState* st, int32_t layer, const void* q, int64_t q_stride,
                           void* out, int64_t out_stride, float* lse, float softmax_scale,
                           uint32_t flags, void* stream) {
  CHESS_NVTX("chess_sparse_decode_ex");
  Workspace ws;
  int rc = state_ws(st, &ws);
  if (rc) return rc;
  if (layer < 0 || layer >= st->d.layers) return fail(CHESS_ERR_INDEX, "layer %d out of range", layer);
  if (!q || !out) return fail(CHESS_ERR_SHAPE, "sparse_decode: null q/out");
  const int64_t row = (int64_t)st->d.q_heads * st->d.head_dim;
  if (q_stride < row || out_stride < row) return fail(CHESS_ERR_SHAPE, "sparse_decode: stride < q_heads*head_dim");
  if (flags & ~(uint32_t)CHESS_ATTN_AFTER_DECODE) return fail(CHESS_ERR_CONFIG, "sparse_decode: unknown flags %#x", flags);
  return launch_sparse_decode(*st, ws, layer, q, q_stride, out, out_stride, lse, softmax_scale, flags,
                              (cudaStream_t)stream);
}

static int check_peer_outputs(const ChessState* st, const ChessPeerOutputs* po) {
  if (!st || !po) return fail(CHESS_ERR_CONFIG, "null state / peer outputs");
  if (po->world < 1 || po->world > kMaxPeers || po->rank < 0 || po->rank >= po->world)
    return fail(CHESS_ERR_CONFIG, "peer outputs: rank %d / world %d invalid (world <= %d)", po->rank, po->world,
                kMaxPeers);
  if (!po->regions || !po->flags || !po->my_flags || !po->gen || !po->err)
    return fail(CHESS_ERR_CONFIG, "peer outputs: null regions/flags/my_flags/gen/err");
  for (int p = 0; p < po->world; ++p)
    if (!po->regions[p] || (reinterpret_cast<uintptr_t>(po->regions[p]) & 15))
      return fail(CHESS_ERR_CONFIG, "peer outputs: region %d null or not 16-byte aligned", p);
  return CHESS_OK;
}

// elements of one (layer, rank) block of a region
static int64_t gather_block(const ChessDims& d) { return (int64_t)d.batch * d.q_heads * d.head_dim; }

int chess_sparse_decode_gather(const ChessState* st, int32_t layer, const void* q, int64_t q_stride,
                               void* out, int64_t out_stride, float* lse, float softmax_scale,
                               uint32_t flags, const ChessPeerOutputs* po, void* stream) {
  CHESS_NVTX("chess_sparse_decode_gather");
  Workspace ws;
  int rc = state_ws(st, &ws);
  if (rc) return rc;
  if ((rc = check_peer_outputs(st, po))) return rc;
  if (layer < 0 || layer >= st->d.layers) return fail(CHESS_ERR_INDEX, "layer %d out of range", layer);
  const int64_t row = (int64_t)st->d.q_heads * st->d.head_dim;
  if (!q || q_stride < row) return fail(CHESS_ERR_SHAPE, "sparse_decode_gather: null q / q_stride < q_heads*head_dim");
  if (!out || out_stride != row)
    return fail(CHESS_ERR_SHAPE, "sparse_decode_gather: out must be this rank's [batch][q_heads*head_dim] block "
                "with out_stride == q_heads*head_dim");
  const int64_t blk = gather_block(st->d);
  const int64_t off = ((int64_t)layer * po->world + po->rank) * blk;
  PeerOut pe;
  pe.n_peer = 0;
  for (int p = 0; p < po->world; ++p)
    if (p != po->rank) pe.peer_out[pe.n_peer++] = static_cast<__nv_bfloat16*>(po->regions[p]) + off;
  if (flags & ~(uint32_t)CHESS_ATTN_AFTER_DECODE)
    return fail(CHESS_ERR_CONFIG, "sparse_decode_gather: unknown flags %#x", flags);
  return launch_sparse_decode(*st, ws, layer, q, q_stride, out, row, lse, softmax_scale, flags,
                              (cudaStream_t)stream, &pe);
}

int chess_gather_finish(const ChessState* st, const ChessPeerOutputs* po, void* out, void* stream) {
  CHESS_NVTX("chess_gather_finish");
  int rc;
  if ((rc = check_peer_outputs(st, po))) return rc;
  const int64_t elems = (int64_t)st->d.layers * po->world * gather_block(st->d);
  if (elems % 8 || (reinterpret_cast<uintptr_t>(out) & 15))
    return fail(CHESS_ERR_SHAPE, "gather_finish: output must be 16-byte aligned with a multiple of 8 elements");
  return launch_gather_finish(po->flags, po->my_flags, po->world, po->rank, po->gen, po->err,
                              po->regions[po->rank], elems, gather_block(st->d), out, (cudaStream_t)stream);
}

int chess_entropy_trigger(const ChessState* st, const float* logits, int64_t vocab, int64_t ld,
                          const ChessTriggerCfg* cfg, double* entropy_out, void* stream) {
  CHESS_NVTX("chess_entropy_trigger");
  Workspace ws;
  int rc = state_ws(st, &ws);
  if (rc) return rc;
  if (!cfg || !logits || vocab < 1 || ld < vocab) return fail(CHESS_ERR_SHAPE, "entropy_trigger: bad logits");
  if (cfg->policy < 0 || cfg->policy > 4) return fail(CHESS_ERR_CONFIG, "unknown policy %d", cfg->policy);
  if (cfg->policy == CHESS_POLICY_FIXED && cfg->interval < 1) return fail(CHESS_ERR_CONFIG, "fixed interval must be >= 1 page");
  if (cfg->mode != 0 && cfg->mode != 1) return fail(CHESS_ERR_VALUE, "unknown trigger mode %d", cfg->mode);
  return launch_entropy_trigger(*st, ws, logits, vocab, ld, *cfg, entropy_out, (cudaStream_t)stream);
}

int chess_score_rows(const void* rows, int32_t dtype, int64_t n_rows, int64_t dim, int64_t ld,
                     const double* anchor, double* scores, void* stream) {
  CHESS_NVTX("chess_score_rows");
  if (n_rows < 0 || dim < 0 || ld < dim) return fail(CHESS_ERR_SHAPE, "score_rows: bad shape");
  if (dtype < 0 || dtype > 2) return fail(CHESS_ERR_CONFIG, "bad dtype");
  return launch_score_rows(rows, dtype, n_rows, dim, ld, anchor, scores, (cudaStream_t)stream);
}

int chess_mean_rows(const void* rows, int32_t dtype, int64_t n_rows, int64_t dim, int64_t ld,
                    double* out, void* stream) {
  CHESS_NVTX("chess_mean_rows");
  if (n_rows < 1) return fail(CHESS_ERR_EMPTY_CONTEXT, "no rows to average");
  if (dim < 0 || ld < dim) return fail(CHESS_ERR_SHAPE, "mean_rows: bad shape");
  if (dim == 0) return CHESS_OK;
  return launch_mean_rows(rows, dtype, n_rows, dim, ld, out, (cudaStream_t)stream);
}

size_t chess_prune_workspace_bytes(int32_t G, int32_t C, int32_t P) {
  if (G < 0 || C < 0 || P < 0) return 0;
  // keys (8 B) + kept (4 B) + cand (4 B) per candidate, then the kept-grid /
  // kept-chunk masks (4 B each) — prune_kernel's layout
  return 16 * ((size_t)G + C + P) + 4 * ((size_t)G + C);
}

int chess_prune(const double* s_g, int32_t G, const double* s_c, int32_t C, const double* s_p,
                int32_t P, const int64_t* page_to_chunk, const int64_t* chunk_to_grid,
                double rho_grid, double rho_chunk, double rho_page, int32_t* out_pages,
                int32_t* out_count, void* workspace, void* stream) {
  CHESS_NVTX("chess_prune");
  if (G < 0 || C < 0 || P < 0) return fail(CHESS_ERR_SHAPE, "prune: negative sizes");
  return launch_prune(s_g, G, s_c, C, s_p, P, page_to_chunk, chunk_to_grid, rho_grid, rho_chunk,
                      rho_page, out_pages, out_count, workspace, (cudaStream_t)stream);
}

int chess_topk(const double* scores, int32_t n, int32_t k, const uint8_t* active,
               int32_t* out_idx, int32_t* out_count, int32_t sorted, void* workspace,
               void* stream) {
  CHESS_NVTX("chess_topk");
  if (n < 0) return fail(CHESS_ERR_SHAPE, "topk: negative n");
  return launch_topk(scores, n, k, active, out_idx, out_count, sorted, workspace,
                     (cudaStream_t)stream);
}

int chess_working_set(const int32_t* selected, int32_t n_sel, int32_t n_pages, int32_t window,
                      int32_t sinks, const int32_t* page_table, int32_t* out_pages,
                      int8_t* out_prov, int32_t* out_phys, int32_t* out_len, void* stream) {
  CHESS_NVTX("chess_working_set");
  if (window < 1) return fail(CHESS_ERR_CONFIG, "window_pages must be >= 1");
  if (sinks < 0) return fail(CHESS_ERR_CONFIG, "sink_pages must be >= 0");
  if (n_pages < 0 || n_sel < 0) return fail(CHESS_ERR_SHAPE, "working_set: negative sizes");
  return launch_working_set(selected, n_sel, n_pages, window, sinks, page_table, out_pages,
                            out_prov, out_phys, out_len, (cudaStream_t)stream);
}

int chess_gather_pages(const int32_t* page_table, int32_t n_pages, const int64_t* idx, int32_t n,
                       int32_t* out, int32_t* err, void* stream) {
  CHESS_NVTX("chess_gather_pages");
  return launch_gather_pages(page_table, n_pages, idx, n, out, err, (cudaStream_t)stream);
}

int chess_entropy_probs(const double* probs, int64_t rows, int64_t n, int64_t ld, double* out,
                        int32_t* flags, void* stream) {
  CHESS_NVTX("chess_entropy_probs");
  if (rows < 0 || n < 1 || ld < n) return fail(CHESS_ERR_SHAPE, "entropy_probs: bad shape");
  return launch_entropy_probs(probs, rows, n, ld, out, flags, (cudaStream_t)stream);
}

size_t chess_entropy_workspace_bytes(int64_t rows) {
  return (size_t)rows * (kEntSplit * 3 * 8 + 8) + 512;
}

int chess_entropy_logits(const float* logits, int64_t rows, int64_t vocab, int64_t ld, double* out,
                         void* workspace, void* stream) {
  CHESS_NVTX("chess_entropy_logits");
  if (rows < 0 || vocab < 1 || ld < vocab) return fail(CHESS_ERR_SHAPE, "entropy_logits: bad shape");
  if (rows == 0) return CHESS_OK;
  Workspace ws{};
  uint8_t* p = reinterpret_cast<uint8_t*>(workspace);
  ws.ent_done = reinterpret_cast<int32_t*>(p);
  ws.ent_part = reinterpret_cast<double*>(p + ((rows * 4 + 255) / 256) * 256);
  return launch_entropy_logits(ws, logits, rows, vocab, ld, out, (cudaStream_t)stream);
}

size_t chess_calibrate_workspace_bytes(int32_t n_pages) {
  return n_pages > 0 ? calibrate_workspace_bytes(n_pages) : 0;
}

int chess_calibrate(const double* entropies, const int32_t* counts, int32_t n_pages, int64_t ld,
                    double percentile, double* out, void* workspace, void* stream) {
  CHESS_NVTX("chess_calibrate");
  // CalibrationError cases (uncertainty.py:66-69) -> ValueError status
  if (n_pages < 1) return fail(CHESS_ERR_VALUE, "cannot calibrate on an empty sample");
  if (!(percentile > 0.0 && percentile < 1.0))
    return fail(CHESS_ERR_VALUE, "percentile must be in (0, 1), got %g", percentile);
  if (!entropies || !counts || !out || !workspace) return fail(CHESS_ERR_SHAPE, "calibrate: null buffer");
  if (ld < 1) return fail(CHESS_ERR_SHAPE, "calibrate: bad row stride");
  // nearest rank, ceil in double as math.ceil(percentile * len) (uncertainty.py:60)
  int rank = (int)ceil(percentile * (double)n_pages);
  rank = rank < 1 ? 1 : rank;
  return launch_calibrate(entropies, counts, n_pages, ld, rank, out, workspace, (cudaStream_t)stream);
}

int chess_page_uncertainty(const double* ent, int32_t n, double* out, void* stream) {
  CHESS_NVTX("chess_page_uncertainty");
  if (n < 1) return fail(CHESS_ERR_VALUE, "page has no generated tokens");

  return launch_page_uncertainty(ent, n, out, (cudaStream_t)stream);
}

}  // extern "C"
