// C ABI of the B200 KPM-DOS hot path (include/kpm.h).  Host orchestration only: every step
// of the path (start block, sweeps, dot products, reductions) runs in the kernels of
// kernels.cu; this file validates arguments, builds the SELL copy, owns device memory and
// enqueues the work on one stream.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <cuda.h>
#include <nccl.h>

#include <array>
#include <chrono>
#include <condition_variable>
#include <map>
#include <mutex>
#include <thread>

#include "../../include/kpm.h"
#include "chunk_order.h"
#include "halo_plan.h"
#include "kpm_internal.h"
#include "sell_build.h"

using namespace kpm;

// In-process group of "virtual ranks" (test harness, kpm.h KPM_VIRTUAL_RANKS): nranks contexts on
// one device, driven by nranks host threads, whose setup collectives and final eta reduction run
// through this host rendezvous instead of NCCL, and whose fused halo exchange stores into the
// other contexts' buffers through plain device pointers instead of CUDA IPC mappings.  The sweep
// kernels, the edge / interior split and the flag-epoch protocol are the multi-GPU ones.
// KPM_TRACE=1 (read once): progress lines on stderr (rank, step) -- hang diagnosis for the
// multi-rank protocol.
static bool trace_on() {
  static const bool on = getenv("KPM_TRACE") && atoi(getenv("KPM_TRACE")) > 0;
  return on;
}
#define KPM_TRACE_LINE(rank, ...)                 \
  do {                                            \
    if (trace_on()) {                             \
      fprintf(stderr, "[kpm r%d] ", (int)(rank)); \
      fprintf(stderr, __VA_ARGS__);               \
      fprintf(stderr, "\n");                      \
      fflush(stderr);                             \
    }                                             \
  } while (0)

struct kpm_vgroup {
  int P = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  int64_t gen = 0;
  std::vector<std::vector<int64_t>> slot, result;
  // all-gather of variable-length int64 vectors; every rank gets every rank's vector
  std::vector<std::vector<int64_t>> allgatherv(int rank, const std::vector<int64_t>& mine) {
    std::unique_lock<std::mutex> lk(mu);
    KPM_TRACE_LINE(rank, "vgroup rendezvous %lld (%zu words)", (long long)gen, mine.size());
    slot[rank] = mine;
    const int64_t g = gen;
    if (++arrived == P) {
      result = slot;
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
    return result;
  }
};

struct kpm_ctx {
  kpm_options opt{};
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  bool sticky = false;
  std::string err;
  int num_sms = 148;
  int variant_override = -1;  // tuning knob: env KPM_VARIANT (index into the width's variants)
  int grid_per_sm = 0;        // 0 -> occupancy (env KPM_GRID_PER_SM)
  int tile_stages = 0;        // 0 -> as many as fit (env KPM_TILE_STAGES)
  std::string last_variant;

  // matrix
  bool have_matrix = false;
  int64_t n_global = 0, row_begin = 0, row_end = 0;
  double a = 0.0, b = 0.0;
  DevSell sell;
  std::vector<int64_t> halo;  // global ids of halo slots
  std::vector<int64_t> cptr_h;  // host copy of cptr

  // work buffers (grow-only)
  double2* X0 = nullptr;
  double2* X1 = nullptr;
  size_t x_cap = 0;  // elements per buffer
  double* partials = nullptr;
  size_t partials_cap = 0;  // doubles
  double2* eta_even = nullptr;
  double2* eta_odd = nullptr;
  size_t eta_cap = 0;  // double2 per array
  double2* h_eta = nullptr;  // pinned staging, 2*eta_cap
  double2* v0_dev = nullptr;
  size_t v0_cap = 0;
  double2* u_naive = nullptr;  // naive stage's u vector
  size_t u_cap = 0;
  int64_t* stage_rp = nullptr;  // device staging of a host CSR (device SELL build)
  int64_t* stage_col = nullptr;
  double2* stage_val = nullptr;
  size_t stage_rp_cap = 0, stage_col_cap = 0, stage_val_cap = 0;
  BuildScratch build_ws;  // device SELL build temporaries

  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};

  // multi-rank (nranks > 1): row distribution, halo exchange plan, NCCL
  ncclComm_t comm = nullptr;
  kpm_vgroup* vg = nullptr;         // virtual ranks (no NCCL): the in-process group
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_edge = nullptr, ev_halo = nullptr;
  std::vector<int64_t> row_begins;  // nranks+1
  std::vector<RecvRun> recv_runs;
  std::vector<SendRun> send_runs;
  int64_t* edge_list = nullptr;     // device: chunks holding sent rows or reading halo slots
  int64_t* interior_list = nullptr; // device: the other chunks
  int64_t n_edge = 0, n_interior = 0;
  std::vector<char> edge_flag;      // host: chunk is an edge chunk
  std::vector<int64_t> order_h;     // chunk processing order given by kpm_set_chunk_order
  bool order_user = false;          // order_h is in force (else the library's own choice)
  int64_t* order_list = nullptr;    // device copy of the installed order for single-rank sweeps
  int64_t order_id = -3;            // installed order: -1 user, 0 storage, 4 G + w: line walk of width w, grid G
  int64_t order_gen = 0;            // bumped by every install (keys of the block-cache plan, CUDA graph)
  std::map<int64_t, std::vector<int64_t>> auto_order;  // line walk per (grid, width) (chunk_order.cpp)
  int adj_state = 0;                // block-neighbour lists: 0 not built, 1 built, -1 unavailable
  std::vector<int64_t> adj_ptr, adj;
  int64_t adj_maxoff = 0;          // typical_block_offset of the matrix (chunks)
  int64_t* halo_rows = nullptr;     // device: global id of each halo slot
  // fused halo exchange (peer stores from the sweep epilogue + stream flag ops)
  bool fused = false;               // chosen per set_matrix (env KPM_HALO=nccl|fused)
  bool fused_ready = false;         // IPC mappings valid for the current X0/X1
  int32_t* flags = nullptr;         // device: flags[src] = last sweep epoch whose halo src wrote
  uint32_t epoch = 0;
  std::map<std::string, void*> ipc_open;  // opened peer handles (by handle bytes)
  std::vector<std::array<double2*, 2>> dst_x;  // per send run: peer's X0/X1 + (peer n_pad + slot)*Rk
  std::vector<int32_t*> dst_flag;   // per destination peer (parallel to dest_peers)
  std::vector<int> dest_peers, src_peers;
  int fused_rk = 0;
  // CUDA graph of the single-rank sweep loop (cached per configuration)
  bool use_graph = true;
  cudaGraphExec_t graph_exec = nullptr;
  std::vector<int64_t> graph_key;
  int64_t matrix_gen = 0;           // bumped by every kpm_set_matrix / kpm_set_chunk_order
  // block-cache feed (single rank): per-position records, tile maps, absolute tile rows
  uint4* bc_rec = nullptr;           // single rank, or the edge list of several ranks
  uint4* bc_rec2 = nullptr;          // the interior list of several ranks
  size_t bc_rec2_cap = 0;
  int* bc_map = nullptr;
  uint16_t* bc_lcol = nullptr;
  int* bc_fail = nullptr;
  size_t bc_rec_cap = 0, bc_map_cap = 0, bc_lcol_cap = 0, bc_fail_cap = 0;
  std::vector<int64_t> bc_key;      // (R, grid, matrix_gen, stages, ...) the buffers were built for
  int chosen[6] = {0, 0, 0, 0, 0, 0};  // per log2(R): selected variant (select_variant) ...
  int64_t chosen_gen[6] = {-1, -1, -1, -1, -1, -1};  // ... for this matrix_gen ...
  int chosen_ovr[6] = {-2, -2, -2, -2, -2, -2};      // ... and this KPM_VARIANT override
  bool bc_ok = false;
  bool lcol_t = false;             // block-cache feed: row-major tile indices (env KPM_LCOL_T)
  double last_total_ms = 0.0, last_sweep_ms = 0.0;
  int last_n_sweeps = 0;
  std::vector<cudaEvent_t> sweep_ev;   // KPM_TIMING: one event after every sweep of a block
  std::vector<double> sweep_times;     // KPM_TIMING: per-sweep ms of the last call (all blocks)
};

static std::string g_create_err;

#define KPM_NCCL(call)                                                              \
  do {                                                                              \
    ncclResult_t r_ = (call);                                                       \
    if (r_ != ncclSuccess) {                                                        \
      ctx->err = std::string(#call) + ": " + ncclGetErrorString(r_);                \
      ctx->sticky = true;                                                           \
      return KPM_ENCCL;                                                             \
    }                                                                               \
  } while (0)

#define KPM_CUDA(call)                                                              \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess) {                                                        \
      ctx->err = std::string(#call) + ": " + cudaGetErrorString(e_);                \
      ctx->sticky = true;                                                           \
      return KPM_ECUDA;                                                             \
    }                                                                               \
  } while (0)

static bool load_stream_memops();

static kpm_status fail(kpm_ctx* ctx, kpm_status st, const std::string& msg) {
  ctx->err = msg;
  return st;
}

static int env_int(const char* name, int dflt) {
  const char* s = getenv(name);
  return s ? atoi(s) : dflt;
}

extern "C" kpm_status kpm_create(kpm_ctx** out, const kpm_options* opt) {
  if (!out) return KPM_EINVAL;
  *out = nullptr;
  if (!opt) {
    g_create_err = "opt is NULL";
    return KPM_EINVAL;
  }
  if (opt->nranks < 1 || opt->rank < 0 || opt->rank >= opt->nranks || (opt->nranks > 1 && !opt->nccl_unique_id)) {
    g_create_err = "bad nranks / rank / nccl_unique_id";
    return KPM_EINVAL;
  }
  const int C = opt->sell_C ? opt->sell_C : kC;
  const int sigma = opt->sell_sigma ? opt->sell_sigma : 1;
  if (C != kC || sigma < 1 || (sigma > 1 && sigma % C != 0)) {
    g_create_err = "unsupported SELL parameters (C must be 32, sigma 1 or a multiple of 32)";
    return KPM_EINVAL;
  }
  const bool virt = (opt->flags & KPM_VIRTUAL_RANKS) != 0;
  if (virt && (!opt->nccl_unique_id || static_cast<const kpm_vgroup*>(opt->nccl_unique_id)->P != opt->nranks)) {
    g_create_err = "KPM_VIRTUAL_RANKS needs nccl_unique_id = a kpm_vgroup of nranks ranks";
    return KPM_EINVAL;
  }
  if (virt && opt->nranks > 1) {
    // every virtual rank's stream may block in cuStreamWaitValue32 on another rank's flag; with
    // fewer hardware queues than streams two ranks could share one and deadlock
    const char* mc = getenv("CUDA_DEVICE_MAX_CONNECTIONS");
    if (!mc || atoi(mc) < 2 * opt->nranks) {
      g_create_err = "KPM_VIRTUAL_RANKS with nranks = " + std::to_string(opt->nranks) +
                     " needs CUDA_DEVICE_MAX_CONNECTIONS >= " + std::to_string(2 * opt->nranks) +
                     " in the environment before CUDA starts (one hardware queue per stream)";
      return KPM_EINVAL;
    }
  }
  if (opt->flags & ~(unsigned)(KPM_CHECK_HERMITIAN | KPM_DETERMINISTIC | KPM_TIMING | KPM_VIRTUAL_RANKS)) {
    g_create_err = "unknown kpm_options.flags bits";
    return KPM_EINVAL;
  }
  kpm_ctx* ctx = new kpm_ctx();
  ctx->opt = *opt;
  ctx->opt.sell_C = C;
  ctx->opt.sell_sigma = sigma;
  cudaError_t e = cudaSetDevice(opt->device);
  if (e == cudaSuccess && opt->cuda_stream) {
    ctx->stream = (cudaStream_t)opt->cuda_stream;
  } else if (e == cudaSuccess) {
    e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
    ctx->own_stream = (e == cudaSuccess);
  }
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, opt->device);
  for (int i = 0; i < 4 && e == cudaSuccess; ++i) e = cudaEventCreate(&ctx->ev[i]);
  if (e != cudaSuccess) {
    g_create_err = std::string("CUDA: ") + cudaGetErrorString(e);
    kpm_destroy(ctx);
    return KPM_ECUDA;
  }
  if (opt->nranks > 1) {
    ncclUniqueId id;
    ncclResult_t r = ncclSuccess;
    if (virt) {
      ctx->vg = static_cast<kpm_vgroup*>(const_cast<void*>(opt->nccl_unique_id));
    } else {
      std::memcpy(&id, opt->nccl_unique_id, sizeof(id));
      r = ncclCommInitRank(&ctx->comm, opt->nranks, id, opt->rank);
    }
    if (r == ncclSuccess) {
      e = cudaStreamCreateWithFlags(&ctx->comm_stream, cudaStreamNonBlocking);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_edge, cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_halo, cudaEventDisableTiming);
    }
    if (r != ncclSuccess || e != cudaSuccess) {
      g_create_err = r != ncclSuccess ? std::string("NCCL: ") + ncclGetErrorString(r)
                                      : std::string("CUDA: ") + cudaGetErrorString(e);
      kpm_destroy(ctx);
      return r != ncclSuccess ? KPM_ENCCL : KPM_ECUDA;
    }
  }
  if (opt->nranks > 1 && (e = preload_aux_kernels()) != cudaSuccess) {  // before any flag wait can exist
    g_create_err = std::string("CUDA: ") + cudaGetErrorString(e);
    kpm_destroy(ctx);
    return KPM_ECUDA;
  }
  ctx->variant_override = env_int("KPM_VARIANT", -1);
  ctx->grid_per_sm = std::max(0, env_int("KPM_GRID_PER_SM", 0));
  ctx->tile_stages = std::max(0, env_int("KPM_TILE_STAGES", 0));
  ctx->use_graph = env_int("KPM_GRAPH", 1) != 0;
  ctx->lcol_t = env_int("KPM_LCOL_T", 1) != 0;
  *out = ctx;
  return KPM_OK;
}

static void free_sell(DevSell& s);

extern "C" void kpm_destroy(kpm_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->opt.device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->graph_exec) cudaGraphExecDestroy(ctx->graph_exec);
  free_sell(ctx->sell);
  cudaFree(ctx->X0);
  cudaFree(ctx->X1);
  cudaFree(ctx->partials);
  cudaFree(ctx->eta_even);
  cudaFree(ctx->eta_odd);
  cudaFree(ctx->v0_dev);
  cudaFree(ctx->u_naive);
  cudaFree(ctx->stage_rp);
  cudaFree(ctx->stage_col);
  cudaFree(ctx->stage_val);
  ctx->build_ws.release();
  if (ctx->h_eta) cudaFreeHost(ctx->h_eta);
  for (int i = 0; i < 4; ++i)
    if (ctx->ev[i]) cudaEventDestroy(ctx->ev[i]);
  for (cudaEvent_t e : ctx->sweep_ev) cudaEventDestroy(e);
  cudaFree(ctx->edge_list);
  cudaFree(ctx->interior_list);
  cudaFree(ctx->halo_rows);
  for (auto& kv : ctx->ipc_open) cudaIpcCloseMemHandle(kv.second);
  cudaFree(ctx->order_list);
  cudaFree(ctx->bc_rec);
  cudaFree(ctx->bc_rec2);
  cudaFree(ctx->bc_map);
  cudaFree(ctx->bc_lcol);
  cudaFree(ctx->bc_fail);
  cudaFree(ctx->flags);
  if (ctx->comm) ncclCommDestroy(ctx->comm);
  if (ctx->comm_stream) cudaStreamDestroy(ctx->comm_stream);
  if (ctx->ev_edge) cudaEventDestroy(ctx->ev_edge);
  if (ctx->ev_halo) cudaEventDestroy(ctx->ev_halo);
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

extern "C" kpm_status kpm_vgroup_create(int nranks, kpm_vgroup** out) {
  if (!out || nranks < 1) return KPM_EINVAL;
  kpm_vgroup* g = new kpm_vgroup();
  g->P = nranks;
  g->slot.resize(nranks);
  *out = g;
  return KPM_OK;
}

extern "C" void kpm_vgroup_destroy(kpm_vgroup* g) { delete g; }

extern "C" kpm_status kpm_get_unique_id(void* out) {
  if (!out) return KPM_EINVAL;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return KPM_ENCCL;
  std::memcpy(out, &id, sizeof(id));
  return KPM_OK;
}

static kpm_status wait_stream(kpm_ctx* ctx, cudaStream_t str);

// Small host<->device collective helpers for the setup (synchronous, compute stream).
static kpm_status allgather_i64(kpm_ctx* ctx, const std::vector<int64_t>& mine, std::vector<int64_t>& all) {
  const size_t n = mine.size(), P = (size_t)ctx->opt.nranks;
  KPM_TRACE_LINE(ctx->opt.rank, "allgather of %zu words", n);
  if (ctx->vg) {
    all.clear();
    for (const auto& v : ctx->vg->allgatherv(ctx->opt.rank, mine)) all.insert(all.end(), v.begin(), v.end());
    return KPM_OK;
  }
  int64_t* d = nullptr;
  KPM_CUDA(cudaMalloc(&d, sizeof(int64_t) * n * (P + 1)));
  KPM_CUDA(cudaMemcpy(d, mine.data(), sizeof(int64_t) * n, cudaMemcpyHostToDevice));
  KPM_NCCL(ncclAllGather(d, d + n, n, ncclInt64, ctx->comm, ctx->stream));
  all.resize(n * P);
  KPM_CUDA(cudaMemcpyAsync(all.data(), d + n, sizeof(int64_t) * n * P, cudaMemcpyDeviceToHost, ctx->stream));
  const kpm_status ws = wait_stream(ctx, ctx->stream);
  if (ws != KPM_OK) return ws;
  KPM_CUDA(cudaFree(d));
  return KPM_OK;
}

// Multi-rank: every rank learns whether any rank failed a local step (allocation, validation,
// plan) before the next collective, so that no rank is left waiting in NCCL or on a halo flag.
// Returns this rank's status, or KPM_EINVAL/the other rank's status if only another rank failed.
static kpm_status agree(kpm_ctx* ctx, kpm_status mine) {
  if (ctx->opt.nranks == 1) return mine;
  std::vector<int64_t> all;
  const std::string saved = ctx->err;
  const kpm_status st = allgather_i64(ctx, {(int64_t)mine}, all);
  if (st != KPM_OK) return st;
  ctx->err = saved;
  if (mine != KPM_OK) return mine;
  for (size_t q = 0; q < all.size(); ++q)
    if (all[q] != KPM_OK && all[q] != KPM_WDIVERGED)
      return fail(ctx, (kpm_status)all[q], "rank " + std::to_string(q) + " failed with status " + std::to_string(all[q]));
  return KPM_OK;
}

extern "C" const char* kpm_last_error(const kpm_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_create_err.c_str();
}

static void free_sell(DevSell& s) {
  cudaFree(s.val);
  cudaFree(s.col);
  cudaFree(s.cptr);
  cudaFree(s.perm_buf);
  cudaFree(s.lcol);
  cudaFree(s.nruns);
  cudaFree(s.runs);
  for (int i = 0; i < 12; ++i) cudaFree(s.rec[i]);
  s = DevSell();
}

// Forget the matrix but keep the device buffers for the next one (grow-only reuse).
static void reset_sell(DevSell& s) {
  DevSell k;
  k.val = s.val, k.col = s.col, k.cptr = s.cptr, k.perm_buf = s.perm_buf, k.lcol = s.lcol, k.nruns = s.nruns, k.runs = s.runs;
  k.val_cap = s.val_cap, k.col_cap = s.col_cap, k.cptr_cap = s.cptr_cap, k.perm_cap = s.perm_cap;
  k.lcol_cap = s.lcol_cap, k.nruns_cap = s.nruns_cap, k.runs_cap = s.runs_cap;
  for (int i = 0; i < 12; ++i) {
    k.rec[i] = s.rec[i];
    k.rec_cap[i] = s.rec_cap[i];
  }
  s = k;
}

// Halo exchange plan (collective): receive runs from the halo list, requests to the owners,
// send runs from the requests, edge / interior chunk split (halo_plan.h).
static kpm_status plan_exchange(kpm_ctx* ctx, const std::vector<int64_t>& halo, int64_t n_pad,
                                const std::vector<int32_t>& perm, const std::vector<char>& reads_halo) {
  const int P = ctx->opt.nranks, me = ctx->opt.rank;
  const int64_t row_begin = ctx->row_begins[me], row_end = ctx->row_begins[me + 1];
  ctx->recv_runs = plan_recv_runs(halo, ctx->row_begins);
  // requests: per owner q the (gfirst, count) pairs, in slot order
  std::vector<std::vector<int64_t>> req(P);
  for (const RecvRun& r : ctx->recv_runs) {  // (first global row, count, first halo slot)
    req[r.peer].push_back(r.gfirst);
    req[r.peer].push_back(r.count);
    req[r.peer].push_back(r.slot);
  }
  std::vector<int64_t> counts(P), all;
  for (int q = 0; q < P; ++q) counts[q] = (int64_t)req[q].size();
  kpm_status st = allgather_i64(ctx, counts, all);  // all[p*P + q] = #int64 p requests from q
  if (st != KPM_OK) return st;
  int64_t tot_out = 0, tot_in = 0;
  for (int q = 0; q < P; ++q) tot_out += all[(size_t)me * P + q];
  for (int p = 0; p < P; ++p) tot_in += all[(size_t)p * P + me];
  std::vector<int64_t> incoming(tot_in);
  if (ctx->vg) {  // virtual ranks: every rank sees every rank's requests, keeps those sent to it
    std::vector<int64_t> flat;
    for (int q = 0; q < P; ++q) flat.insert(flat.end(), req[q].begin(), req[q].end());
    const auto got = ctx->vg->allgatherv(me, flat);
    int64_t in = 0;
    for (int p = 0; p < P; ++p) {
      int64_t o = 0;
      for (int q = 0; q < me; ++q) o += all[(size_t)p * P + q];
      for (int64_t i = 0; i < all[(size_t)p * P + me]; ++i) incoming[in++] = got[p][o + i];
    }
  } else {
  int64_t* dbuf = nullptr;
  KPM_CUDA(cudaMalloc(&dbuf, sizeof(int64_t) * std::max<int64_t>(1, tot_out + tot_in)));
  std::vector<int64_t> flat;
  for (int q = 0; q < P; ++q) flat.insert(flat.end(), req[q].begin(), req[q].end());
  if (tot_out) KPM_CUDA(cudaMemcpy(dbuf, flat.data(), sizeof(int64_t) * tot_out, cudaMemcpyHostToDevice));
  KPM_NCCL(ncclGroupStart());
  int64_t o = 0, in = tot_out;
  for (int q = 0; q < P; ++q) {
    const int64_t n = all[(size_t)me * P + q];
    if (n) KPM_NCCL(ncclSend(dbuf + o, n, ncclInt64, q, ctx->comm, ctx->stream));
    o += n;
  }
  for (int p = 0; p < P; ++p) {
    const int64_t n = all[(size_t)p * P + me];
    if (n) KPM_NCCL(ncclRecv(dbuf + in, n, ncclInt64, p, ctx->comm, ctx->stream));
    in += n;
  }
  KPM_NCCL(ncclGroupEnd());
  if (tot_in)
    KPM_CUDA(cudaMemcpyAsync(incoming.data(), dbuf + tot_out, sizeof(int64_t) * tot_in, cudaMemcpyDeviceToHost,
                             ctx->stream));
  KPM_CUDA(cudaStreamSynchronize(ctx->stream));
  KPM_CUDA(cudaFree(dbuf));
  }
  int64_t off = 0;
  for (int p = 0; p < P; ++p) {
    const int64_t n = all[(size_t)p * P + me];
    std::vector<int64_t> rq, slots;
    for (int64_t i = off; i + 2 < off + n; i += 3) {
      rq.push_back(incoming[i]);
      rq.push_back(incoming[i + 1]);
      slots.push_back(incoming[i + 2]);
    }
    off += n;
    const size_t first = ctx->send_runs.size();
    if (!plan_send_runs(p, rq, row_begin, row_end, perm, ctx->send_runs))
      return fail(ctx, KPM_EINVAL, "halo request does not map to contiguous local rows");
    for (size_t i = first; i < ctx->send_runs.size(); ++i) ctx->send_runs[i].peer_slot = slots[i - first];
  }
  std::vector<int64_t> edge, interior;
  plan_edge_chunks((int64_t)ctx->cptr_h.size() - 1, reads_halo, kC, ctx->send_runs, edge, interior);
  ctx->edge_flag.assign(ctx->cptr_h.size() - 1, 0);
  for (int64_t c : edge) ctx->edge_flag[c] = 1;
  KPM_CUDA(cudaMalloc(&ctx->edge_list, sizeof(int64_t) * std::max<size_t>(1, edge.size())));
  KPM_CUDA(cudaMalloc(&ctx->interior_list, sizeof(int64_t) * std::max<size_t>(1, interior.size())));
  KPM_CUDA(cudaMalloc(&ctx->halo_rows, sizeof(int64_t) * std::max<size_t>(1, halo.size())));
  if (!halo.empty())
    KPM_CUDA(cudaMemcpy(ctx->halo_rows, halo.data(), sizeof(int64_t) * halo.size(), cudaMemcpyHostToDevice));
  return KPM_OK;
}

// Install a chunk order (empty = storage order) as the work lists of the sweep launches: single
// rank -> order_list (NULL for storage order); multi-rank -> the edge and the interior list, each
// in that order.  id names it (see kpm_ctx::order_id) so that repeated requests are free.
static kpm_status install_order(kpm_ctx* ctx, const std::vector<int64_t>& ord_in, int64_t id) {
  if (id == ctx->order_id) return KPM_OK;
  const int64_t n = ctx->sell.n_chunks;
  cudaFree(ctx->order_list);
  ctx->order_list = nullptr;
  ctx->order_id = -3;
  ++ctx->order_gen;
  if (ctx->opt.nranks == 1) {
    if (!ord_in.empty()) {
      KPM_CUDA(cudaMalloc(&ctx->order_list, sizeof(int64_t) * n));
      KPM_CUDA(cudaMemcpy(ctx->order_list, ord_in.data(), sizeof(int64_t) * n, cudaMemcpyHostToDevice));
    }
    ctx->order_id = id;
    return KPM_OK;
  }
  std::vector<int64_t> edge, interior;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t c = ord_in.empty() ? i : ord_in[i];
    (ctx->edge_flag[c] ? edge : interior).push_back(c);
  }
  ctx->n_edge = (int64_t)edge.size();
  ctx->n_interior = (int64_t)interior.size();
  if (!edge.empty())
    KPM_CUDA(cudaMemcpy(ctx->edge_list, edge.data(), sizeof(int64_t) * edge.size(), cudaMemcpyHostToDevice));
  if (!interior.empty())
    KPM_CUDA(cudaMemcpy(ctx->interior_list, interior.data(), sizeof(int64_t) * interior.size(), cudaMemcpyHostToDevice));
  ctx->order_id = id;
  return KPM_OK;
}

// Block-neighbour lists of the chunks (chunk_order.cpp), from the tiled feed's run lists.
static kpm_status ensure_adjacency(kpm_ctx* ctx) {
  if (ctx->adj_state != 0) return KPM_OK;
  const DevSell& s = ctx->sell;
  ctx->adj_state = -1;
  if (!s.tiles_ok || s.n_chunks < 1) return KPM_OK;
  std::vector<int> nr(s.n_chunks), rr((size_t)2 * kMaxRuns * s.n_chunks);
  KPM_CUDA(cudaMemcpy(nr.data(), s.nruns, sizeof(int) * nr.size(), cudaMemcpyDeviceToHost));
  KPM_CUDA(cudaMemcpy(rr.data(), s.runs, sizeof(int) * rr.size(), cudaMemcpyDeviceToHost));
  block_neighbours(s.n_chunks, nr.data(), rr.data(), kMaxRuns, kC, ctx->adj_ptr, ctx->adj);
  ctx->adj_maxoff = typical_block_offset(s.n_chunks, ctx->adj_ptr, ctx->adj);
  ctx->adj_state = 1;
  return KPM_OK;
}

// The chunk order a launch of `grid` CTAs runs: the caller's (kpm_set_chunk_order), else the
// line walk when want_lines (block-cache kernels; any kernel whose storage-order neighbour
// window exceeds 32 MB), else storage order.
static kpm_status ensure_order(kpm_ctx* ctx, int64_t grid, bool bc_kernel, int Rk, int width) {
  if (ctx->order_user) return install_order(ctx, ctx->order_h, -1);
  kpm_status st = ensure_adjacency(ctx);
  if (st != KPM_OK) return st;
  // V rows a storage-order sweep must keep in L2 between a row's first and last use: both sides
  // of the reuse distance (TI: two x-planes; C4 at R = 32: 65.5 MB, C3: 16.4 MB)
  const bool big_window = ctx->adj_state == 1 && 2.0 * (double)ctx->adj_maxoff * kC * Rk * 16.0 > 32e6;
  if (ctx->adj_state == 1 && (bc_kernel || big_window) && env_int("KPM_AUTO_ORDER", 1)) {
    const int64_t id = grid * 4 + width;
    std::vector<int64_t>& o = ctx->auto_order[id];
    if (o.empty()) {
      std::vector<char> skip;
      if (ctx->opt.nranks > 1) skip = ctx->edge_flag;
      o = line_order(ctx->sell.n_chunks, ctx->adj_ptr, ctx->adj, grid, skip, width);
    }
    return install_order(ctx, o, id);
  }
  return install_order(ctx, {}, 0);
}

extern "C" kpm_status kpm_set_chunk_order(kpm_ctx* ctx, const int64_t* order, int64_t n) {
  if (!ctx) return KPM_EINVAL;
  if (ctx->sticky) return fail(ctx, KPM_ESTATE, "context has a sticky CUDA/NCCL error: " + ctx->err);
  if (!ctx->have_matrix) return fail(ctx, KPM_ESTATE, "kpm_set_matrix has not been called");
  KPM_CUDA(cudaSetDevice(ctx->opt.device));
  if (order) {
    if (n != ctx->sell.n_chunks) return fail(ctx, KPM_EINVAL, "order must list every chunk once");
    std::vector<char> seen(n, 0);
    for (int64_t i = 0; i < n; ++i) {
      if (order[i] < 0 || order[i] >= n || seen[order[i]]) return fail(ctx, KPM_EINVAL, "order is not a permutation");
      seen[order[i]] = 1;
    }
  }
  ctx->order_user = order != nullptr;
  ctx->order_h.assign(order, order + (order ? n : 0));
  ctx->order_id = -3;  // (re)installed by the next kpm_moments*
  ++ctx->matrix_gen;   // the kernel choice and its block-cache plan depend on the order
  return KPM_OK;
}

// After a sweep: owners' new rows of X -> the neighbours' halo slots of X (grouped NCCL P2P).
static kpm_status exchange_halo(kpm_ctx* ctx, double2* X, int Rk, cudaStream_t s) {
  const int64_t n_pad = ctx->sell.n_pad;
  if (ctx->vg) {  // virtual ranks: pull the halo rows from the owners' buffers (sigma = 1 positions)
    KPM_CUDA(cudaStreamSynchronize(s));
    const auto xs = ctx->vg->allgatherv(ctx->opt.rank, {(int64_t)X});  // everyone's rows are final
    for (const RecvRun& r : ctx->recv_runs) {
      const double2* src = reinterpret_cast<const double2*>(xs[r.peer][0]) + (r.gfirst - ctx->row_begins[r.peer]) * Rk;
      KPM_CUDA(cudaMemcpyAsync(X + (n_pad + r.slot) * Rk, src, sizeof(double2) * r.count * Rk, cudaMemcpyDeviceToDevice, s));
    }
    KPM_CUDA(cudaStreamSynchronize(s));
    ctx->vg->allgatherv(ctx->opt.rank, {});  // nobody overwrites its rows before all copies are done
    return KPM_OK;
  }
  KPM_NCCL(ncclGroupStart());
  for (const SendRun& r : ctx->send_runs)
    KPM_NCCL(ncclSend(X + r.pos * Rk, (size_t)r.count * Rk * 2, ncclDouble, r.peer, ctx->comm, s));
  for (const RecvRun& r : ctx->recv_runs)
    KPM_NCCL(ncclRecv(X + (n_pad + r.slot) * Rk, (size_t)r.count * Rk * 2, ncclDouble, r.peer, ctx->comm, s));
  KPM_NCCL(ncclGroupEnd());
  return KPM_OK;
}

extern "C" kpm_status kpm_set_matrix(kpm_ctx* ctx, const kpm_csr* H, double a, double b) {
  if (!ctx) return KPM_EINVAL;
  if (ctx->sticky) return fail(ctx, KPM_ESTATE, "context has a sticky CUDA/NCCL error: " + ctx->err);
  if (!H || !H->row_ptr || !H->col || !H->val) return fail(ctx, KPM_EINVAL, "NULL matrix pointer");
  if (!(a > 0.0) || !std::isfinite(a) || !std::isfinite(b)) return fail(ctx, KPM_EINVAL, "need finite a > 0 and finite b");
  if (H->mem != KPM_MEM_HOST && H->mem != KPM_MEM_DEVICE) return fail(ctx, KPM_EINVAL, "bad mem kind");
  const int64_t n_loc = H->row_end - H->row_begin;
  if (H->n_global < 1 || H->row_begin < 0 || n_loc < 1 || H->row_end > H->n_global)
    return fail(ctx, KPM_EINVAL, "bad row range");
  if (ctx->opt.nranks == 1 && (H->row_begin != 0 || H->row_end != H->n_global))
    return fail(ctx, KPM_EINVAL, "single rank must own all rows");
  KPM_CUDA(cudaSetDevice(ctx->opt.device));
  std::vector<int64_t> row_begins{0, H->n_global};
  if (ctx->opt.nranks > 1) {  // collective: every rank's row range, must tile [0, n_global) in rank order
    if (ctx->opt.sell_sigma != 1) return fail(ctx, KPM_EINVAL, "nranks > 1 needs sell_sigma = 1");
    std::vector<int64_t> all;
    kpm_status st0 = allgather_i64(ctx, {H->row_begin, H->row_end, H->n_global}, all);
    if (st0 != KPM_OK) return st0;
    row_begins.assign(1, 0);
    for (int q = 0; q < ctx->opt.nranks; ++q) {
      if (all[3 * q] != row_begins.back() || all[3 * q + 2] != H->n_global)
        return fail(ctx, KPM_EINVAL, "row ranges do not tile [0, n_global) in rank order");
      row_begins.push_back(all[3 * q + 1]);
    }
    if (row_begins.back() != H->n_global) return fail(ctx, KPM_EINVAL, "row ranges do not cover n_global");
  }

  if (ctx->opt.flags & KPM_CHECK_HERMITIAN) {
    std::vector<int64_t> rp_h, col_h;
    std::vector<double> val_h;
    const int64_t *rp = H->row_ptr, *col = H->col;
    const double* val = H->val;
    if (H->mem == KPM_MEM_DEVICE) {
      rp_h.resize(n_loc + 1);
      KPM_CUDA(cudaMemcpy(rp_h.data(), H->row_ptr, sizeof(int64_t) * (n_loc + 1), cudaMemcpyDeviceToHost));
      if (rp_h[n_loc] < 0) return fail(ctx, KPM_EINVAL, "malformed row_ptr");
      col_h.resize(rp_h[n_loc]);
      val_h.resize(2 * rp_h[n_loc]);
      KPM_CUDA(cudaMemcpy(col_h.data(), H->col, sizeof(int64_t) * col_h.size(), cudaMemcpyDeviceToHost));
      KPM_CUDA(cudaMemcpy(val_h.data(), H->val, sizeof(double) * val_h.size(), cudaMemcpyDeviceToHost));
      rp = rp_h.data(), col = col_h.data(), val = val_h.data();
    }
    std::string herr;
    const int hs = check_hermitian(rp, col, val, n_loc, H->row_begin, H->row_end, H->n_global, 1e-12, herr);
    if (hs) fail(ctx, (kpm_status)hs, herr);
    kpm_status ag = agree(ctx, (kpm_status)hs);
    if (ag != KPM_OK) return ag;
  } else if (ctx->opt.nranks > 1) {
    kpm_status ag = agree(ctx, KPM_OK);  // keep the collective sequence identical on every rank
    if (ag != KPM_OK) return ag;
  }

  reset_sell(ctx->sell);
  ctx->have_matrix = false;
  DevSell& d = ctx->sell;
  std::vector<int64_t> halo;       // global ids of the halo slots
  std::vector<int32_t> perm_h;     // host perm (empty = identity)
  std::vector<char> reads_halo;    // per chunk, multi-rank planning
  auto build = [&]() -> kpm_status {

    // sigma = 1 builds on the device (sell_device.cu); a host CSR is staged to the device first
    // (one H2D copy, then the same kernels), unless that does not fit or KPM_HOST_BUILD=1.
    bool dev_build = ctx->opt.sell_sigma == 1 && env_int("KPM_HOST_BUILD", 0) == 0;
    int64_t* st_rp = nullptr;
    int64_t* st_col = nullptr;
    double2* st_val = nullptr;
    if (dev_build && H->mem == KPM_MEM_HOST) {
      const int64_t nnz = H->row_ptr[n_loc];
      if (H->row_ptr[0] != 0 || nnz < 0) return fail(ctx, KPM_EINVAL, "malformed row_ptr");
      if (reserve((void**)&ctx->stage_rp, &ctx->stage_rp_cap, sizeof(int64_t) * (n_loc + 1)) != cudaSuccess ||
          reserve((void**)&ctx->stage_col, &ctx->stage_col_cap, sizeof(int64_t) * nnz) != cudaSuccess ||
          reserve((void**)&ctx->stage_val, &ctx->stage_val_cap, sizeof(double2) * nnz) != cudaSuccess) {
        cudaGetLastError();
        dev_build = false;  // not enough device memory for the staging copy: host build
      } else {
        st_rp = ctx->stage_rp;
        st_col = ctx->stage_col;
        st_val = ctx->stage_val;
        KPM_CUDA(cudaMemcpyAsync(st_rp, H->row_ptr, sizeof(int64_t) * (n_loc + 1), cudaMemcpyHostToDevice, ctx->stream));
        KPM_CUDA(cudaMemcpyAsync(st_col, H->col, sizeof(int64_t) * nnz, cudaMemcpyHostToDevice, ctx->stream));
        KPM_CUDA(cudaMemcpyAsync(st_val, H->val, sizeof(double2) * nnz, cudaMemcpyHostToDevice, ctx->stream));
      }
    }
    if (dev_build) {
      // device build: the CSR never leaves the GPU
      DeviceBuild db;
      std::string berr;
      const bool staged = st_rp != nullptr;
      const int st = build_sell_device(staged ? st_rp : H->row_ptr, staged ? st_col : H->col,
                                       staged ? st_val : reinterpret_cast<const double2*>(H->val), n_loc,
                                       H->row_begin, H->row_end, H->n_global, d, db, ctx->build_ws, berr, ctx->stream);
      if (staged) cudaStreamSynchronize(ctx->stream);
      if (st) {
        reset_sell(ctx->sell);
        cudaGetLastError();
        if (st == 5) {
          ctx->sticky = true;
          return fail(ctx, KPM_ECUDA, berr);
        }
        return fail(ctx, (kpm_status)st, berr);
      }
      halo = std::move(db.halo);
      reads_halo = std::move(db.reads_halo);
      ctx->cptr_h = std::move(db.cptr);
    } else {
      // host build (device input is staged through the host)
      std::vector<int64_t> rp_h, col_h;
      std::vector<double> val_h;
      const int64_t* rp = H->row_ptr;
      const int64_t* col = H->col;
      const double* val = H->val;
      if (H->mem == KPM_MEM_DEVICE) {
        rp_h.resize(n_loc + 1);
        KPM_CUDA(cudaMemcpy(rp_h.data(), H->row_ptr, sizeof(int64_t) * (n_loc + 1), cudaMemcpyDeviceToHost));
        const int64_t nnz = rp_h[n_loc];
        if (nnz < 0) return fail(ctx, KPM_EINVAL, "malformed row_ptr");
        col_h.resize(nnz);
        val_h.resize(2 * nnz);
        KPM_CUDA(cudaMemcpy(col_h.data(), H->col, sizeof(int64_t) * nnz, cudaMemcpyDeviceToHost));
        KPM_CUDA(cudaMemcpy(val_h.data(), H->val, sizeof(double) * 2 * nnz, cudaMemcpyDeviceToHost));
        rp = rp_h.data();
        col = col_h.data();
        val = val_h.data();
      }
      if (rp[0] != 0) return fail(ctx, KPM_EINVAL, "row_ptr[0] != 0");
      for (int64_t i = 0; i < n_loc; ++i)
        if (rp[i + 1] < rp[i]) return fail(ctx, KPM_EINVAL, "row_ptr not non-decreasing");
      const int64_t nnz = rp[n_loc];
      for (int64_t k = 0; k < nnz; ++k) {
        if (col[k] < 0 || col[k] >= H->n_global) return fail(ctx, KPM_ERANGE, "column outside [0, n_global)");
        if (!std::isfinite(val[2 * k]) || !std::isfinite(val[2 * k + 1])) return fail(ctx, KPM_EINVAL, "non-finite value");
      }
      HostSell hs;
      std::string berr;
      int st = build_sell_host(rp, col, val, n_loc, H->row_begin, H->row_end, ctx->opt.sell_C, ctx->opt.sell_sigma, hs,
                               berr);
      if (st) return fail(ctx, (kpm_status)st, berr);
      d.n_loc = hs.n_loc;
      d.n_pad = hs.n_pad;
      d.n_chunks = hs.n_chunks;
      d.n_slots = hs.cptr[hs.n_chunks];
      d.n_halo = hs.n_halo;
      d.max_width = 0;
      for (int64_t c = 0; c < hs.n_chunks; ++c) d.max_width = std::max(d.max_width, (hs.cptr[c + 1] - hs.cptr[c]) / hs.C);
      cudaError_t e = reserve((void**)&d.val, &d.val_cap, sizeof(double2) * d.n_slots);
      if (e == cudaSuccess) e = reserve((void**)&d.col, &d.col_cap, sizeof(int) * d.n_slots);
      if (e == cudaSuccess) e = reserve((void**)&d.cptr, &d.cptr_cap, sizeof(int64_t) * (d.n_chunks + 1));
      if (e == cudaSuccess && hs.sigma > 1) e = reserve((void**)&d.perm_buf, &d.perm_cap, sizeof(int) * d.n_loc);
      if (e == cudaSuccess && hs.sigma > 1) d.perm = d.perm_buf;
      if (e != cudaSuccess) {
        reset_sell(ctx->sell);
        cudaGetLastError();
        return fail(ctx, KPM_ENOMEM, std::string("device allocation for the matrix failed: ") + cudaGetErrorString(e));
      }
      KPM_CUDA(cudaMemcpy(d.val, hs.val.data(), sizeof(double2) * d.n_slots, cudaMemcpyHostToDevice));
      KPM_CUDA(cudaMemcpy(d.col, hs.col.data(), sizeof(int) * d.n_slots, cudaMemcpyHostToDevice));
      KPM_CUDA(cudaMemcpy(d.cptr, hs.cptr.data(), sizeof(int64_t) * (d.n_chunks + 1), cudaMemcpyHostToDevice));
      if (hs.sigma > 1) {
        KPM_CUDA(cudaMemcpy(d.perm, hs.perm.data(), sizeof(int) * d.n_loc, cudaMemcpyHostToDevice));
        perm_h = hs.perm;
      }
      // gather plan of the tiled feed: lcol + fixed-capacity run lists (records per R on use)
      HostTiles t;
      build_tiles_host(hs, t);
      d.tiles_ok = t.ok && t.max_runs <= kMaxRuns;
      d.max_other = t.max_other;
      d.max_runs = t.max_runs;
      if (d.tiles_ok) {
        std::vector<int> nr(d.n_chunks), rr((size_t)2 * kMaxRuns * d.n_chunks, 0);
        for (int64_t c = 0; c < d.n_chunks; ++c) {
          nr[c] = (int)(t.run_ptr[c + 1] - t.run_ptr[c]);
          for (int64_t k = t.run_ptr[c]; k < t.run_ptr[c + 1]; ++k) {
            rr[c * 2 * kMaxRuns + 2 * (k - t.run_ptr[c])] = t.runs[2 * k];
            rr[c * 2 * kMaxRuns + 2 * (k - t.run_ptr[c]) + 1] = t.runs[2 * k + 1];
          }
        }
        if (reserve((void**)&d.lcol, &d.lcol_cap, sizeof(uint16_t) * t.lcol.size()) != cudaSuccess ||
            reserve((void**)&d.nruns, &d.nruns_cap, sizeof(int) * nr.size()) != cudaSuccess ||
            reserve((void**)&d.runs, &d.runs_cap, sizeof(int) * rr.size()) != cudaSuccess) {
          cudaGetLastError();
          d.tiles_ok = false;  // the other feeds still work
        } else {
          KPM_CUDA(cudaMemcpy(d.lcol, t.lcol.data(), sizeof(uint16_t) * t.lcol.size(), cudaMemcpyHostToDevice));
          KPM_CUDA(cudaMemcpy(d.nruns, nr.data(), sizeof(int) * nr.size(), cudaMemcpyHostToDevice));
          KPM_CUDA(cudaMemcpy(d.runs, rr.data(), sizeof(int) * rr.size(), cudaMemcpyHostToDevice));
        }
      }
      halo = hs.halo;
      ctx->cptr_h = hs.cptr;
      if (!halo.empty()) {
        reads_halo.assign(d.n_chunks, 0);
        for (int64_t c = 0; c < d.n_chunks; ++c)
          for (int64_t k = hs.cptr[c]; k < hs.cptr[c + 1]; ++k)
            if (hs.col[k] >= hs.n_pad) {
              reads_halo[c] = 1;
              break;
            }
      }
    }
    KPM_CUDA(cudaStreamSynchronize(ctx->stream));
    return KPM_OK;
  };
  {
    const kpm_status bst = agree(ctx, build());
    if (bst != KPM_OK) {
      if (!ctx->sticky) reset_sell(ctx->sell);
      return bst;
    }
  }
  if (ctx->opt.nranks == 1 && d.n_halo != 0) return fail(ctx, KPM_EINVAL, "internal: halo on a single rank");
  ctx->halo = halo;
  ctx->row_begins = row_begins;
  ctx->recv_runs.clear();
  ctx->send_runs.clear();
  cudaFree(ctx->edge_list);
  cudaFree(ctx->interior_list);
  cudaFree(ctx->halo_rows);
  ctx->edge_list = ctx->interior_list = ctx->halo_rows = nullptr;
  ctx->n_edge = 0;
  ctx->n_interior = d.n_chunks;
  cudaFree(ctx->order_list);
  ctx->order_list = nullptr;
  ctx->fused = false;
  ctx->fused_ready = false;
  ctx->order_h.clear();
  ctx->order_user = false;
  ctx->order_id = -3;
  ctx->auto_order.clear();
  ctx->adj_state = 0;
  ctx->adj_ptr.clear();
  ctx->adj.clear();
  if (ctx->opt.nranks > 1) {
    kpm_status st1 = plan_exchange(ctx, halo, d.n_pad, perm_h, reads_halo);
    if (st1 != KPM_OK) return st1;
    if ((st1 = install_order(ctx, {}, 0)) != KPM_OK) return st1;
    const char* mode = getenv("KPM_HALO");
    ctx->fused = (ctx->vg || !(mode && std::string(mode) == "nccl")) && ctx->send_runs.size() <= (size_t)kMaxPeerRuns &&
                 load_stream_memops();
    if (ctx->fused) {  // Hermitian => symmetric pattern => I receive from exactly the ranks I send to
      std::vector<int> d, r;
      for (const SendRun& x : ctx->send_runs) d.push_back(x.peer);
      for (const RecvRun& x : ctx->recv_runs) r.push_back(x.peer);
      std::sort(d.begin(), d.end());
      d.erase(std::unique(d.begin(), d.end()), d.end());
      std::sort(r.begin(), r.end());
      r.erase(std::unique(r.begin(), r.end()), r.end());
      ctx->dest_peers = d;
      ctx->src_peers = r;
      if (d != r) ctx->fused = false;
    }
    // the mode must agree on all ranks
    std::vector<int64_t> all;
    kpm_status st2 = allgather_i64(ctx, {ctx->fused ? 1 : 0}, all);
    if (st2 != KPM_OK) return st2;
    for (int64_t v : all) ctx->fused = ctx->fused && v == 1;
    if (ctx->fused && !ctx->flags) {
      KPM_CUDA(cudaMalloc(&ctx->flags, sizeof(int32_t) * ctx->opt.nranks));
      KPM_CUDA(cudaMemset(ctx->flags, 0, sizeof(int32_t) * ctx->opt.nranks));
      ctx->epoch = 0;
    }
  }
  ++ctx->matrix_gen;
  ctx->n_global = H->n_global;
  ctx->row_begin = H->row_begin;
  ctx->row_end = H->row_end;
  ctx->a = a;
  ctx->b = b;
  ctx->have_matrix = true;
  return KPM_OK;
}

static int block_width(int r) {
  int w = 1;
  while (w < r) w <<= 1;
  return w;
}

static kpm_status ensure(kpm_ctx* ctx, void** p, size_t* cap, size_t need, size_t elsize) {
  if (*cap >= need) return KPM_OK;
  cudaFree(*p);
  *p = nullptr;
  *cap = 0;
  cudaError_t e = cudaMalloc(p, need * elsize);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(ctx, KPM_ENOMEM, std::string("device allocation failed: ") + cudaGetErrorString(e));
  }
  *cap = need;
  return KPM_OK;
}

// Driver stream memory operations (wait / write a 32-bit flag), resolved at run time through
// the runtime's entry-point query, so the library needs no link-time libcuda.
typedef CUresult (*WaitValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*WriteValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
static WaitValue32Fn g_wait_value32 = nullptr;
static WriteValue32Fn g_write_value32 = nullptr;

static bool load_stream_memops() {
  if (g_wait_value32 && g_write_value32) return true;
  cudaDriverEntryPointQueryResult q1, q2;
  void *f1 = nullptr, *f2 = nullptr;
  if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &f1, cudaEnableDefault, &q1) != cudaSuccess ||
      q1 != cudaDriverEntryPointSuccess)
    return false;
  if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &f2, cudaEnableDefault, &q2) != cudaSuccess ||
      q2 != cudaDriverEntryPointSuccess)
    return false;
  g_wait_value32 = reinterpret_cast<WaitValue32Fn>(f1);
  g_write_value32 = reinterpret_cast<WriteValue32Fn>(f2);
  return true;
}

// Fused exchange setup (collective): every rank publishes CUDA IPC handles of X0, X1 and
// its flag array plus its n_pad; each rank maps the buffers of the peers it sends to and
// precomputes, per send run, the destination address of the run in the peer's halo slots.
static kpm_status setup_fused(kpm_ctx* ctx, int Rk) {
  if (ctx->vg) {  // virtual ranks: the peers' buffers are on this device, plain pointers
    std::vector<int64_t> all;
    kpm_status st = allgather_i64(ctx, {(int64_t)ctx->X0, (int64_t)ctx->X1, (int64_t)ctx->flags, ctx->sell.n_pad}, all);
    if (st != KPM_OK) return st;
    ctx->dst_x.clear();
    for (const SendRun& r : ctx->send_runs) {
      const int64_t off = (all[4 * r.peer + 3] + r.peer_slot) * Rk;
      ctx->dst_x.push_back({reinterpret_cast<double2*>(all[4 * r.peer]) + off, reinterpret_cast<double2*>(all[4 * r.peer + 1]) + off});
    }
    ctx->dst_flag.clear();
    for (int q : ctx->dest_peers) ctx->dst_flag.push_back(reinterpret_cast<int32_t*>(all[4 * q + 2]) + ctx->opt.rank);
    ctx->fused_ready = true;
    ctx->fused_rk = Rk;
    return KPM_OK;
  }
  struct Pub {
    cudaIpcMemHandle_t x0, x1, fl;
    int64_t n_pad;
  };
  static_assert(sizeof(Pub) % 8 == 0, "Pub must be int64-aligned");
  Pub mine;
  KPM_CUDA(cudaIpcGetMemHandle(&mine.x0, ctx->X0));
  KPM_CUDA(cudaIpcGetMemHandle(&mine.x1, ctx->X1));
  KPM_CUDA(cudaIpcGetMemHandle(&mine.fl, ctx->flags));
  mine.n_pad = ctx->sell.n_pad;
  std::vector<int64_t> v(sizeof(Pub) / 8), all;
  std::memcpy(v.data(), &mine, sizeof(Pub));
  kpm_status st = allgather_i64(ctx, v, all);
  if (st != KPM_OK) return st;
  const int P = ctx->opt.nranks;
  std::vector<Pub> pubs(P);
  for (int q = 0; q < P; ++q) std::memcpy(&pubs[q], all.data() + (size_t)q * v.size(), sizeof(Pub));
  auto open = [&](const cudaIpcMemHandle_t& h, void** out) -> kpm_status {
    const std::string key(reinterpret_cast<const char*>(&h), sizeof(h));
    auto it = ctx->ipc_open.find(key);
    if (it == ctx->ipc_open.end()) {
      void* p = nullptr;
      KPM_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
      it = ctx->ipc_open.emplace(key, p).first;
    }
    *out = it->second;
    return KPM_OK;
  };
  ctx->dst_x.clear();
  for (const SendRun& r : ctx->send_runs) {
    void *x0, *x1;
    if ((st = open(pubs[r.peer].x0, &x0)) != KPM_OK) return st;
    if ((st = open(pubs[r.peer].x1, &x1)) != KPM_OK) return st;
    const int64_t off = (pubs[r.peer].n_pad + r.peer_slot) * Rk;
    ctx->dst_x.push_back({static_cast<double2*>(x0) + off, static_cast<double2*>(x1) + off});
  }
  ctx->dst_flag.clear();
  for (int q : ctx->dest_peers) {
    void* fl;
    if ((st = open(pubs[q].fl, &fl)) != KPM_OK) return st;
    ctx->dst_flag.push_back(static_cast<int32_t*>(fl) + ctx->opt.rank);
  }
  ctx->fused_ready = true;
  ctx->fused_rk = Rk;
  return KPM_OK;
}

// One block of up to 32 columns: start block, M/2 sweeps, eta reduction, D2H.
// eta_cols: host, [(r*M + n)] double2 for the rb columns of this block.
// Tiled-feed plan (shared-memory layout + copy records, built once per matrix) for block width
// Rk and one W placement; plan.stages == 0 if the matrix does not fit the tiled feed.
static kpm_status plan_tiled_feed(kpm_ctx* ctx, int Rk, bool with_w, int pref_stages, TileLayout& plan) {
  const DevSell& s = ctx->sell;
  const int want = ctx->tile_stages ? std::min(ctx->tile_stages, 4) : pref_stages;
  plan = s.tiles_ok ? plan_tiles(Rk, s.max_other, s.max_width, want, with_w) : TileLayout();
  const int ri = 2 * __builtin_ctz(Rk) + (with_w ? 1 : 0);
  if (plan.stages >= 1 && !ctx->sell.rec_valid[ri] && !ctx->sell.rec_failed[ri]) {
    if (reserve((void**)&ctx->sell.rec[ri], &ctx->sell.rec_cap[ri], sizeof(uint4) * kRecSlots * s.n_chunks) !=
        cudaSuccess) {
      cudaGetLastError();
      ctx->sell.rec_failed[ri] = true;  // no memory for the records: another feed runs
      plan = TileLayout();
      return KPM_OK;
    }
    KPM_CUDA(launch_build_records(s.cptr, s.nruns, s.runs, s.n_chunks, Rk, plan.off_w, plan.off_val, plan.off_lcol,
                                  ctx->sell.rec[ri], ctx->stream));
    ctx->sell.rec_valid[ri] = true;
  }
  if (!ctx->sell.rec_valid[ri]) plan = TileLayout();
  return KPM_OK;
}

// Failure detection: wait for the compute stream of a multi-rank call while polling
// NCCL's asynchronous error state; an error NCCL reports aborts the communicator and leaves the
// context sticky (KPM_ENCCL) instead of waiting forever.  (A peer that dies silently is not
// detected: a blocked NCCL host call or a halo-flag wait would need a watchdog thread and device
// progress counters -- DESIGN.md §11.)  Single rank: a plain synchronize.
static kpm_status wait_stream(kpm_ctx* ctx, cudaStream_t str) {
  if (!ctx->comm) {
    KPM_CUDA(cudaStreamSynchronize(str));
    return KPM_OK;
  }
  for (;;) {
    const cudaError_t q = cudaStreamQuery(str);
    if (q == cudaSuccess) return KPM_OK;
    if (q != cudaErrorNotReady) KPM_CUDA(q);
    ncclResult_t ar = ncclSuccess;
    if (ncclCommGetAsyncError(ctx->comm, &ar) == ncclSuccess && ar != ncclSuccess && ar != ncclInProgress) {
      KPM_TRACE_LINE(ctx->opt.rank, "wait_stream: NCCL async error %d, aborting", (int)ar);
      ncclCommAbort(ctx->comm);
      ctx->comm = nullptr;
      ctx->sticky = true;
      return fail(ctx, KPM_ENCCL, std::string("NCCL asynchronous error: ") + ncclGetErrorString(ar));
    }
    std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
}

// Block-cache plan (per-position copy records, tile maps, absolute tile rows) of variant v for
// this grid and chunk order, built once and cached under bc_key.  ok = every tile fits.
static kpm_status build_bc_plan(kpm_ctx* ctx, int Rk, int v, const TileLayout& tl, int grid, bool& ok) {
  const DevSell& s = ctx->sell;
  const bool wst = variant_wstage(Rk, v);
  const std::vector<int64_t> key = {Rk, grid, ctx->matrix_gen, ctx->order_gen, tl.stages, wst ? 1 : 0, tl.pool_slots,
                                    tl.lt_stride};
  if (key == ctx->bc_key) {
    ok = ctx->bc_ok;
    return KPM_OK;
  }
  ctx->bc_key.clear();
  const bool mem_ok =
      reserve((void**)&ctx->bc_rec, &ctx->bc_rec_cap, sizeof(uint4) * kRecSlots * s.n_chunks) == cudaSuccess &&
      (ctx->opt.nranks == 1 ||
       reserve((void**)&ctx->bc_rec2, &ctx->bc_rec2_cap, sizeof(uint4) * kRecSlots * s.n_chunks) == cudaSuccess) &&
      reserve((void**)&ctx->bc_map, &ctx->bc_map_cap, sizeof(int) * kBcMapInts * s.n_chunks) == cudaSuccess &&
      reserve((void**)&ctx->bc_lcol, &ctx->bc_lcol_cap,
              sizeof(uint16_t) * std::max<int64_t>(s.n_slots, s.n_chunks * kC * (int64_t)tl.lt_stride)) == cudaSuccess &&
      reserve((void**)&ctx->bc_fail, &ctx->bc_fail_cap, sizeof(int)) == cudaSuccess;
  if (!mem_ok) {  // no room for the plan: another variant runs
    cudaGetLastError();
    ctx->bc_ok = ok = false;
    ctx->bc_key = key;
    return KPM_OK;
  }
  KPM_CUDA(cudaMemsetAsync(ctx->bc_fail, 0, sizeof(int), ctx->stream));
  // one plan per launch list (single rank: the chunk order; several ranks: the edge and the
  // interior list, whose chunks are disjoint, so they share the lcol array)
  if (ctx->opt.nranks == 1) {
    KPM_CUDA(launch_build_bc(s.cptr, s.nruns, s.runs, s.col, ctx->order_list, s.n_chunks, grid, Rk, wst, tl, ctx->bc_rec,
                             ctx->bc_map, ctx->bc_lcol, ctx->bc_fail, ctx->stream));
  } else {
    if (ctx->n_edge)
      KPM_CUDA(launch_build_bc(s.cptr, s.nruns, s.runs, s.col, ctx->edge_list, ctx->n_edge, grid, Rk, wst, tl,
                               ctx->bc_rec, ctx->bc_map, ctx->bc_lcol, ctx->bc_fail, ctx->stream));
    if (ctx->n_interior)
      KPM_CUDA(launch_build_bc(s.cptr, s.nruns, s.runs, s.col, ctx->interior_list, ctx->n_interior, grid, Rk, wst, tl,
                               ctx->bc_rec2, ctx->bc_map, ctx->bc_lcol, ctx->bc_fail, ctx->stream));
  }
  int hfail = 0;
  KPM_CUDA(cudaMemcpyAsync(&hfail, ctx->bc_fail, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  KPM_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx->bc_ok = ok = hfail == 0;
  ctx->bc_key = key;
  return KPM_OK;
}

// The sweep kernel of block width Rk: the requested variant (KPM_VARIANT, else the width's
// default), or the first later one in table order whose feed fits the matrix (the last entry of
// every width, the direct feed, always does).  With several ranks every rank takes the same
// variant: each candidate is agreed on with one allgather, once per matrix (cached).
static kpm_status select_variant(kpm_ctx* ctx, int Rk, int& variant, TileLayout& tl, int& grid, bool& bc) {
  const DevSell& s = ctx->sell;
  const int n = variant_count(Rk);
  const int lg = __builtin_ctz(Rk);
  const bool cached = ctx->chosen_gen[lg] == ctx->matrix_gen && ctx->chosen_ovr[lg] == ctx->variant_override;
  std::vector<int> cand;
  if (cached) {
    cand.push_back(ctx->chosen[lg]);
  } else {
    if (ctx->variant_override >= 0 && ctx->variant_override < n) cand.push_back(ctx->variant_override);
    for (int v = 0; v < n; ++v)
      if (cand.empty() || v != cand[0]) cand.push_back(v);
  }
  for (int v : cand) {
    TileLayout pl;
    bool ok = true;
    const int bcc = variant_bc(Rk, v);
    kpm_status st;
    if (bcc) {
      // the block-cache kernels read row-major tile indices only (KPM_LCOL_T=0 turns them off)
      pl = s.tiles_ok && ctx->lcol_t ? plan_tiles_bc(Rk, s.max_width, variant_wstage(Rk, v), variant_stages(Rk, v), bcc,
                                                     true)
                                     : TileLayout();
      ok = pl.stages >= 1;
    } else if (variant_tiled(Rk, v)) {
      if ((st = plan_tiled_feed(ctx, Rk, variant_wstage(Rk, v), variant_stages(Rk, v), pl)) != KPM_OK) return st;
      ok = pl.stages >= 1;
    } else if (variant_staged(Rk, v)) {
      ok = s.max_width <= staged_max_width();
    }
    int g = 1;
    if (ok) {
      const int dyn = variant_tiled(Rk, v) ? pl.pool_bytes + pl.stages * pl.stage_bytes : 0;
      const int occ_q = sweep_occupancy(Rk, v, dyn);  // also loads the variant's kernels (kernels.cu)
      const int occ = ctx->grid_per_sm ? ctx->grid_per_sm : std::max(1, occ_q);
      g = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)ctx->num_sms * occ, s.n_chunks));
      if ((st = ensure_order(ctx, g, bcc > 0, Rk, variant_strip(Rk, v))) != KPM_OK) return st;
      if (bcc && (st = build_bc_plan(ctx, Rk, v, pl, g, ok)) != KPM_OK) return st;
    }
    if (ctx->opt.nranks > 1 && !cached) {  // agree, so that every rank runs the same launches
      std::vector<int64_t> all;
      if ((st = allgather_i64(ctx, {ok ? 1 : 0}, all)) != KPM_OK) return st;
      for (int64_t x : all) ok = ok && x == 1;
    }
    if (ok) {
      // re-install the chosen kernel's order (a plan tried after it may have replaced it; both
      // calls are no-ops when nothing changed)
      if ((st = ensure_order(ctx, g, bcc > 0, Rk, variant_strip(Rk, v))) != KPM_OK) return st;
      if (bcc && (st = build_bc_plan(ctx, Rk, v, pl, g, ok)) != KPM_OK) return st;
      if (!ok) return fail(ctx, KPM_ESTATE, "internal: block-cache plan changed");
      variant = v;
      tl = pl;
      grid = g;
      bc = bcc > 0;
      ctx->chosen[lg] = v;
      ctx->chosen_gen[lg] = ctx->matrix_gen;
      ctx->chosen_ovr[lg] = ctx->variant_override;
      return KPM_OK;
    }
  }
  return fail(ctx, KPM_ESTATE, cached ? "internal: the cached kernel variant no longer fits" : "no kernel variant fits");
}

static kpm_status run_block(kpm_ctx* ctx, int M, int rb, int64_t col_begin, uint64_t seed, const double* v0,
                            double2* eta_cols, bool first, bool last) {
  const int Rk = block_width(rb);
  const int n_sweeps = M / 2;
  const DevSell& s = ctx->sell;
  const int64_t n_rows_total = s.n_pad + s.n_halo;
  kpm_status st;
  size_t xcap = ctx->x_cap;
  st = ensure(ctx, (void**)&ctx->X0, &xcap, (size_t)n_rows_total * Rk, sizeof(double2));
  if (st == KPM_OK) {
    xcap = ctx->x_cap;
    st = ensure(ctx, (void**)&ctx->X1, &xcap, (size_t)n_rows_total * Rk, sizeof(double2));
    if (xcap != ctx->x_cap) ctx->fused_ready = false;
    if (st == KPM_OK) ctx->x_cap = xcap;
  }
  if ((st = agree(ctx, st)) != KPM_OK) return st;
  if (ctx->opt.nranks > 1 && ctx->fused) {  // collective: re-publish when any rank's buffers changed
    std::vector<int64_t> all;
    if ((st = allgather_i64(ctx, {ctx->fused_ready && ctx->fused_rk == Rk ? 1 : 0}, all)) != KPM_OK) return st;
    bool ready = true;
    for (int64_t v : all) ready = ready && v == 1;
    if (!ready) {
      // IPC mapping can fail (no P2P between the GPUs, restricted containers): then every rank
      // falls back to the NCCL exchange together
      const kpm_status fst = setup_fused(ctx, Rk);
      if (fst != KPM_OK) {
        cudaGetLastError();
        ctx->sticky = false;
        ctx->fused_ready = false;
      }
      std::vector<int64_t> oks;
      if ((st = allgather_i64(ctx, {fst == KPM_OK ? 1 : 0}, oks)) != KPM_OK) return st;
      for (int64_t v : oks)
        if (v != 1) ctx->fused = false;
      if (!ctx->fused) fprintf(stderr, "kpm: fused NVLink halo exchange unavailable (%s); using NCCL P2P\n",
                               fst == KPM_OK ? "another rank failed" : ctx->err.c_str());
    }
  }

  int variant = 0, grid = 1;
  TileLayout tl;
  bool bc = false;
  st = select_variant(ctx, Rk, variant, tl, grid, bc);
  // a local failure after the (cached) choice must not leave the other ranks in the next collective
  if (ctx->opt.nranks > 1 && !ctx->sticky) st = agree(ctx, st);
  if (st != KPM_OK) return st;
  KPM_TRACE_LINE(ctx->opt.rank, "variant selected: %s (fused %d, edge %lld, interior %lld)", variant_name(Rk, variant),
                 (int)ctx->fused, (long long)ctx->n_edge, (long long)ctx->n_interior);
  const int rec_index = 2 * __builtin_ctz(Rk) + (variant_wstage(Rk, variant) ? 1 : 0);
  ctx->last_variant = variant_name(Rk, variant);
  const bool multi = ctx->opt.nranks > 1;
  const int parts = multi ? 2 : 1;  // edge + interior launches per sweep
  const size_t per_sweep = (size_t)3 * Rk * grid * parts;
  st = ensure(ctx, (void**)&ctx->partials, &ctx->partials_cap, per_sweep * n_sweeps, sizeof(double));
  size_t ecap = ctx->eta_cap;
  if (st == KPM_OK) st = ensure(ctx, (void**)&ctx->eta_even, &ecap, (size_t)n_sweeps * kMaxBlockWidth, sizeof(double2));
  if (st == KPM_OK) {
    ecap = ctx->eta_cap;
    st = ensure(ctx, (void**)&ctx->eta_odd, &ecap, (size_t)n_sweeps * kMaxBlockWidth, sizeof(double2));
  }
  if (st == KPM_OK && (ecap > ctx->eta_cap || !ctx->h_eta)) {
    if (ctx->h_eta) cudaFreeHost(ctx->h_eta);
    ctx->h_eta = nullptr;
    if (cudaMallocHost((void**)&ctx->h_eta, sizeof(double2) * 2 * ecap) != cudaSuccess) {
      cudaGetLastError();
      st = fail(ctx, KPM_ENOMEM, "pinned host allocation failed");
    }
  }
  if (st == KPM_OK) ctx->eta_cap = ecap;
  if (v0 && st == KPM_OK) {
    size_t vcap = ctx->v0_cap;
    st = ensure(ctx, (void**)&ctx->v0_dev, &vcap, (size_t)s.n_loc * rb, sizeof(double2));
    if (st == KPM_OK) ctx->v0_cap = vcap;
  }
  if ((st = agree(ctx, st)) != KPM_OK) return st;

  cudaStream_t str = ctx->stream;
  if (first) KPM_CUDA(cudaEventRecord(ctx->ev[0], str));
  // a1: start block
  if (v0) {
    KPM_CUDA(cudaMemcpyAsync(ctx->v0_dev, v0, sizeof(double2) * s.n_loc * rb, cudaMemcpyHostToDevice, str));
    KPM_CUDA(launch_v0_upload_permute(ctx->X0, ctx->X1, ctx->v0_dev, s.perm, s.n_loc, s.n_pad, n_rows_total, Rk, rb, str));
    if (multi && (st = exchange_halo(ctx, ctx->X0, Rk, str)) != KPM_OK) return st;
  } else {  // halo slots get their Z4 values directly from their global ids: no exchange for nu_0
    KPM_CUDA(launch_z4_init(ctx->X0, ctx->X1, s.perm, s.n_loc, s.n_pad, ctx->halo_rows, n_rows_total, Rk,
                            ctx->row_begin, col_begin, rb, seed, str));
  }
  SweepArgs sa;
  sa.val = s.val;
  sa.col = s.col;
  sa.cptr = s.cptr;
  sa.n_loc = s.n_loc;
  sa.chunk_list = ctx->order_list;  // NULL: storage order
  sa.chunk_begin = 0;
  sa.chunk_end = s.n_chunks;
  sa.rec = bc ? ctx->bc_rec : s.rec[rec_index];
  sa.lcol = bc ? ctx->bc_lcol : s.lcol;
  sa.tl = tl;
  sa.b = ctx->b;
  sa.pstride = (int64_t)grid * parts;
  sa.n_peer = 0;
  sa.v_evict_last = env_int("KPM_V_EVICT_LAST", 1);
  // One sweep m (m = 0: init sweep W = a(H - b)V; m >= 1: W <- 2a(H - b)V - W), with the
  // fused eta_2m, eta_2m+1 partials.  Multi-rank: edge chunks first, then the new boundary
  // rows go to the neighbours on the comm stream while the interior chunks run (a5).
  auto sweep = [&](int m) -> kpm_status {
    const bool init = (m == 0);
    sa.V = (m & 1) ? ctx->X1 : ctx->X0;
    sa.W = (m & 1) ? ctx->X0 : ctx->X1;
    sa.scale = init ? ctx->a : 2.0 * ctx->a;
    double* part = ctx->partials + per_sweep * m;
    if (!multi) {
      sa.partials = part;
      KPM_CUDA(launch_aug_spmmv(Rk, variant, init, sa, grid, str));
      return KPM_OK;
    }
    sa.chunk_list = ctx->edge_list;
    sa.chunk_begin = 0;
    sa.chunk_end = ctx->n_edge;
    sa.partials = part;
    if (bc) sa.rec = ctx->bc_rec;
    if (ctx->fused) {
      // Virtual ranks: every rank has enqueued its flag write for this epoch before any rank
      // enqueues a wait for it, so no stream ever waits on work its host thread has yet to
      // enqueue -- an implicit device synchronisation by one thread (e.g. a lazy module load in
      // a launch) would otherwise wait for a stream that waits for that very thread.
      if (ctx->vg && m > 0) ctx->vg->allgatherv(ctx->opt.rank, {});
      // V's halo slots were written by the neighbours' previous edge launch: wait for their flags
      if (m > 0)
        for (int q : ctx->src_peers)
          if (g_wait_value32(str, (CUdeviceptr)(ctx->flags + q), ctx->epoch, CU_STREAM_WAIT_VALUE_GEQ) !=
              CUDA_SUCCESS)
            return fail(ctx, KPM_ECUDA, "cuStreamWaitValue32 failed");
      KPM_TRACE_LINE(ctx->opt.rank, "sweep %d: waits on %zu peers for epoch %u enqueued", m,
                     m > 0 ? ctx->src_peers.size() : (size_t)0, ctx->epoch);
      const bool send = m + 1 < n_sweeps;
      sa.n_peer = send ? (int)ctx->send_runs.size() : 0;
      for (int i = 0; i < sa.n_peer; ++i)
        sa.peer[i] = PeerRun{ctx->send_runs[i].pos, ctx->send_runs[i].count, ctx->dst_x[i][(m + 1) & 1]};
      KPM_CUDA(launch_aug_spmmv(Rk, variant, init, sa, grid, str));
      sa.n_peer = 0;
      if (send) {
        ++ctx->epoch;
        for (int32_t* f : ctx->dst_flag)
          if (g_write_value32(str, (CUdeviceptr)f, ctx->epoch, CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
            return fail(ctx, KPM_ECUDA, "cuStreamWriteValue32 failed");
      }
      sa.chunk_list = ctx->interior_list;
      sa.chunk_end = ctx->n_interior;
      if (bc) sa.rec = ctx->bc_rec2;
      sa.partials = part + grid;
      KPM_CUDA(launch_aug_spmmv(Rk, variant, init, sa, grid, str));
      return KPM_OK;
    }
    if (m > 0) KPM_CUDA(cudaStreamWaitEvent(str, ctx->ev_halo, 0));  // V's halo slots have arrived
    KPM_CUDA(launch_aug_spmmv(Rk, variant, init, sa, grid, str));
    if (m + 1 < n_sweeps) {
      KPM_CUDA(cudaEventRecord(ctx->ev_edge, str));
      KPM_CUDA(cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_edge, 0));
      kpm_status est = exchange_halo(ctx, sa.W, Rk, ctx->comm_stream);
      if (est != KPM_OK) return est;
      KPM_CUDA(cudaEventRecord(ctx->ev_halo, ctx->comm_stream));
    }
    sa.chunk_list = ctx->interior_list;
    sa.chunk_end = ctx->n_interior;
    if (bc) sa.rec = ctx->bc_rec2;
    sa.partials = part + grid;
    KPM_CUDA(launch_aug_spmmv(Rk, variant, init, sa, grid, str));
    return KPM_OK;
  };
  // KPM_TIMING: an event before the init sweep and after every sweep (no graph, per-launch)
  const bool timing = (ctx->opt.flags & KPM_TIMING) != 0;
  if (timing) {
    while ((int)ctx->sweep_ev.size() < n_sweeps + 1) {
      cudaEvent_t e;
      KPM_CUDA(cudaEventCreate(&e));
      ctx->sweep_ev.push_back(e);
    }
    KPM_CUDA(cudaEventRecord(ctx->sweep_ev[0], str));
  }
  KPM_TRACE_LINE(ctx->opt.rank, "run_block: start block enqueued, %d sweeps, variant %s, grid %d", n_sweeps,
                 ctx->last_variant.c_str(), grid);
  // a2: init sweep, eta_0, eta_1
  if ((st = sweep(0)) != KPM_OK) return st;
  if (timing) KPM_CUDA(cudaEventRecord(ctx->sweep_ev[1], str));
  // a3: main sweeps, eta_2m, eta_2m+1.  Single rank: the M/2-1 launches are captured once
  // into a CUDA graph per configuration and replayed (launch overhead matters for small
  // matrices, e.g. C1's 5-us sweeps); env KPM_GRAPH=0 launches them one by one.
  KPM_CUDA(cudaEventRecord(ctx->ev[1], str));
  // graphs pay off only when a sweep is short (launch overhead ~ 4 us vs the sweep); for large
  // matrices a re-capture after every kpm_set_matrix would cost more than it saves
  const double sweep_bytes = 20.0 * (double)s.n_slots + 48.0 * Rk * (double)s.n_pad;
  const bool use_graph = !multi && !timing && ctx->use_graph && n_sweeps > 2 && sweep_bytes < 512e6;
  if (use_graph) {
    int64_t abits, bbits;  // the exact scale factors (bit patterns) the captured launches carry
    std::memcpy(&abits, &ctx->a, sizeof abits);
    std::memcpy(&bbits, &ctx->b, sizeof bbits);
    const std::vector<int64_t> key = {Rk, variant, grid, n_sweeps, (int64_t)ctx->X0, (int64_t)ctx->X1,
                                      (int64_t)ctx->partials, (int64_t)sa.chunk_list, (int64_t)sa.rec,
                                      (int64_t)s.val, abits, bbits, ctx->matrix_gen, ctx->order_gen, tl.stages};
    if (!ctx->graph_exec || key != ctx->graph_key) {
      if (ctx->graph_exec) cudaGraphExecDestroy(ctx->graph_exec);
      ctx->graph_exec = nullptr;
      cudaGraph_t g;
      KPM_CUDA(cudaStreamBeginCapture(str, cudaStreamCaptureModeThreadLocal));
      for (int m = 1; m < n_sweeps; ++m)
        if ((st = sweep(m)) != KPM_OK) {
          if (cudaStreamEndCapture(str, &g) == cudaSuccess && g) cudaGraphDestroy(g);
          cudaGetLastError();
          return st;
        }
      KPM_CUDA(cudaStreamEndCapture(str, &g));
      KPM_CUDA(cudaGraphInstantiate(&ctx->graph_exec, g, 0));
      KPM_CUDA(cudaGraphDestroy(g));
      ctx->graph_key = key;
    }
    KPM_CUDA(cudaGraphLaunch(ctx->graph_exec, str));
  } else {
    for (int m = 1; m < n_sweeps; ++m) {
      if ((st = sweep(m)) != KPM_OK) return st;
      if (timing) KPM_CUDA(cudaEventRecord(ctx->sweep_ev[m + 1], str));
      KPM_TRACE_LINE(ctx->opt.rank, "sweep %d enqueued (epoch %u)", m, ctx->epoch);
    }
  }
  KPM_TRACE_LINE(ctx->opt.rank, "all sweeps enqueued");
  KPM_CUDA(cudaEventRecord(ctx->ev[2], str));
  // a4: deterministic grid reduction of all sweeps' partials
  KPM_CUDA(launch_eta_finalize(ctx->partials, n_sweeps, Rk, grid * parts, ctx->eta_even, ctx->eta_odd, str));
  if (multi && ctx->vg) {  // virtual ranks: host all-gather, sum in rank order, back to the device
    const size_t ne = (size_t)n_sweeps * Rk * 2;
    std::vector<int64_t> mine(2 * ne);
    KPM_TRACE_LINE(ctx->opt.rank, "eta reduction: waiting for the stream");
    KPM_CUDA(cudaStreamSynchronize(str));
    KPM_TRACE_LINE(ctx->opt.rank, "eta reduction: stream done");
    KPM_CUDA(cudaMemcpyAsync(mine.data(), ctx->eta_even, sizeof(double) * ne, cudaMemcpyDeviceToHost, str));
    KPM_CUDA(cudaMemcpyAsync(mine.data() + ne, ctx->eta_odd, sizeof(double) * ne, cudaMemcpyDeviceToHost, str));
    KPM_CUDA(cudaStreamSynchronize(str));
    const auto all = ctx->vg->allgatherv(ctx->opt.rank, mine);
    std::vector<double> sum(2 * ne, 0.0);
    for (const auto& v : all)
      for (size_t i = 0; i < 2 * ne; ++i) {
        double x;
        std::memcpy(&x, &v[i], sizeof x);
        sum[i] += x;
      }
    KPM_CUDA(cudaMemcpyAsync(ctx->eta_even, sum.data(), sizeof(double) * ne, cudaMemcpyHostToDevice, str));
    KPM_CUDA(cudaMemcpyAsync(ctx->eta_odd, sum.data() + ne, sizeof(double) * ne, cudaMemcpyHostToDevice, str));
    KPM_CUDA(cudaStreamSynchronize(str));
  } else if (multi) {  // a6: the single global reduction, once, at the end (Table III)
    KPM_NCCL(ncclAllReduce(ctx->eta_even, ctx->eta_even, (size_t)n_sweeps * Rk * 2, ncclDouble, ncclSum, ctx->comm, str));
    KPM_NCCL(ncclAllReduce(ctx->eta_odd, ctx->eta_odd, (size_t)n_sweeps * Rk * 2, ncclDouble, ncclSum, ctx->comm, str));
  }
  KPM_CUDA(cudaMemcpyAsync(ctx->h_eta, ctx->eta_even, sizeof(double2) * n_sweeps * Rk, cudaMemcpyDeviceToHost, str));
  KPM_CUDA(cudaMemcpyAsync(ctx->h_eta + ctx->eta_cap, ctx->eta_odd, sizeof(double2) * n_sweeps * Rk,
                           cudaMemcpyDeviceToHost, str));
  if (last) KPM_CUDA(cudaEventRecord(ctx->ev[3], str));
  if ((st = wait_stream(ctx, str)) != KPM_OK) return st;
  for (int r = 0; r < rb; ++r)
    for (int m = 0; m < n_sweeps; ++m) {
      eta_cols[(size_t)r * M + 2 * m] = ctx->h_eta[(size_t)m * Rk + r];
      eta_cols[(size_t)r * M + 2 * m + 1] = ctx->h_eta[ctx->eta_cap + (size_t)m * Rk + r];
    }
  float ms = 0.f;
  if (n_sweeps > 1) {
    KPM_CUDA(cudaEventElapsedTime(&ms, ctx->ev[1], ctx->ev[2]));
    ctx->last_sweep_ms = ms / (n_sweeps - 1);
    ctx->last_n_sweeps = n_sweeps - 1;
  } else {
    ctx->last_sweep_ms = 0.0;
    ctx->last_n_sweeps = 0;
  }
  if (timing)
    for (int m = 0; m < n_sweeps; ++m) {
      KPM_CUDA(cudaEventElapsedTime(&ms, ctx->sweep_ev[m], ctx->sweep_ev[m + 1]));
      ctx->sweep_times.push_back(ms);
    }
  if (last) {
    KPM_CUDA(cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[3]));
    ctx->last_total_ms = ms;
  }
  return KPM_OK;
}

// a6: eta -> mu (doubling identities, stochastic trace)
static kpm_status finish_mu(kpm_ctx* ctx, int M, int R, const std::vector<double2>& eta_all, bool explicit_v0,
                            double* mu, double* eta) {
  bool zero_norm = false;
  std::vector<double> acc(M, 0.0);
  std::vector<double2> m(M);
  for (int r = 0; r < R; ++r) {
    const double2* e = eta_all.data() + (size_t)r * M;
    if (e[0].x == 0.0) zero_norm = true;
    m[0] = e[0];
    m[1] = e[1];
    for (int k = 1; 2 * k < M; ++k) {
      m[2 * k] = make_double2(2.0 * e[2 * k].x - m[0].x, 2.0 * e[2 * k].y - m[0].y);
      m[2 * k + 1] = make_double2(2.0 * e[2 * k + 1].x - m[1].x, 2.0 * e[2 * k + 1].y - m[1].y);
    }
    for (int n = 0; n < M; ++n) acc[n] += m[n].x;
  }
  bool diverged = false;
  for (int n = 0; n < M; ++n) mu[n] = acc[n] / (double)R;
  for (int n = 1; n < M; ++n)
    if (!(std::fabs(mu[n]) <= std::fabs(mu[0]) * (1.0 + 1e-8))) diverged = true;
  if (eta) std::memcpy(eta, eta_all.data(), sizeof(double2) * (size_t)R * M);
  if (explicit_v0 && zero_norm) return fail(ctx, KPM_EZERONORM, "a start column has eta_0 = 0");
  if (diverged) return fail(ctx, KPM_WDIVERGED, "|mu_n| > mu_0: a, b do not map the spectrum into [-1, 1]");
  return KPM_OK;
}

static kpm_status moments_common(kpm_ctx* ctx, int M, int R, uint64_t seed, const double* v0, double* mu,
                                 double* eta) {
  if (!ctx) return KPM_EINVAL;
  if (ctx->sticky) return fail(ctx, KPM_ESTATE, "context has a sticky CUDA/NCCL error: " + ctx->err);
  if (!ctx->have_matrix) return fail(ctx, KPM_ESTATE, "kpm_set_matrix has not been called");
  if (M < 2 || (M % 2) != 0) return fail(ctx, KPM_EINVAL, "M must be even and >= 2");
  if (R < 1) return fail(ctx, KPM_EINVAL, "R must be >= 1");
  if (!mu) return fail(ctx, KPM_EINVAL, "mu is NULL");
  KPM_CUDA(cudaSetDevice(ctx->opt.device));
  ctx->sweep_times.clear();
  std::vector<double2> eta_all((size_t)R * M);
  const int64_t n_loc = ctx->sell.n_loc;
  std::vector<double> v0_block;
  for (int c0 = 0; c0 < R; c0 += kMaxBlockWidth) {
    const int rb = std::min(kMaxBlockWidth, R - c0);
    const double* v0b = nullptr;
    if (v0) {  // columns c0..c0+rb-1 of the caller's n_loc x R block, repacked n_loc x rb
      v0_block.resize((size_t)2 * n_loc * rb);
      for (int64_t i = 0; i < n_loc; ++i)
        for (int r = 0; r < rb; ++r) {
          v0_block[2 * (i * rb + r)] = v0[2 * (i * R + c0 + r)];
          v0_block[2 * (i * rb + r) + 1] = v0[2 * (i * R + c0 + r) + 1];
        }
      v0b = v0_block.data();
    }
    kpm_status st = run_block(ctx, M, rb, c0, seed, v0b, eta_all.data() + (size_t)c0 * M, c0 == 0,
                              c0 + kMaxBlockWidth >= R);
    if (st != KPM_OK) return st;
  }
  return finish_mu(ctx, M, R, eta_all, v0 != nullptr, mu, eta);
}

// Naive stage-0 KPM of Fig. 3 for one column (naive.cu), same outputs as run_block.
static kpm_status naive_column(kpm_ctx* ctx, int M, int64_t col_begin, uint64_t seed, double2* eta_cols, bool first,
                               bool last) {
  const int n_sweeps = M / 2;
  const DevSell& s = ctx->sell;
  const int64_t n_rows_total = s.n_pad + s.n_halo;
  kpm_status st;
  size_t xcap = ctx->x_cap;
  if ((st = ensure(ctx, (void**)&ctx->X0, &xcap, (size_t)n_rows_total, sizeof(double2))) != KPM_OK) return st;
  xcap = ctx->x_cap;
  if ((st = ensure(ctx, (void**)&ctx->X1, &xcap, (size_t)n_rows_total, sizeof(double2))) != KPM_OK) return st;
  if (xcap != ctx->x_cap) ctx->fused_ready = false;
  ctx->x_cap = xcap;
  if ((st = ensure(ctx, (void**)&ctx->u_naive, &ctx->u_cap, (size_t)s.n_pad, sizeof(double2))) != KPM_OK) return st;
  const int g = naive_grid();
  if ((st = ensure(ctx, (void**)&ctx->partials, &ctx->partials_cap, (size_t)3 * g * n_sweeps, sizeof(double))) != KPM_OK)
    return st;
  size_t ecap = ctx->eta_cap;
  if ((st = ensure(ctx, (void**)&ctx->eta_even, &ecap, (size_t)n_sweeps * kMaxBlockWidth, sizeof(double2))) != KPM_OK)
    return st;
  ecap = ctx->eta_cap;
  if ((st = ensure(ctx, (void**)&ctx->eta_odd, &ecap, (size_t)n_sweeps * kMaxBlockWidth, sizeof(double2))) != KPM_OK)
    return st;
  if (ecap > ctx->eta_cap || !ctx->h_eta) {
    if (ctx->h_eta) cudaFreeHost(ctx->h_eta);
    ctx->h_eta = nullptr;
    if (cudaMallocHost((void**)&ctx->h_eta, sizeof(double2) * 2 * ecap) != cudaSuccess) {
      cudaGetLastError();
      return fail(ctx, KPM_ENOMEM, "pinned host allocation failed");
    }
  }
  ctx->eta_cap = ecap;
  cudaStream_t str = ctx->stream;
  if (first) KPM_CUDA(cudaEventRecord(ctx->ev[0], str));
  KPM_CUDA(launch_z4_init(ctx->X0, ctx->X1, s.perm, s.n_loc, s.n_pad, ctx->halo_rows, n_rows_total, 1, ctx->row_begin,
                          col_begin, 1, seed, str));
  KPM_CUDA(naive_sweep(s, ctx->X0, ctx->X1, ctx->u_naive, ctx->a, ctx->b, true, ctx->partials, str));
  KPM_CUDA(cudaEventRecord(ctx->ev[1], str));
  for (int m = 1; m < n_sweeps; ++m) {  // swap(|w>, |v>) is the pointer swap
    const double2* v = (m & 1) ? ctx->X1 : ctx->X0;
    double2* w = (m & 1) ? ctx->X0 : ctx->X1;
    KPM_CUDA(naive_sweep(s, v, w, ctx->u_naive, ctx->a, ctx->b, false, ctx->partials + (size_t)3 * g * m, str));
  }
  KPM_CUDA(cudaEventRecord(ctx->ev[2], str));
  KPM_CUDA(launch_eta_finalize(ctx->partials, n_sweeps, 1, g, ctx->eta_even, ctx->eta_odd, str));
  KPM_CUDA(cudaMemcpyAsync(ctx->h_eta, ctx->eta_even, sizeof(double2) * n_sweeps, cudaMemcpyDeviceToHost, str));
  KPM_CUDA(cudaMemcpyAsync(ctx->h_eta + ctx->eta_cap, ctx->eta_odd, sizeof(double2) * n_sweeps, cudaMemcpyDeviceToHost,
                           str));
  if (last) KPM_CUDA(cudaEventRecord(ctx->ev[3], str));
  KPM_CUDA(cudaStreamSynchronize(str));
  for (int m = 0; m < n_sweeps; ++m) {
    eta_cols[2 * m] = ctx->h_eta[m];
    eta_cols[2 * m + 1] = ctx->h_eta[ctx->eta_cap + m];
  }
  float ms = 0.f;
  if (n_sweeps > 1) {
    KPM_CUDA(cudaEventElapsedTime(&ms, ctx->ev[1], ctx->ev[2]));
    ctx->last_sweep_ms = ms / (n_sweeps - 1);
    ctx->last_n_sweeps = n_sweeps - 1;
  }
  if (last) {
    KPM_CUDA(cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[3]));
    ctx->last_total_ms = ms;
  }
  return KPM_OK;
}

extern "C" kpm_status kpm_moments(kpm_ctx* ctx, int M, int R, uint64_t seed, double* mu, double* eta) {
  return moments_common(ctx, M, R, seed, nullptr, mu, eta);
}

extern "C" kpm_status kpm_moments_stage(kpm_ctx* ctx, int stage, int M, int R, uint64_t seed, double* mu,
                                        double* eta) {
  if (stage == KPM_STAGE_AUG_SPMMV) return moments_common(ctx, M, R, seed, nullptr, mu, eta);
  if (!ctx) return KPM_EINVAL;
  if (stage != KPM_STAGE_NAIVE && stage != KPM_STAGE_AUG_SPMV) return fail(ctx, KPM_EINVAL, "unknown stage");
  if (ctx->sticky) return fail(ctx, KPM_ESTATE, "context has a sticky CUDA/NCCL error: " + ctx->err);
  if (!ctx->have_matrix) return fail(ctx, KPM_ESTATE, "kpm_set_matrix has not been called");
  if (M < 2 || (M % 2) != 0) return fail(ctx, KPM_EINVAL, "M must be even and >= 2");
  if (R < 1 || !mu) return fail(ctx, KPM_EINVAL, "R must be >= 1 and mu non-NULL");
  if (stage == KPM_STAGE_NAIVE && ctx->opt.nranks > 1) return fail(ctx, KPM_EINVAL, "the naive stage is single-rank");
  KPM_CUDA(cudaSetDevice(ctx->opt.device));
  std::vector<double2> eta_all((size_t)R * M);
  for (int r = 0; r < R; ++r) {  // outer loop over the random vectors (Figs. 3, 4: P:266)
    const kpm_status st = stage == KPM_STAGE_NAIVE
                              ? naive_column(ctx, M, r, seed, eta_all.data() + (size_t)r * M, r == 0, r == R - 1)
                              : run_block(ctx, M, 1, r, seed, nullptr, eta_all.data() + (size_t)r * M, r == 0, r == R - 1);
    if (st != KPM_OK) return st;
  }
  if (stage == KPM_STAGE_NAIVE) ctx->last_variant = "naive.blas1";
  return finish_mu(ctx, M, R, eta_all, false, mu, eta);
}

extern "C" kpm_status kpm_moments_v0(kpm_ctx* ctx, int M, int R, const double* v0, double* mu, double* eta) {
  if (ctx && !v0) return fail(ctx, KPM_EINVAL, "v0 is NULL");
  return moments_common(ctx, M, R, 0, v0, mu, eta);
}

extern "C" kpm_status kpm_sweep_kernel(kpm_ctx* ctx, int kind, int R, uint64_t seed, int n_sweeps,
                                       double* ms_per_sweep, double* w_out) {
  if (!ctx) return KPM_EINVAL;
  if (ctx->sticky) return fail(ctx, KPM_ESTATE, "context has a sticky CUDA/NCCL error: " + ctx->err);
  if (!ctx->have_matrix) return fail(ctx, KPM_ESTATE, "kpm_set_matrix has not been called");
  if (ctx->opt.nranks > 1) return fail(ctx, KPM_ESTATE, "kpm_sweep_kernel is single-rank");
  if (kind < KPM_SWEEP_AUG || kind > KPM_SWEEP_SPMMV) return fail(ctx, KPM_EINVAL, "unknown sweep kind");
  if (R < 1 || R > kMaxBlockWidth || (R & (R - 1))) return fail(ctx, KPM_EINVAL, "R must be 1, 2, 4, 8, 16 or 32");
  if (n_sweeps < 1) return fail(ctx, KPM_EINVAL, "n_sweeps must be >= 1");
  KPM_CUDA(cudaSetDevice(ctx->opt.device));
  const DevSell& s = ctx->sell;
  const int64_t n_rows_total = s.n_pad + s.n_halo;
  kpm_status st;
  size_t xcap = ctx->x_cap;
  if ((st = ensure(ctx, (void**)&ctx->X0, &xcap, (size_t)n_rows_total * R, sizeof(double2))) != KPM_OK) return st;
  xcap = ctx->x_cap;
  if ((st = ensure(ctx, (void**)&ctx->X1, &xcap, (size_t)n_rows_total * R, sizeof(double2))) != KPM_OK) return st;
  ctx->x_cap = xcap;
  TileLayout tl;
  const int bv = base_variant(R);  // the analysis kernels use the regular tiled feed
  if (variant_tiled(R, bv) && (st = plan_tiled_feed(ctx, R, variant_wstage(R, bv), variant_stages(R, bv), tl)) != KPM_OK)
    return st;
  if (!variant_tiled(R, bv) || tl.stages < 1)
    return fail(ctx, KPM_ESTATE, "the matrix does not fit the tiled feed of the analysis kernels");
  const int dyn_smem = tl.stages * tl.stage_bytes;
  const int occ = ctx->grid_per_sm ? ctx->grid_per_sm : std::max(1, sweep_occupancy(R, bv, dyn_smem));
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)ctx->num_sms * occ, s.n_chunks));
  if ((st = ensure(ctx, (void**)&ctx->partials, &ctx->partials_cap, (size_t)3 * R * grid, sizeof(double))) != KPM_OK)
    return st;
  cudaStream_t str = ctx->stream;
  KPM_CUDA(launch_z4_init(ctx->X0, ctx->X1, s.perm, s.n_loc, s.n_pad, ctx->halo_rows, n_rows_total, R, ctx->row_begin, 0,
                          R, seed, str));
  SweepArgs sa;
  sa.val = s.val;
  sa.col = s.col;
  sa.cptr = s.cptr;
  sa.n_loc = s.n_loc;
  sa.chunk_list = ctx->order_list;
  sa.chunk_begin = 0;
  sa.chunk_end = s.n_chunks;
  sa.rec = s.rec[2 * __builtin_ctz(R) + (variant_wstage(R, bv) ? 1 : 0)];
  sa.lcol = s.lcol;
  sa.tl = tl;
  sa.b = ctx->b;
  sa.scale = 2.0 * ctx->a;
  sa.V = ctx->X0;
  sa.W = ctx->X1;
  sa.partials = ctx->partials;
  sa.pstride = grid;
  sa.n_peer = 0;
  sa.v_evict_last = env_int("KPM_V_EVICT_LAST", 1);
  KPM_CUDA(cudaEventRecord(ctx->ev[1], str));
  for (int i = 0; i < n_sweeps; ++i) KPM_CUDA(launch_sweep_kind(R, kind, sa, grid, str));
  KPM_CUDA(cudaEventRecord(ctx->ev[2], str));
  KPM_CUDA(cudaStreamSynchronize(str));
  float ms = 0.f;
  KPM_CUDA(cudaEventElapsedTime(&ms, ctx->ev[1], ctx->ev[2]));
  if (ms_per_sweep) *ms_per_sweep = ms / n_sweeps;
  static const char* kSuffix[] = {"", ".nodot", ".spmmv"};
  ctx->last_variant = std::string(variant_name(R, bv)) + kSuffix[kind];
  if (w_out) {  // stored position p holds local row perm[p] (identity when sigma = 1)
    std::vector<double2> wh((size_t)s.n_pad * R);
    KPM_CUDA(cudaMemcpy(wh.data(), ctx->X1, sizeof(double2) * wh.size(), cudaMemcpyDeviceToHost));
    std::vector<int> perm;
    if (s.perm) {
      perm.resize(s.n_loc);
      KPM_CUDA(cudaMemcpy(perm.data(), s.perm, sizeof(int) * s.n_loc, cudaMemcpyDeviceToHost));
    }
    for (int64_t p = 0; p < s.n_loc; ++p) {
      const int64_t row = s.perm ? perm[p] : p;
      for (int r = 0; r < R; ++r) {
        w_out[2 * (row * R + r)] = wh[(size_t)p * R + r].x;
        w_out[2 * (row * R + r) + 1] = wh[(size_t)p * R + r].y;
      }
    }
  }
  return KPM_OK;
}

extern "C" kpm_status kpm_last_timing(const kpm_ctx* ctx, double* total_ms, double* sweep_ms, int* n_sweeps) {
  if (!ctx) return KPM_EINVAL;
  if (total_ms) *total_ms = ctx->last_total_ms;
  if (sweep_ms) *sweep_ms = ctx->last_sweep_ms;
  if (n_sweeps) *n_sweeps = ctx->last_n_sweeps;
  return KPM_OK;
}

extern "C" const char* kpm_last_kernel(const kpm_ctx* ctx) { return ctx ? ctx->last_variant.c_str() : ""; }

extern "C" const char* kpm_variant_name(int R, int variant) { return kpm::variant_name(R, variant); }

extern "C" kpm_status kpm_get_sell_info(const kpm_ctx* ctx, kpm_sell_info* info) {
  if (!ctx || !info) return KPM_EINVAL;
  if (!ctx->have_matrix) return KPM_ESTATE;
  info->n_loc = ctx->sell.n_loc;
  info->n_pad = ctx->sell.n_pad;
  info->n_chunks = ctx->sell.n_chunks;
  info->n_slots = ctx->sell.n_slots;
  info->n_halo = ctx->sell.n_halo;
  info->C = ctx->opt.sell_C;
  info->sigma = ctx->opt.sell_sigma;
  return KPM_OK;
}

extern "C" kpm_status kpm_export_sell(const kpm_ctx* ctx_c, double* val, int32_t* col, int64_t* cptr, int32_t* perm,
                                      int64_t* halo) {
  kpm_ctx* ctx = const_cast<kpm_ctx*>(ctx_c);
  if (!ctx) return KPM_EINVAL;
  if (!ctx->have_matrix) return fail(ctx, KPM_ESTATE, "no matrix");
  KPM_CUDA(cudaSetDevice(ctx->opt.device));
  const DevSell& s = ctx->sell;
  if (val) KPM_CUDA(cudaMemcpy(val, s.val, sizeof(double2) * s.n_slots, cudaMemcpyDeviceToHost));
  if (col) KPM_CUDA(cudaMemcpy(col, s.col, sizeof(int) * s.n_slots, cudaMemcpyDeviceToHost));
  if (cptr) KPM_CUDA(cudaMemcpy(cptr, s.cptr, sizeof(int64_t) * (s.n_chunks + 1), cudaMemcpyDeviceToHost));
  if (perm && s.perm) KPM_CUDA(cudaMemcpy(perm, s.perm, sizeof(int) * s.n_loc, cudaMemcpyDeviceToHost));
  if (perm && !s.perm)
    for (int64_t p = 0; p < s.n_loc; ++p) perm[p] = (int32_t)p;  // sigma = 1: identity
  if (halo && !ctx->halo.empty()) std::memcpy(halo, ctx->halo.data(), sizeof(int64_t) * ctx->halo.size());
  return KPM_OK;
}

extern "C" kpm_status kpm_last_sweep_times(const kpm_ctx* ctx, double* ms, int64_t* n) {
  if (!ctx || !n) return KPM_EINVAL;
  const int64_t have = (int64_t)ctx->sweep_times.size();
  if (ms) {
    const int64_t k = std::min(*n, have);
    std::memcpy(ms, ctx->sweep_times.data(), sizeof(double) * k);
    *n = k;
  } else {
    *n = have;
  }
  return KPM_OK;
}

extern "C" kpm_status kpm_export_halo(const kpm_ctx* ctx_c, int64_t* n_recv, int64_t* recv, int64_t* n_send,
                                      int64_t* send) {
  kpm_ctx* ctx = const_cast<kpm_ctx*>(ctx_c);
  if (!ctx || !n_recv || !n_send) return KPM_EINVAL;
  if (!ctx->have_matrix) return fail(ctx, KPM_ESTATE, "no matrix");
  const int64_t nr = (int64_t)ctx->recv_runs.size(), ns = (int64_t)ctx->send_runs.size();
  if (recv) {
    if (*n_recv < nr) return fail(ctx, KPM_EINVAL, "recv capacity too small");
    for (int64_t i = 0; i < nr; ++i) {
      const RecvRun& r = ctx->recv_runs[i];
      recv[4 * i] = r.peer, recv[4 * i + 1] = r.gfirst, recv[4 * i + 2] = r.count, recv[4 * i + 3] = r.slot;
    }
  }
  if (send) {
    if (*n_send < ns) return fail(ctx, KPM_EINVAL, "send capacity too small");
    for (int64_t i = 0; i < ns; ++i) {
      const SendRun& r = ctx->send_runs[i];
      send[4 * i] = r.peer, send[4 * i + 1] = r.pos, send[4 * i + 2] = r.count, send[4 * i + 3] = r.peer_slot;
    }
  }
  *n_recv = nr;
  *n_send = ns;
  return KPM_OK;
}
