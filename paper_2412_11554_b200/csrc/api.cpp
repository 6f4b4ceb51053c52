// Host driver of the ACCORD-FBS hot path: the C ABI of include/accord.h.
//
// One accord_ctx per rank owns the rank's row block of Omega (CSR), the
// replicated X (variable-major), the GEMM operand copies and all scratch.
// accord_step runs Algorithm 1:
//   GEMM + fused candidate epilogue (once per outer iteration; reading R3)
//   -> finalize C -> trial loop { prox(tau) -> SpMM -> reduce -> allreduce ->
//   host decision } -> compact Omega+, swap Y.
#include "accord_internal.h"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <map>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <chrono>
#include <mutex>
#include <new>
#include <thread>
#include <string>
#include <vector>

using namespace accord;

namespace {

thread_local std::string g_create_err;

struct Fail {
  accord_status s;
  std::string msg;
};

#define CK(call)                                                                      \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess)                                                            \
      throw Fail{e_ == cudaErrorMemoryAllocation ? ACCORD_E_NOMEM : ACCORD_E_CUDA,     \
                 std::string(#call) + ": " + cudaGetErrorString(e_)};                 \
  } while (0)

// --- NCCL, loaded lazily (the process may already hold torch's libnccl) -----
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t);
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t);
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t);
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  ncclResult_t (*CommDestroy)(ncclComm_t);
  const char* (*GetErrorString)(ncclResult_t);
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*);   // watchdog (may be NULL)
  ncclResult_t (*CommAbort)(ncclComm_t);
};

NcclApi* nccl_api() {
  static std::once_flag once;
  static NcclApi api;
  static bool ok = false;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
#define SYM(name) api.name = (decltype(api.name))dlsym(h, "nccl" #name)
    SYM(GetUniqueId); SYM(CommInitRank); SYM(AllReduce); SYM(AllGather); SYM(Broadcast);
    SYM(GroupStart); SYM(GroupEnd); SYM(CommDestroy); SYM(GetErrorString);
    SYM(Send); SYM(Recv); SYM(CommSplit);   // ring of the sharded mode (checked at use)
    SYM(CommGetAsyncError); SYM(CommAbort);
#undef SYM
    ok = api.GetUniqueId && api.CommInitRank && api.AllReduce && api.AllGather &&
         api.Broadcast && api.GroupStart && api.GroupEnd && api.CommDestroy &&
         api.GetErrorString;
  });
  return ok ? &api : nullptr;
}

#define NK(call)                                                                  \
  do {                                                                            \
    ncclResult_t r_ = (call);                                                     \
    if (r_ != ncclSuccess)                                                        \
      throw Fail{ACCORD_E_NCCL, std::string(#call) + ": " + nccl_api()->GetErrorString(r_)}; \
  } while (0)

// Caller-owned workspace (accord_init_params.workspace): every device buffer
// of the context is carved out of it, first fit with 256-B alignment, freed
// blocks coalesced. The library then never calls cudaMalloc; a request that
// does not fit is ACCORD_E_CAPACITY with the size asked for.
struct Arena {
  char* base = nullptr;
  size_t size = 0, in_use = 0, high = 0;
  std::map<size_t, size_t> free_, used_;   // offset -> length
  void init(void* b, size_t s) {
    const uintptr_t a = ((uintptr_t)b + 255) & ~(uintptr_t)255;
    base = (char*)a;
    size = s > (a - (uintptr_t)b) ? (s - (a - (uintptr_t)b)) & ~(size_t)255 : 0;
    if (size) free_[0] = size;
  }
  void* alloc(size_t b) {
    b = (std::max<size_t>(b, 1) + 255) & ~(size_t)255;
    for (auto it = free_.begin(); it != free_.end(); ++it) {
      if (it->second < b) continue;
      const size_t off = it->first, len = it->second;
      free_.erase(it);
      if (len > b) free_[off + b] = len - b;
      used_[off] = b;
      in_use += b;
      high = std::max(high, in_use);
      return base + off;
    }
    return nullptr;
  }
  bool release(void* p) {
    if (!base || (char*)p < base || (char*)p >= base + size) return false;
    auto it = used_.find((size_t)((char*)p - base));
    if (it == used_.end()) return false;
    size_t off = it->first, len = it->second;
    used_.erase(it);
    in_use -= len;
    auto nx = free_.lower_bound(off);
    if (nx != free_.end() && off + len == nx->first) {
      len += nx->second;
      nx = free_.erase(nx);
    }
    if (nx != free_.begin()) {
      auto pv = std::prev(nx);
      if (pv->first + pv->second == off) {
        pv->second += len;
        return true;
      }
    }
    free_[off] = len;
    return true;
  }
  size_t largest_free() const {
    size_t m = 0;
    for (auto& f : free_) m = std::max(m, f.second);
    return m;
  }
};

}  // namespace

struct accord_ctx {
  int device = 0;
  cudaStream_t st = nullptr;
  int sm_count = 0, cc_major = 0, cc_minor = 0;
  int64_t n = 0, p = 0, r0 = 0, r1 = 0, pk = 0, ldk = 0, p_pad = 0, pk_pad = 0;
  int dtype = ACCORD_F32;
  size_t tsz = 4;
  int gemm = ACCORD_GEMM_SIMT;
  double lam = 0, tau0 = 0, beta = 0, inv_L = 0, L = 0;
  int rank = 0, world = 1, comm = ACCORD_COMM_NONE;
  accord_allreduce_fn ar = nullptr;
  accord_allgatherv_fn agv = nullptr;
  void* cu = nullptr;
  ncclComm_t nccl = nullptr;

  // X sharded by variables (NEXT(3), 1DMM ring of Alg. 2): Xt holds this
  // rank's slab (columns [r0, r1)); vb[q] .. vb[q+1] is rank q's slab
  bool sharded = false;
  int64_t xrows_pad = 0;                   // rows of Xt / Xhi / Xlo
  std::vector<int64_t> vb;
  void* rbuf[2] = {nullptr, nullptr};      // ring buffers (f32/f64), max slab rows
  __nv_bfloat16* rhi[2] = {nullptr, nullptr};
  __nv_bfloat16* rlo[2] = {nullptr, nullptr};
  int64_t rrows_pad = 0;
  double *yacc = nullptr, *dacc = nullptr; // SpMM partial sums across the ring steps
  cudaStream_t cs = nullptr;               // ring transfers (NCCL)
  cudaEvent_t ev_comp[2] = {}, ev_recv[2] = {};
  ncclComm_t nccl_ring = nullptr;          // split communicator for the ring
  accord_sendrecv_fn sr = nullptr;
  void *h_send = nullptr, *h_recv = nullptr;   // pinned staging (ACCORD_COMM_HOST)
  int64_t ring_steps = 0;                  // slab exchanges so far (diagnostic)

  // work items (row chunks) of the current CSR for the TMA SpMM and the refine
  bool tma_spmm = false;
  int32_t *itm_n = nullptr, *itm_s = nullptr, *row_done = nullptr;
  int64_t *itm_ptr = nullptr, *slot_ptr = nullptr;
  double *part_y = nullptr, *part_d = nullptr, *part_d2 = nullptr;
  int64_t part_slots = 0, n_items = 0, n_slots = 0;
  double *itm_dd = nullptr, *itm_l1 = nullptr, *itm_logd = nullptr;   // per-item prox sums
  int32_t* itm_nnz = nullptr;
  int64_t itm_cap = 0;
  int32_t* item_row = nullptr;             // [itm_cap] item -> row
  const int64_t* items_of = nullptr;       // the CSR row_ptr the map was built for

  void* Xt = nullptr;
  __nv_bfloat16 *Xhi = nullptr, *Xlo = nullptr;
  void* Y[2] = {nullptr, nullptr};
  __nv_bfloat16* Yhi[2] = {nullptr, nullptr};
  __nv_bfloat16* Ylo[2] = {nullptr, nullptr};
  float* row_A[2] = {nullptr, nullptr};   // ||y_i - bf16(y_i)|| per Y buffer (filter bound)
  float* row_B[2] = {nullptr, nullptr};   // ||y_i||
  float2* col_sd = nullptr;               // per-column constants of the filter bound
  int cur = 0;
  // int8 GEMM operands (I8_FILTER, or AUTO's adaptive switch; gemm stays
  // BF16_FILTER internally: the same certified-filter pipeline)
  bool i8 = false;                         // int8 operands allocated
  bool i8_force = false;                   // I8_FILTER requested: every GEMM in int8
  bool i8_on = false;                      // the next GEMM in int8
  bool i8_last = false;                    // the last GEMM ran in int8 (filter audit)
  double i8_at = 48.0, i8_off = 384.0;     // AUTO: on at |C|/p <= i8_at (bf16), off above i8_off
  double i8_excess = 5e-4;                 // AUTO: off for good if int8 adds > i8_excess p^2 to |C|
  double i8_nnz = 256.0, i8_ccap = 512.0;  // AUTO: on at nnz/p <= i8_nnz with |C|/p <= i8_ccap
  bool i8_banned = false;
  // Y_hi / row_A / row_B of each Y buffer match its Y (the SpMM skips the bf16
  // operand while the int8 GEMM is on; a bf16 GEMM re-derives it first)
  bool yhi_ok[2] = {true, true};
  int64_t gemm_launches_i8 = 0;
  float2* col_sd_q = nullptr;              // int8 column constants of the bound
  float2* blk_q = nullptr;                 // their 256-column tile maxima
  int8_t* Xq = nullptr;                    // X^T int8, block scale per 256 variables
  float* xq_scale = nullptr;               // [p_pad / 256]
  int8_t* Yq[2] = {nullptr, nullptr};      // Y int8, per-row scale (quantised before each GEMM)
  float *yq_s[2] = {}, *yq_A[2] = {}, *yq_B[2] = {};
  int32_t* xperm = nullptr;                // [p_pad] Xq row k' holds variable xperm[k']

  int64_t cap = 0;  // entries of pool / C / keys / Omega arrays
  int64_t* om_ptr = nullptr;
  int32_t* om_col = nullptr;
  void* om_val = nullptr;
  int64_t* c_ptr = nullptr;
  int64_t* c_ptr2 = nullptr;               // C's row pointers after the support dedupe (swapped)
  int32_t* c_col = nullptr;
  void *c_g = nullptr, *c_w = nullptr, *c_wn = nullptr;
  void* c_wn2 = nullptr;                   // prox at the second step of a paired trial
  bool pair_ls = true;                     // paired line-search passes (ACCORD_LS_PAIRS=0: off)
  int refine_ff = 0;                       // 1: float-float refine (ACCORD_REFINE=ff; A-B, slower)
  int x_drop = 0;                          // mantissa bits dropped from X^T_hi (filter path)
  int x_drop_target = 0;                   // ACCORD_XDROP: width once |C| is small (A-B)
  int y_drop = 0, y_drop_target = 0;       // the same for the Y_hi operand (ACCORD_YDROP)
  double x_drop_at = 64.0;                 // ACCORD_XDROP_AT: switch at |C| / p below this
  bool omega_identity = false;             // Omega is exactly I (set at create, cleared on change)
  bool c_sym = false;                      // C = C^T from the symmetric first GEMM (sym 1)
  double *row_dd2 = nullptr, *row_l1_2 = nullptr, *row_logd2 = nullptr, *row_D2b = nullptr;
  double *diag_xx = nullptr, *diag_xz = nullptr, *diag_zz = nullptr, *diag_a = nullptr;
  int32_t* row_nnz2 = nullptr;
  uint64_t *keys = nullptr, *keys_tmp = nullptr;
  int32_t *pool_row = nullptr, *pool_col = nullptr;
  void *pool_g = nullptr, *pool_w = nullptr;
  int32_t *row_cnt = nullptr, *rcur = nullptr, *long_rows = nullptr;
  unsigned int* chunk_next = nullptr;      // pool chunks handed out (device counter)
  unsigned long long* chunk_fill = nullptr;   // [nchunks] entries per chunk
  int64_t chunk = 0, nchunks = 0;          // pool chunking (see PoolView)
  int gemm_warps = 0;                      // epilogue warps of the tcgen05 GEMM (0 = SIMT)
  double *row_D2 = nullptr, *row_Y2 = nullptr, *row_dd = nullptr, *row_l1 = nullptr,
         *row_logd = nullptr;
  int32_t* row_nnz = nullptr;
  double* red_d = nullptr;
  int32_t* bad_diag = nullptr;
  void* scan_tmp = nullptr;
  size_t scan_tmp_sz = 0;
  double* h_red = nullptr;                 // pinned [16]
  unsigned long long* h_seg = nullptr;     // pinned [2]: chunks handed out, chunk_fill[0]
  TcGemmPlan* plan = nullptr;
  cudaEvent_t ev[8] = {};
  float* audit_acc = nullptr;              // accord_filter_audit (diagnostic)
  int64_t audit_ld = 0;
  bool plan_a_x = false;                   // plan A map 2 = X^T_hi rows (lambda_max)
  int lanczos_steps = 0;                   // diagnostic (ACCORD_TRACE)
  // symmetric first GEMM across ranks (EpiParams::sym = 2)
  bool sym2_ok = false;                    // every rank's block starts on a 256-row tile
  std::vector<int64_t> rb;                 // all ranks' global row boundaries [world + 1]
  int64_t* rb_dev = nullptr;
  int32_t *mir_row = nullptr, *mir_col = nullptr, *mir_send = nullptr, *mir_recv = nullptr;
  unsigned long long* mir_cnt = nullptr;   // [1 + 2 world]: written, per-owner counts, cursors
  int64_t mir_cap = 0, mir_recv_cap = 0, mir_recv_n = 0;
  int64_t mirrored_sent = 0;               // cumulative (diagnostic, accord_info)

  // bias-correction refit (Eq. 3.8): fixed support S_hat, penalty phi * lambda
  bool refit = false;
  double phi = 1.0;
  int64_t* refit_ptr = nullptr;
  int32_t* refit_col = nullptr;
  int64_t refit_nnz = 0;
  // optional per-kernel tracing (ACCORD_TRACE=1): events after each launch,
  // printed to stderr at the end of every iteration
  bool trace = false;
  std::vector<cudaEvent_t> tr_pool;
  std::vector<std::pair<const char*, cudaEvent_t>> tr_marks;
  int64_t launches = 0, gemm_launches = 0, iters = 0, nnz_local = 0, nnz_global = 0;
  double f = 0, parts[3] = {0, 0, 0};
  std::vector<void*> allocs;
  size_t bytes = 0;
  Arena arena;                             // caller-owned workspace (empty: cudaMalloc)
  std::string err;

  void* dalloc_bytes(size_t b) {
    void* ptr = nullptr;
    b = std::max<size_t>(b, 1);
    if (arena.base) {
      ptr = arena.alloc(b);
      if (!ptr) {
        char m[200];
        std::snprintf(m, sizeof m,
                      "workspace exhausted: %zu more bytes needed (%zu of %zu in use, largest "
                      "free block %zu); recreate with a larger workspace",
                      b, arena.in_use, arena.size, arena.largest_free());
        throw Fail{ACCORD_E_CAPACITY, m};
      }
    } else {
      CK(cudaMalloc(&ptr, b));
    }
    allocs.push_back(ptr);
    bytes += b;
    return ptr;
  }
  template <typename T>
  T* dalloc(size_t count) {
    return (T*)dalloc_bytes(std::max<size_t>(count, 1) * sizeof(T));
  }
  void dfree(void* ptr, size_t b) {
    if (!ptr) return;
    auto it = std::find(allocs.begin(), allocs.end(), ptr);
    if (it != allocs.end()) allocs.erase(it);
    if (!arena.release(ptr)) cudaFree(ptr);
    bytes -= std::min(bytes, b);
  }
};

namespace {

// Host wait for the stream. With NCCL this is a watchdog: poll the stream and
// the communicators' asynchronous error state, and give up after
// ACCORD_NCCL_TIMEOUT_S seconds (default 1800) -- a dead or diverged rank
// otherwise hangs every survivor in cudaStreamSynchronize forever. On either
// failure the communicators are aborted (they cannot be reused) and the call
// returns ACCORD_E_NCCL.
double nccl_timeout_s() {
  const char* e = std::getenv("ACCORD_NCCL_TIMEOUT_S");
  const double v = e ? std::atof(e) : 0.0;
  return v > 0 ? v : 1800.0;
}

void nccl_abort(accord_ctx* c) {
  NcclApi* api = nccl_api();
  if (!api || !api->CommAbort) return;
  if (c->nccl_ring) api->CommAbort(c->nccl_ring);
  if (c->nccl) api->CommAbort(c->nccl);
  c->nccl_ring = nullptr;
  c->nccl = nullptr;
}

void csync(accord_ctx* c, cudaStream_t s) {
  if (c->comm != ACCORD_COMM_NCCL || !c->nccl) {
    CK(cudaStreamSynchronize(s));
    return;
  }
  NcclApi* api = nccl_api();
  const auto t0 = std::chrono::steady_clock::now();
  const double limit = nccl_timeout_s();
  for (int spin = 0;; ++spin) {
    const cudaError_t q = cudaStreamQuery(s);
    if (q == cudaSuccess) return;
    if (q != cudaErrorNotReady) CK(q);
    if ((spin & 63) == 0) {
      for (ncclComm_t cm : {c->nccl, c->nccl_ring}) {
        if (!api->CommGetAsyncError) break;
        if (!cm) continue;
        ncclResult_t r = ncclSuccess;
        api->CommGetAsyncError(cm, &r);
        if (r != ncclSuccess && r != ncclInProgress) {
          const std::string m = std::string("NCCL asynchronous error: ") + api->GetErrorString(r);
          nccl_abort(c);
          throw Fail{ACCORD_E_NCCL, m};
        }
      }
      const double el =
          std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (el > limit) {
        nccl_abort(c);
        throw Fail{ACCORD_E_NCCL, "NCCL watchdog: stream not done after " +
                                      std::to_string((int)el) +
                                      " s (a peer rank died or diverged); communicators aborted"};
      }
    }
    if (spin > 2000) std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
}

void allreduce(accord_ctx* c, double* d_buf, double* h_buf, int count) {
  // d_buf (device) -> h_buf (host), summed over ranks. Synchronizes the stream.
  if (const char* h = std::getenv("ACCORD_DEBUG_STALL_MS"))   // test of the watchdog only:
    c->launches += launch_spin(std::atoi(h), c->st);           // a slow "peer" on the stream
  if (c->comm == ACCORD_COMM_NCCL) {   // (a 1-rank communicator is exercised by the tests)
    NK(nccl_api()->AllReduce(d_buf, d_buf, count, ncclDouble, ncclSum, c->nccl, c->st));
  }
  CK(cudaMemcpyAsync(h_buf, d_buf, count * sizeof(double), cudaMemcpyDeviceToHost, c->st));
  csync(c, c->st);
  if (c->world > 1 && c->comm == ACCORD_COMM_HOST) {
    if (c->ar(c->cu, h_buf, count) != 0) throw Fail{ACCORD_E_COMM, "host allreduce failed"};
  }
}

// Global maximum of one value per rank (KKT certificate).
double allreduce_max(accord_ctx* c, double* d_val) {
  double h = 0;
  if (c->comm == ACCORD_COMM_NCCL)
    NK(nccl_api()->AllReduce(d_val, d_val, 1, ncclDouble, ncclMax, c->nccl, c->st));
  CK(cudaMemcpyAsync(&h, d_val, 8, cudaMemcpyDeviceToHost, c->st));
  csync(c, c->st);
  if (c->world > 1 && c->comm == ACCORD_COMM_HOST) {
    std::vector<double> v(c->world, 0.0);
    v[c->rank] = h;
    if (c->ar(c->cu, v.data(), c->world) != 0) throw Fail{ACCORD_E_COMM, "host allreduce failed"};
    h = *std::max_element(v.begin(), v.end());
  }
  return h;
}

// Sum a device vector of doubles across ranks in place (stream-ordered for
// NCCL; the host transport synchronizes). Power iteration of the sharded mode.
void dev_allreduce(accord_ctx* c, double* d, int count) {
  if (c->world == 1) return;
  if (c->comm == ACCORD_COMM_NCCL) {
    NK(nccl_api()->AllReduce(d, d, count, ncclDouble, ncclSum, c->nccl, c->st));
    return;
  }
  std::vector<double> h(count);
  CK(cudaMemcpyAsync(h.data(), d, count * 8, cudaMemcpyDeviceToHost, c->st));
  csync(c, c->st);
  if (c->ar(c->cu, h.data(), count) != 0) throw Fail{ACCORD_E_COMM, "host allreduce failed"};
  CK(cudaMemcpyAsync(d, h.data(), count * 8, cudaMemcpyHostToDevice, c->st));
  csync(c, c->st);
}

OmegaView omega_view(accord_ctx* c) { return OmegaView{c->om_ptr, c->om_col, c->om_val}; }

PoolView pool_view(accord_ctx* c) {
  return PoolView{c->pool_row, c->pool_col, c->pool_g, c->pool_w, c->chunk, c->nchunks,
                  c->chunk_next, c->chunk_fill, c->row_cnt};
}

// ---- X sharded by variables: the ring over the slabs (NEXT(3), Alg. 2) ----
// At ring step s this rank holds slab j = (rank + s) mod P (the variables
// [vb[j], vb[j+1]) of X, variable-major); while step s computes on it, slab
// j+1 arrives from rank+1 and slab j leaves for rank-1 (the
// 1DMM rotation, here of the X slabs, since Omega's rows stay put). NCCL
// transfers run on their own stream and communicator and overlap the
// compute; the host-callback transport (tests) is synchronous.
int64_t slab_rows(const accord_ctx* c, int q) { return c->vb[q + 1] - c->vb[q]; }

void ring_exchange(accord_ctx* c, int s, const void* slab, int j) {
  const int P = c->world;
  const int jn = (j + 1) % P;
  const size_t sb = (size_t)slab_rows(c, j) * c->ldk * c->tsz;
  const size_t rb = (size_t)slab_rows(c, jn) * c->ldk * c->tsz;
  const int left = (c->rank + P - 1) % P, right = (c->rank + 1) % P;
  void* target = c->rbuf[s & 1];
  c->ring_steps++;
  if (c->comm == ACCORD_COMM_NCCL) {
    NcclApi* api = nccl_api();
    // rbuf[s & 1] was the resident slab of step s-1: wait until that step's
    // kernels (and its bf16 split) are done with it
    if (s >= 2) CK(cudaStreamWaitEvent(c->cs, c->ev_comp[s & 1], 0));
    NK(api->GroupStart());
    NK(api->Send(slab, sb, ncclChar, left, c->nccl_ring, c->cs));
    NK(api->Recv(target, rb, ncclChar, right, c->nccl_ring, c->cs));
    NK(api->GroupEnd());
    CK(cudaEventRecord(c->ev_recv[s & 1], c->cs));
  } else {
    CK(cudaMemcpyAsync(c->h_send, slab, sb, cudaMemcpyDeviceToHost, c->st));
    csync(c, c->st);
    if (c->sr(c->cu, c->h_send, (int64_t)sb, left, c->h_recv, (int64_t)rb, right) != 0)
      throw Fail{ACCORD_E_COMM, "host sendrecv failed"};
    CK(cudaMemcpyAsync(target, c->h_recv, rb, cudaMemcpyHostToDevice, c->st));
  }
}

// fn(slab, bsel, v0, v1, first, last): Xt rows of the columns [v0, v1) at
// `slab`; bsel = the GEMM B operand holding its bf16 copy (when want_bf16).
// Collective: every rank runs the P steps.
template <typename F>
void ring_pass(accord_ctx* c, bool want_bf16, F&& fn) {
  const int P = c->world;
  for (int s = 0; s < P; ++s) {
    const int j = (c->rank + s) % P;
    const void* slab = s == 0 ? c->Xt : c->rbuf[(s - 1) & 1];
    if (s + 1 < P) ring_exchange(c, s, slab, j);
    int bsel = 0;
    if (s > 0) {
      const int b = (s - 1) & 1;
      if (c->comm == ACCORD_COMM_NCCL) CK(cudaStreamWaitEvent(c->st, c->ev_recv[b], 0));
      if (want_bf16) {
        c->launches += launch_split_bf16((const float*)c->rbuf[b],
                                         round_up(slab_rows(c, j), kRowPad) * c->ldk, c->rhi[b],
                                         c->rlo[b], c->st);
        bsel = 1 + b;
      }
    }
    fn(slab, bsel, c->vb[j], c->vb[j + 1], s == 0, s == P - 1);
    if (s > 0 && c->comm == ACCORD_COMM_NCCL) CK(cudaEventRecord(c->ev_comp[(s - 1) & 1], c->st));
  }
}

// Work items of the CSR `ptr` (this rank's rows): one per row, hub rows split
// into chunks of kItemEntries; scratch for the split rows grown on demand.
// One small D2H (item and slot totals).
void build_items(accord_ctx* c, const int64_t* ptr) {
  c->launches += launch_item_map(c->pk, ptr, kItemEntries, c->itm_n, c->itm_s, c->itm_ptr,
                                 c->slot_ptr, c->scan_tmp, c->scan_tmp_sz, c->st);
  int64_t h[2] = {0, 0};
  CK(cudaMemcpyAsync(&h[0], c->itm_ptr + c->pk, 8, cudaMemcpyDeviceToHost, c->st));
  CK(cudaMemcpyAsync(&h[1], c->slot_ptr + c->pk, 8, cudaMemcpyDeviceToHost, c->st));
  csync(c, c->st);
  c->n_items = h[0];
  c->n_slots = h[1];
  if (c->tma_spmm && c->n_slots > c->part_slots) {
    const size_t b = (size_t)c->part_slots * c->ldk * 8;
    c->dfree(c->part_y, b);
    c->dfree(c->part_d, b);
    c->dfree(c->part_d2, b);
    c->part_slots = c->n_slots + c->n_slots / 4 + 16;
    c->part_y = c->dalloc<double>((size_t)c->part_slots * c->ldk);
    c->part_d = c->dalloc<double>((size_t)c->part_slots * c->ldk);
    c->part_d2 = c->dalloc<double>((size_t)c->part_slots * c->ldk);
  }
  if (c->n_items > c->itm_cap) {
    c->dfree(c->itm_dd, c->itm_cap * 8);
    c->dfree(c->itm_l1, c->itm_cap * 8);
    c->dfree(c->itm_logd, c->itm_cap * 8);
    c->dfree(c->itm_nnz, c->itm_cap * 4);
    c->dfree(c->item_row, c->itm_cap * 4);
    c->itm_cap = c->n_items + c->n_items / 8 + 1024;
    c->itm_dd = c->dalloc<double>(c->itm_cap);
    c->itm_l1 = c->dalloc<double>(c->itm_cap);
    c->itm_logd = c->dalloc<double>(c->itm_cap);
    c->itm_nnz = c->dalloc<int32_t>(c->itm_cap);
    c->item_row = c->dalloc<int32_t>(c->itm_cap);
  }
  c->launches += launch_item_rows(c->pk, c->itm_ptr, c->item_row, c->st);
  c->items_of = ptr;
}

SpmmItems items_view(accord_ctx* c) {
  return SpmmItems{c->itm_ptr, c->item_row, c->slot_ptr, c->part_y, c->part_d, c->part_d2,
                   c->row_done, kItemEntries};
}

// Does the next GEMM need Y's bf16 operand? Not while the int8 GEMM is on
// (it quantises Y itself); the SpMM then writes Y alone (ACCORD_SPMM_BF16=1:
// always write it, A-B).
bool want_yhi(accord_ctx* c) {
  static const bool always = [] {
    const char* e = std::getenv("ACCORD_SPMM_BF16");
    return e && e[0] == '1';
  }();
  return !(c->i8 && c->i8_on && c->y_drop == 0 && !c->sharded && !always);
}

// Y_hi, row_A, row_B of buffer b from its Y (after SpMM passes that skipped
// them), before a bf16 GEMM
void ensure_yhi(accord_ctx* c, int b) {
  if (c->yhi_ok[b] || !c->Yhi[b]) return;
  c->launches += launch_split_bf16((const float*)c->Y[b], c->pk_pad * c->ldk, c->Yhi[b], nullptr,
                                   c->st);
  c->launches += launch_row_ab(c->pk, c->ldk, (const float*)c->Y[b], c->row_A[b], c->row_B[b],
                               c->st, 0);
  c->yhi_ok[b] = true;
}

// SpMM Y+ = W X^T (and D = (W - Wold) X^T) over all of X: one launch, or a
// ring pass accumulating in float64 when X is sharded.
void spmm_all(accord_ctx* c, const int64_t* ptr, const int32_t* col, const void* wn,
              const void* wo, int yb, double* row_D2, double* row_Y2) {
  const bool hi = want_yhi(c) && c->Yhi[yb];
  c->yhi_ok[yb] = hi || !c->Yhi[yb];
  if (!c->sharded && c->tma_spmm) {
    if (c->items_of != ptr) build_items(c, ptr);
    c->launches += launch_spmm_tma(c->pk, c->ldk, ptr, col, (const float*)wn, (const float*)wo,
                                   (const float*)c->Xt, (float*)c->Y[yb],
                                   hi ? c->Yhi[yb] : nullptr, hi ? c->Ylo[yb] : nullptr,
                                   c->row_A[yb], c->row_B[yb], row_D2, row_Y2, items_view(c),
                                   c->sm_count, c->st, nullptr, nullptr, c->y_drop);
    return;
  }
  if (!c->sharded) {
    c->launches += launch_spmm(c->dtype, c->pk, c->n, c->ldk, ptr, col, wn, wo, c->Xt, c->Y[yb],
                               hi ? c->Yhi[yb] : nullptr, hi ? c->Ylo[yb] : nullptr, c->row_A[yb],
                               c->row_B[yb], row_D2, row_Y2, c->st, nullptr, c->y_drop);
    return;
  }
  ring_pass(c, false, [&](const void* slab, int, int64_t v0, int64_t v1, bool first, bool last) {
    SpmmRing rg{v0, v1, c->yacc, c->dacc, first ? 1 : 0, last ? 1 : 0};
    c->launches += launch_spmm(c->dtype, c->pk, c->n, c->ldk, ptr, col, wn, wo, slab, c->Y[yb],
                               c->Yhi[yb], c->Ylo[yb], c->row_A[yb], c->row_B[yb], row_D2,
                               row_Y2, c->st, &rg, c->y_drop);
  });
}

// Exact candidate values c_g = (1/n) <Y_i, X_k> over all of X (Y = the
// current Y buffer, or `yrows` = the rank's rows of X^T for lambda_max).
void refine_all(accord_ctx* c, const void* yrows = nullptr) {
  const void* Y = yrows ? yrows : c->Y[c->cur];
  if (!c->sharded) {
    // hub rows (up to ~1.6e5 candidates) split over several work items
    if (c->items_of != c->c_ptr) build_items(c, c->c_ptr);
    // C = C^T at Omega = I (Y = X^T, G = S): half the gathers, the rest mirrored
    // (ACCORD_REFINE_NOSYM: off; ACCORD_DEBUG_MIRROR_MISS: every twin looked up
    // is treated as missing, a test of the fallback)
    const int sym = c->c_sym && !yrows && !std::getenv("ACCORD_REFINE_NOSYM")
                        ? (std::getenv("ACCORD_DEBUG_MIRROR_MISS") ? 2 : 1)
                        : 0;
    c->launches += launch_refine(c->dtype, c->pk, c->n, c->ldk, c->c_ptr, c->c_col, Y, c->Xt,
                                 c->c_g, c->st, 0, INT64_MAX, c->itm_ptr, c->n_items,
                                 kItemEntries, c->item_row, c->refine_ff, sym);
    return;
  }
  ring_pass(c, false, [&](const void* slab, int, int64_t v0, int64_t v1, bool, bool) {
    c->launches += launch_refine(c->dtype, c->pk, c->n, c->ldk, c->c_ptr, c->c_col, Y, slab,
                                 c->c_g, c->st, v0, v1, nullptr, 0, 0, nullptr,
                                 c->refine_ff);
  });
}

// Candidate-indexed arrays (C, sort keys, pool) at capacity `cap`; on an
// allocation failure the ones allocated are released and the error rethrown.
void alloc_entry_arrays(accord_ctx* c, int64_t cap) {
  const size_t T = c->tsz;
  const bool vals = c->gemm != ACCORD_GEMM_BF16_FILTER;   // the filter emits positions only
  int64_t ch = cap, nch = 1;
  if (c->gemm_warps != 0) {
    // the tcgen05 epilogue warps take private chunks of 2048..8192 entries
    // (>= one emission batch: 32 rows x 32 columns, twice that when the
    // symmetric first GEMM mirrors its survivors); SIMT: one chunk
    ch = 8192;
    while (ch > 2048 && cap / ch < 4 * (int64_t)c->gemm_warps) ch >>= 1;
    nch = std::max<int64_t>(1, cap / ch);
  }
  struct A {
    void** dst;
    size_t bytes;
  } list[] = {{(void**)&c->c_col, (size_t)cap * 4},      {(void**)&c->c_g, (size_t)cap * T},
              {(void**)&c->c_w, (size_t)cap * T},        {(void**)&c->c_wn, (size_t)cap * T},
              {(void**)&c->c_wn2, (size_t)cap * T},      {(void**)&c->keys, (size_t)cap * 8},
              {(void**)&c->keys_tmp, (size_t)cap * 8},   {(void**)&c->pool_row, (size_t)cap * 4},
              {(void**)&c->pool_col, (size_t)cap * 4},
              {(void**)&c->pool_g, vals ? (size_t)cap * T : 0},
              {(void**)&c->pool_w, vals ? (size_t)cap * T : 0},
              {(void**)&c->chunk_fill, (size_t)nch * 8}};
  size_t k = 0;
  try {
    for (; k < sizeof(list) / sizeof(list[0]); ++k)
      *list[k].dst = list[k].bytes ? c->dalloc_bytes(list[k].bytes) : nullptr;
  } catch (...) {
    for (size_t j = 0; j < k; ++j) {
      c->dfree(*list[j].dst, list[j].bytes);
      *list[j].dst = nullptr;
    }
    throw;
  }
  c->chunk = ch;
  c->nchunks = nch;
}

void free_entry_arrays(accord_ctx* c, int64_t cap) {
  const size_t T = c->tsz;
  c->dfree(c->c_col, cap * 4);     c->c_col = nullptr;
  c->dfree(c->c_g, cap * T);       c->c_g = nullptr;
  c->dfree(c->c_w, cap * T);       c->c_w = nullptr;
  c->dfree(c->c_wn, cap * T);      c->c_wn = nullptr;
  c->dfree(c->c_wn2, cap * T);     c->c_wn2 = nullptr;
  c->dfree(c->keys, cap * 8);      c->keys = nullptr;
  c->dfree(c->keys_tmp, cap * 8);  c->keys_tmp = nullptr;
  c->dfree(c->pool_row, cap * 4);  c->pool_row = nullptr;
  c->dfree(c->pool_col, cap * 4);  c->pool_col = nullptr;
  c->dfree(c->pool_g, cap * T);    c->pool_g = nullptr;
  c->dfree(c->pool_w, cap * T);    c->pool_w = nullptr;
  c->dfree(c->chunk_fill, c->nchunks * 8);
  c->chunk_fill = nullptr;
}

// (Re)allocate the entry-indexed arrays for capacity `cap`, preserving Omega.
// Transactional: if the new arrays do not fit (a caller workspace that is too
// small), the context keeps a valid state at the old capacity and the error
// (ACCORD_E_CAPACITY / NOMEM) propagates; nothing of the iterate is lost.
void grow(accord_ctx* c, int64_t cap, int64_t keep_nnz) {
  const size_t T = c->tsz;
  const int64_t oc = c->cap;
  // Omega first, copied (the old arrays stay until the new ones exist)
  int32_t* om_col = c->dalloc<int32_t>(cap);
  void* om_val = nullptr;
  try {
    om_val = c->dalloc_bytes(cap * T);
  } catch (...) {
    c->dfree(om_col, cap * 4);
    throw;
  }
  if (c->om_col && keep_nnz > 0) {
    CK(cudaMemcpyAsync(om_col, c->om_col, keep_nnz * 4, cudaMemcpyDeviceToDevice, c->st));
    CK(cudaMemcpyAsync(om_val, c->om_val, keep_nnz * T, cudaMemcpyDeviceToDevice, c->st));
  }
  csync(c, c->st);
  c->dfree(c->om_col, oc * 4);
  c->dfree(c->om_val, oc * T);
  c->om_col = om_col;
  c->om_val = om_val;
  // C / keys / pool: contents are rebuilt by the next GEMM
  if (oc > 0) free_entry_arrays(c, oc);
  try {
    alloc_entry_arrays(c, cap);
  } catch (...) {
    if (oc > 0) alloc_entry_arrays(c, oc);   // the blocks just freed: fits again
    c->cap = oc;                              // (Omega's arrays are larger: fine)
    throw;
  }
  c->cap = cap;
}

// Objective and nnz of the current Omega (collective). Y[cur] must be current
// and row_Y2 must hold ||Y_i||^2.
void refresh_objective(accord_ctx* c) {
  CK(cudaMemsetAsync(c->bad_diag, 0, 4, c->st));
  c->launches += launch_omega_stats(c->dtype, c->pk, c->r0, c->om_ptr, c->om_col, c->om_val,
                                    c->row_l1, c->row_logd, c->row_nnz, c->bad_diag, c->st);
  c->launches += launch_reduce_rows(c->pk, nullptr, nullptr, c->row_logd, c->row_Y2, c->row_l1,
                                    c->row_nnz, nullptr, c->red_d, c->st);
  int32_t bad = 0;
  double loc[8];
  CK(cudaMemcpyAsync(&bad, c->bad_diag, 4, cudaMemcpyDeviceToHost, c->st));
  CK(cudaMemcpyAsync(loc, c->red_d, sizeof(loc), cudaMemcpyDeviceToHost, c->st));
  csync(c, c->st);
  c->nnz_local = (int64_t)loc[5];
  loc[7] = bad ? 1.0 : 0.0;   // make the domain check collective
  CK(cudaMemcpyAsync(c->red_d, loc, sizeof(loc), cudaMemcpyHostToDevice, c->st));
  allreduce(c, c->red_d, c->h_red, 8);
  const bool bad_any = c->h_red[7] > 0;
  c->nnz_global = (int64_t)c->h_red[5];
  const double* r = c->h_red;
  c->parts[0] = -r[2];
  c->parts[1] = r[3] / (2.0 * (double)c->n);
  c->parts[2] = (c->refit ? c->phi * c->lam : c->lam) * r[4];
  c->f = c->parts[0] + c->parts[1] + c->parts[2];
  if (bad_any) throw Fail{ACCORD_E_DOMAIN, "Omega has a missing or nonpositive diagonal entry"};
}

// Y = Omega X^T for the current Omega into Y[cur] (+ row norms).
void recompute_y(accord_ctx* c) {
  c->omega_identity = false;   // every change of Omega comes through here
  c->items_of = nullptr;   // Omega's structure may have been replaced (warm start, path)
  spmm_all(c, c->om_ptr, c->om_col, c->om_val, nullptr, c->cur, nullptr, c->row_Y2);
}

void validate(const accord_init_params* prm) {
  auto bad = [](const std::string& m) { throw Fail{ACCORD_E_INVALID, m}; };
  if (!prm) bad("params is NULL");
  if (prm->abi_version != ACCORD_ABI_VERSION) bad("abi_version mismatch");
  if (prm->n < 1 || prm->p < 1) bad("need n >= 1 and p >= 1");
  if (prm->p > INT32_MAX - 1024) bad("p too large for int32 column indices");
  if (!prm->X) bad("X is NULL");
  if (prm->dtype != ACCORD_F32 && prm->dtype != ACCORD_F64) bad("dtype must be F32 or F64");
  if (prm->layout != ACCORD_LAYOUT_SAMPLES_ROW_MAJOR &&
      prm->layout != ACCORD_LAYOUT_VARIABLES_ROW_MAJOR)
    bad("bad layout");
  const bool shard = prm->x_sharded && prm->world > 1;
  const int64_t pv = shard ? prm->row_end - prm->row_begin : prm->p;   // variables held
  const int64_t minld = prm->layout == ACCORD_LAYOUT_SAMPLES_ROW_MAJOR ? pv : prm->n;
  if (prm->ldx != 0 && prm->ldx < minld) bad("ldx smaller than the row length");
  if (!(prm->lambda >= 0) || !std::isfinite(prm->lambda)) bad("lambda must be finite and >= 0");
  if (!(prm->tau0 > 0) || !std::isfinite(prm->tau0)) bad("tau0 must be > 0");
  if (!(prm->beta > 0 && prm->beta <= 1)) bad("beta must be in (0, 1]");
  if (!(prm->inv_L >= 0) || !std::isfinite(prm->inv_L)) bad("inv_L must be >= 0");
  if (prm->row_begin < 0 || prm->row_end > prm->p || prm->row_begin >= prm->row_end)
    bad("bad row range");
  if (prm->world < 1 || prm->rank < 0 || prm->rank >= prm->world) bad("bad rank/world");
  if (prm->world > 1 && prm->comm == ACCORD_COMM_NONE) bad("world > 1 needs a communicator");
  if (prm->comm == ACCORD_COMM_NCCL && !prm->nccl_id) bad("nccl_id is NULL");
  if (prm->comm == ACCORD_COMM_HOST && !prm->allreduce) bad("allreduce callback is NULL");
  if (shard && prm->comm == ACCORD_COMM_HOST && !prm->sendrecv)
    bad("x_sharded with the host communicator needs a sendrecv callback");

  if (prm->gemm < ACCORD_GEMM_AUTO || prm->gemm > ACCORD_GEMM_I8_FILTER) bad("bad gemm kind");
  if (prm->dtype == ACCORD_F64 &&
      (prm->gemm == ACCORD_GEMM_BF16X3 || prm->gemm == ACCORD_GEMM_BF16_FILTER ||
       prm->gemm == ACCORD_GEMM_I8_FILTER))
    bad("tensor-core GEMM kinds need dtype F32");
  if (prm->gemm == ACCORD_GEMM_I8_FILTER && shard)
    bad("I8_FILTER needs X replicated (x_sharded uses BF16_FILTER)");
  if (prm->gemm == ACCORD_GEMM_I8_FILTER && prm->n >= 133000)
    bad("I8_FILTER needs n < 133000 (exact s32 accumulation)");
}

// Default candidate-pool capacity (entries): the first iteration (G = S) has
// the most candidates (config 5: ~380 per row), so size for ~512 per row; at
// least 2 M entries (104 MB), which small problems whose int8 filter admits
// more than 512 per row need (config 2 at lambda = 0.1: ~1.3 M)
int64_t default_capacity(int64_t pk, int64_t p) {
  const int64_t dense = pk * p;
  int64_t cap = std::min<int64_t>(dense, std::max<int64_t>(pk * 512, 1 << 21));
  return std::max<int64_t>(cap, std::min<int64_t>(dense, pk * 16));
}

// Device bytes accord_create takes for `prm` (mirrors create_impl buffer by
// buffer, each rounded to the 256-B arena granule), for the workspace query.
// Pure host arithmetic: no CUDA call. Upper bound: AUTO is resolved as on an
// sm_100 device (tensor-core operand copies), the sharded ring buffers assume
// no rank's slab exceeds max(p_k, ceil(p / world)) rows, and the per-iteration
// scratch of hub rows (work items split at kItemEntries) is reserved for
// 64 + p_k / 64 split slots.
// The GEMM kind a create resolves to (AUTO: F32 on sm_100 -> the certified
// filter, I8 operands unless X is sharded; else SIMT).
// Order of the variables in the int8 X^T (quant_i8.cu): a stable counting
// sort by log2 max|x_k| in 1/32-octave buckets, so each 256-variable block
// (one block scale) holds nearly equal maxima; deterministic (ties keep the
// variable order). Entries [p, p_pad) are the padding rows themselves.
std::vector<int32_t> scale_permutation(const std::vector<float>& mx, int64_t p_pad) {
  const int64_t p = (int64_t)mx.size();
  constexpr int kB = 32 * 160;                      // 2^-80 .. 2^80
  std::vector<int32_t> key(p);
  std::vector<int64_t> cnt(kB + 1, 0);
  for (int64_t k = 0; k < p; ++k) {
    const float m = mx[k];
    int b = 0;
    if (m > 0.f && std::isfinite(m))
      b = std::clamp((int)std::floor(32.0 * std::log2((double)m)) + kB / 2, 1, kB - 1);
    key[k] = b;
    cnt[b + 1]++;
  }
  for (int b = 0; b < kB; ++b) cnt[b + 1] += cnt[b];
  std::vector<int32_t> perm(p_pad);
  for (int64_t k = 0; k < p; ++k) perm[cnt[key[k]]++] = (int32_t)k;
  for (int64_t k = p; k < p_pad; ++k) perm[k] = (int32_t)k;
  return perm;
}

// *i8_ops: int8 operands are allocated (I8_FILTER, or AUTO's adaptive
// bf16 -> int8 switch; ACCORD_AUTO_GEMM=bf16 turns the switch off).
int resolve_gemm(const accord_init_params* prm, bool tc_ok, bool* i8_ops) {
  const bool sharded = prm->x_sharded && prm->world > 1;
  *i8_ops = prm->gemm == ACCORD_GEMM_I8_FILTER;
  if (prm->gemm != ACCORD_GEMM_AUTO) return prm->gemm;
  if (prm->dtype != ACCORD_F32 || !tc_ok) return ACCORD_GEMM_SIMT;
  const char* e = std::getenv("ACCORD_AUTO_GEMM");   // A-B: "bf16" = no int8 switch
  *i8_ops = !sharded && !(e && std::strcmp(e, "bf16") == 0);
  return ACCORD_GEMM_BF16_FILTER;
}

struct Footprint {
  size_t total = 0, transient = 0;
  int64_t cap = 0;
};
Footprint footprint(const accord_init_params* prm) {
  auto R = [](size_t b) { return (std::max<size_t>(b, 1) + 255) & ~(size_t)255; };
  Footprint f;
  const int64_t n = prm->n, p = prm->p, pk = prm->row_end - prm->row_begin;
  const int64_t ldk = round_up(n, kKPad), p_pad = round_up(p, kRowPad),
                pk_pad = round_up(pk, kRowPad);
  const size_t T = prm->dtype == ACCORD_F64 ? 8 : 4;
  const bool sharded = prm->x_sharded && prm->world > 1;
  bool i8 = false;
  const int gemm = resolve_gemm(prm, true, &i8);
  const bool x3 = gemm == ACCORD_GEMM_BF16X3,
             filt = gemm == ACCORD_GEMM_BF16_FILTER || gemm == ACCORD_GEMM_I8_FILTER,
             tc = x3 || filt;
  const int64_t pv = sharded ? pk : p;
  const int64_t xrows_pad = sharded ? pk_pad : p_pad;
  size_t a = 0;
  a += R(16 * 8);                                      // red_d
  a += R((size_t)xrows_pad * ldk * T);                 // Xt
  a += R(8);                                           // bad index
  // transient: host staging of X, or the Lanczos vectors (freed before Y)
  size_t tr = 0;
  if (!prm->x_on_device) {
    tr = R((size_t)n * pv * T);
  }
  if (!(prm->inv_L > 0)) {
    const int64_t nsplit = std::min<int64_t>(256, std::max<int64_t>(1, pv / 256));
    tr = std::max(tr, 2 * R(ldk * 8) + R(std::max<int64_t>(pv, 1) * 8) + R(nsplit * ldk * 8));
  }
  a += 2 * R((size_t)pk_pad * ldk * T);                // Y (x2)
  if (tc) {
    a += R((size_t)xrows_pad * ldk * 2) * (x3 ? 2 : 1); // X^T bf16 (hi, lo)
    a += 2 * R((size_t)pk_pad * ldk * 2) * (x3 ? 2 : 1); // Y bf16 (x2)
    a += 4 * R(pk * 4);                                // row_A, row_B (x2)
    if (filt) a += R(p * 8);                           // col_sd
    a += R((p_pad / kRowPad) * 8);                     // tile maxima of col_sd
  }
  if (i8) {
    a += R((size_t)xrows_pad * ldk) + R((p_pad / kRowPad) * 4);   // X^T int8, block scales
    a += R(p * 8) + R((p_pad / kRowPad) * 8) + R(p_pad * 4);      // int8 col_sd, tile maxima, perm
    a += R(p * 4);                                               // max |x_k| (transient)
    a += 2 * R((size_t)pk_pad * ldk) + 6 * R(pk * 4);            // Y int8 (x2), row consts
  }
  if (sharded) {
    const int64_t rr = std::max(pk_pad, round_up((p + prm->world - 1) / prm->world, kRowPad));
    a += 2 * R((size_t)rr * ldk * T);                  // ring buffers
    if (tc) a += 2 * R((size_t)rr * ldk * 2) * (x3 ? 2 : 1);
    a += 2 * R((size_t)pk_pad * ldk * 8);              // yacc, dacc
  }
  a += 3 * R((pk + 1) * 8) + 2 * R(pk * 4) + R((pk + 1) * 4) + R(4);   // om/c ptr, counts
  a += 9 * R(pk * 8) + 2 * R(pk * 4) + 4 * R(pk * 8) + R(4);          // per-row sums
  a += R(scan_tmp_bytes(pk + 1));
  a += 2 * R(pk * 4) + 2 * R((pk + 1) * 8) + R(pk * 4);               // work-item maps
  const int64_t cap = std::min<int64_t>(prm->cand_capacity > 0 ? std::max(prm->cand_capacity, pk)
                                                               : default_capacity(pk, p),
                                        (int64_t)UINT32_MAX);
  f.cap = cap;
  size_t pool = R(cap * 4) + R(cap * T)                // Omega col, val
                + R(cap * 4) + 4 * R(cap * T)          // C col, g, w, w+, w+'
                + 2 * R(cap * 8)                       // sort keys
                + 2 * R(cap * 4)                       // pool positions
                + (filt ? 0 : 2 * R(cap * T))          // pool values (BF16X3, SIMT)
                + R((cap / 2048 + 1) * 8);             // chunk fill counts
  a += pool;
  // work items of C: <= p_k + cap / L items; split-row slots reserved
  const int64_t items = pk + cap / kItemEntries + 1024;
  a += 3 * R(items * 8) + 2 * R(items * 4);
  const bool tma = !sharded && spmm_tma_supported(prm->dtype, ldk) && pk >= 65536 &&
                   ldk % 256 == 0;   // mirrors create_impl's choice
  if (tma || std::getenv("ACCORD_SPMM_TMA")) a += 3 * R((size_t)(64 + pk / 64) * ldk * 8);
  f.transient = tr;
  f.total = a + tr;
  return f;
}

// All ranks' per-column filter constants into every rank's col_sd[p]
// (sharded mode; each rank computed its slab's at col_sd + r0).
void gather_col_sd(accord_ctx* c) {
  const int P = c->world;
  if (c->comm == ACCORD_COMM_NCCL) {
    NcclApi* api = nccl_api();
    NK(api->GroupStart());
    for (int q = 0; q < P; ++q)
      NK(api->Broadcast(c->col_sd + c->vb[q], c->col_sd + c->vb[q],
                        (size_t)slab_rows(c, q) * sizeof(float2), ncclChar, q, c->nccl, c->st));
    NK(api->GroupEnd());
    csync(c, c->st);
    return;
  }
  if (!c->agv) throw Fail{ACCORD_E_INVALID, "x_sharded with host comm needs allgatherv"};
  std::vector<float2> mine(c->pk), all(c->p);
  CK(cudaMemcpyAsync(mine.data(), c->col_sd + c->r0, c->pk * sizeof(float2),
                     cudaMemcpyDeviceToHost, c->st));
  csync(c, c->st);
  std::vector<int64_t> counts(P, 0);
  const int64_t bytes = c->pk * (int64_t)sizeof(float2);
  if (c->agv(c->cu, mine.data(), bytes, nullptr, counts.data()) != 0 ||
      c->agv(c->cu, mine.data(), bytes, all.data(), counts.data()) != 0)
    throw Fail{ACCORD_E_COMM, "allgatherv failed"};
  CK(cudaMemcpyAsync(c->col_sd, all.data(), c->p * sizeof(float2), cudaMemcpyHostToDevice,
                     c->st));
  csync(c, c->st);
}

// Largest eigenvalue of the symmetric tridiagonal matrix (alpha, beta) by
// bisection on Sturm counts.
double tridiag_lmax(const std::vector<double>& a, const std::vector<double>& b, int m) {
  double lo = 1e300, hi = -1e300;
  for (int i = 0; i < m; ++i) {   // Gershgorin interval
    const double r = (i > 0 ? std::fabs(b[i - 1]) : 0.0) + (i + 1 < m ? std::fabs(b[i]) : 0.0);
    lo = std::min(lo, a[i] - r);
    hi = std::max(hi, a[i] + r);
  }
  auto below = [&](double x) {   // number of eigenvalues < x
    int cnt = 0;
    double d = 1.0;
    for (int i = 0; i < m; ++i) {
      d = a[i] - x - (i > 0 ? b[i - 1] * b[i - 1] / d : 0.0);
      if (d == 0.0) d = -1e-300;
      if (d < 0) ++cnt;
    }
    return cnt;
  };
  for (int it = 0; it < 200 && hi - lo > 1e-15 * std::max(std::fabs(hi), 1e-300); ++it) {
    const double mid = 0.5 * (lo + hi);
    if (below(mid) >= m) hi = mid; else lo = mid;
  }
  return hi;
}

// Top eigenvalue of G = X X^T / n (n x n; the same nonzero spectrum as S) by
// Lanczos with full reorthogonalisation, the operator applied on the device
// (two passes over this rank's X^T, summed over ranks when X is sharded).
double lanczos_lmax(accord_ctx* c, int64_t pv) {
  const int64_t N = c->ldk;
  const int mmax = (int)std::min<int64_t>(200, c->n);
  const int64_t nsplit = std::min<int64_t>(256, std::max<int64_t>(1, pv / 256));
  double* u = c->dalloc<double>(N);
  double* w = c->dalloc<double>(N);
  double* t = c->dalloc<double>(std::max<int64_t>(pv, 1));
  double* part = c->dalloc<double>(nsplit * N);
  std::vector<double> Q((size_t)(mmax + 1) * N, 0.0), a(mmax), b(mmax), wv(N);
  // start vector: seeded pseudo-random (splitmix64), not the constant vector,
  // which X X^T / n maps to 0 when the columns of X are centered exactly
  {
    double nrm = 0.0;
    uint64_t z = 0x9E3779B97F4A7C15ull;
    for (int64_t i = 0; i < c->n; ++i) {
      z += 0x9E3779B97F4A7C15ull;
      uint64_t x = z;
      x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
      x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
      x ^= x >> 31;
      Q[i] = (double)(x >> 11) * 0x1.0p-53 * 2.0 - 1.0;
      nrm += Q[i] * Q[i];
    }
    nrm = std::sqrt(nrm);
    for (int64_t i = 0; i < c->n; ++i) Q[i] /= nrm;
  }
  double theta = 0.0, prev = -1.0;
  for (int j = 0; j < mmax; ++j) {
    CK(cudaMemcpyAsync(u, &Q[(size_t)j * N], N * 8, cudaMemcpyHostToDevice, c->st));
    c->launches += launch_gram_apply(c->dtype, c->Xt, pv, c->n, N, u, t, part, nsplit, w, c->st);
    if (c->sharded) dev_allreduce(c, w, (int)N);
    CK(cudaMemcpyAsync(wv.data(), w, N * 8, cudaMemcpyDeviceToHost, c->st));
    csync(c, c->st);
    const double* q = &Q[(size_t)j * N];
    double al = 0.0;
    for (int64_t i = 0; i < N; ++i) al += wv[i] * q[i];
    a[j] = al;
    for (int pass = 0; pass < 2; ++pass)   // full reorthogonalisation (twice is enough)
      for (int k = 0; k <= j; ++k) {
        const double* qk = &Q[(size_t)k * N];
        double h = 0.0;
        for (int64_t i = 0; i < N; ++i) h += wv[i] * qk[i];
        for (int64_t i = 0; i < N; ++i) wv[i] -= h * qk[i];
      }
    double bt = 0.0;
    for (int64_t i = 0; i < N; ++i) bt += wv[i] * wv[i];
    bt = std::sqrt(bt);
    b[j] = bt;
    theta = tridiag_lmax(a, b, j + 1);
    c->lanczos_steps = j + 1;
    if (j >= 8 && std::fabs(theta - prev) <= 1e-12 * std::fabs(theta)) break;
    prev = theta;
    if (!(bt > 1e-13 * std::max(std::fabs(theta), 1e-300))) break;   // invariant subspace
    double* qn = &Q[(size_t)(j + 1) * N];
    for (int64_t i = 0; i < N; ++i) qn[i] = wv[i] / bt;
  }
  c->dfree(u, N * 8);
  c->dfree(w, N * 8);
  c->dfree(t, std::max<int64_t>(pv, 1) * 8);
  c->dfree(part, nsplit * N * 8);
  return theta;
}

void create_impl(accord_ctx* c, const accord_init_params* prm) {
  validate(prm);
  // ACCORD_TRACE=1: host wall time of the create phases (stderr)
  const bool ctrace = std::getenv("ACCORD_TRACE") && std::getenv("ACCORD_TRACE")[0] == '1';
  auto tprev = std::chrono::steady_clock::now();
  auto phase = [&](const char* name) {
    if (!ctrace) return;
    cudaStreamSynchronize((cudaStream_t)prm->stream);
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[accord create] %s %.1f ms\n", name,
                 std::chrono::duration<double, std::milli>(t - tprev).count());
    tprev = t;
  };
  if (prm->workspace) {
    if (prm->workspace_bytes == 0) throw Fail{ACCORD_E_INVALID, "workspace_bytes is 0"};
    c->arena.init(prm->workspace, prm->workspace_bytes);
  }
  if (prm->device >= 0) CK(cudaSetDevice(prm->device));
  CK(cudaGetDevice(&c->device));
  CK(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, c->device));
  CK(cudaDeviceGetAttribute(&c->cc_major, cudaDevAttrComputeCapabilityMajor, c->device));
  CK(cudaDeviceGetAttribute(&c->cc_minor, cudaDevAttrComputeCapabilityMinor, c->device));
  c->st = (cudaStream_t)prm->stream;
  c->n = prm->n;
  c->p = prm->p;
  c->r0 = prm->row_begin;
  c->r1 = prm->row_end;
  c->pk = c->r1 - c->r0;
  c->ldk = round_up(c->n, kKPad);
  c->p_pad = round_up(c->p, kRowPad);
  c->pk_pad = round_up(c->pk, kRowPad);
  c->dtype = prm->dtype;
  c->tsz = c->dtype == ACCORD_F64 ? 8 : 4;
  c->lam = prm->lambda;
  c->tau0 = prm->tau0;
  c->beta = prm->beta;
  c->rank = prm->rank;
  c->world = prm->world;
  // world = 1 with NCCL keeps a 1-rank communicator (the collectives then run
  // for real: the single-GPU tests exercise the NCCL code path)
  c->comm = (prm->world > 1 || prm->comm == ACCORD_COMM_NCCL) ? prm->comm : ACCORD_COMM_NONE;
  c->ar = prm->allreduce;
  c->agv = prm->allgatherv;
  c->cu = prm->comm_user;
  const bool tc_ok = tc_supported(c->cc_major, c->cc_minor);
  // F32 on sm_100: the certified bf16 filter for any n (the refine streams
  // X^T rows in 4 KB chunks; the filter bound's gamma grows with n)
  c->gemm = resolve_gemm(prm, tc_ok, &c->i8);
  if (c->gemm == ACCORD_GEMM_I8_FILTER) {   // the filter pipeline with int8 operands
    c->gemm = ACCORD_GEMM_BF16_FILTER;
    c->i8_force = c->i8_on = true;
  }
  if (const char* e = std::getenv("ACCORD_I8_AT")) c->i8_at = std::atof(e);     // tuning
  if (const char* e = std::getenv("ACCORD_I8_OFF")) c->i8_off = std::atof(e);
  if (const char* e = std::getenv("ACCORD_I8_EXCESS")) c->i8_excess = std::atof(e);
  if (const char* e = std::getenv("ACCORD_I8_NNZ")) c->i8_nnz = std::atof(e);
  if (const char* e = std::getenv("ACCORD_I8_CCAP")) c->i8_ccap = std::atof(e);
  const bool tc = c->gemm == ACCORD_GEMM_BF16X3 || c->gemm == ACCORD_GEMM_BF16_FILTER;
  if (tc && !tc_ok) throw Fail{ACCORD_E_UNSUPPORTED, "tcgen05 GEMM needs an sm_100 device"};
  if (tc && prm->x_sharded && prm->world > 1 && prm->row_begin % kRowPad != 0)
    throw Fail{ACCORD_E_INVALID,
               "x_sharded with a tensor-core GEMM: row_begin must be a multiple of 256"};

  for (auto& e : c->ev) CK(cudaEventCreate(&e));
  {
    const char* t = std::getenv("ACCORD_TRACE");
    c->trace = t && t[0] == '1';
  }
  CK(cudaMallocHost(&c->h_red, 16 * sizeof(double)));
  CK(cudaMallocHost(&c->h_seg, 2 * sizeof(unsigned long long)));

  if (c->comm == ACCORD_COMM_NCCL) {
    NcclApi* api = nccl_api();
    if (!api) throw Fail{ACCORD_E_NCCL, "libnccl.so.2 could not be loaded"};
    ncclUniqueId id;
    std::memcpy(&id, prm->nccl_id, sizeof(id));
    NK(api->CommInitRank(&c->nccl, c->world, id, c->rank));
  }
  c->red_d = c->dalloc<double>(16);

  // ---- X sharded by variables (NEXT(3)): every rank's slab boundaries ----
  c->sharded = prm->x_sharded && c->world > 1;
  if (c->sharded) {
    const int P = c->world;
    std::vector<double> mine(2 * P, 0.0), tot(2 * P, 0.0);
    mine[2 * c->rank] = (double)c->r0;
    mine[2 * c->rank + 1] = (double)c->r1;
    for (int q = 0; q < 2 * P; q += 8) {
      const int cnt = std::min(8, 2 * P - q);
      CK(cudaMemcpyAsync(c->red_d, mine.data() + q, cnt * 8, cudaMemcpyHostToDevice, c->st));
      allreduce(c, c->red_d, c->h_red, cnt);
      std::memcpy(tot.data() + q, c->h_red, cnt * 8);
    }
    c->vb.assign(P + 1, 0);
    for (int q = 0; q < P; ++q) {
      c->vb[q] = (int64_t)tot[2 * q];
      if (q > 0 && (int64_t)tot[2 * q] != (int64_t)tot[2 * q - 1])
        throw Fail{ACCORD_E_INVALID, "x_sharded: rank blocks must tile [0, p) in rank order"};
    }
    c->vb[P] = (int64_t)tot[2 * P - 1];
    if (c->vb[0] != 0 || c->vb[P] != c->p)
      throw Fail{ACCORD_E_INVALID, "x_sharded: rank blocks must tile [0, p) in rank order"};
    if (c->comm == ACCORD_COMM_NCCL) {
      NcclApi* api = nccl_api();
      if (!api->Send || !api->Recv || !api->CommSplit)
        throw Fail{ACCORD_E_NCCL, "NCCL without send/recv/split"};
      NK(api->CommSplit(c->nccl, 0, c->rank, &c->nccl_ring, nullptr));
      CK(cudaStreamCreateWithFlags(&c->cs, cudaStreamNonBlocking));
      for (int b = 0; b < 2; ++b) {
        CK(cudaEventCreateWithFlags(&c->ev_comp[b], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->ev_recv[b], cudaEventDisableTiming));
      }
    }
    c->sr = prm->sendrecv;
  }
  if (c->world > 1 && !c->sharded) {
    // every rank's row block (the owner of a mirrored entry of the symmetric
    // first GEMM); the cyclic tile schedule needs blocks on 256-row tiles
    const int P = c->world;
    std::vector<double> mine(2 * P, 0.0), tot(2 * P, 0.0);
    mine[2 * c->rank] = (double)c->r0;
    mine[2 * c->rank + 1] = (double)c->r1;
    for (int q = 0; q < 2 * P; q += 8) {
      const int cnt = std::min(8, 2 * P - q);
      CK(cudaMemcpyAsync(c->red_d, mine.data() + q, cnt * 8, cudaMemcpyHostToDevice, c->st));
      allreduce(c, c->red_d, c->h_red, cnt);
      std::memcpy(tot.data() + q, c->h_red, cnt * 8);
    }
    c->rb.assign(P + 1, 0);
    bool ok = P <= 64;
    for (int q = 0; q < P; ++q) {
      c->rb[q] = (int64_t)tot[2 * q];
      if (q > 0 && (int64_t)tot[2 * q] != (int64_t)tot[2 * q - 1]) ok = false;
      if (c->rb[q] % kRowPad != 0) ok = false;
    }
    c->rb[P] = (int64_t)tot[2 * P - 1];
    if (c->rb[0] != 0 || c->rb[P] != c->p) ok = false;
    c->sym2_ok = ok;
    if (ok) {
      c->rb_dev = c->dalloc<int64_t>(P + 1);
      CK(cudaMemcpyAsync(c->rb_dev, c->rb.data(), (P + 1) * 8, cudaMemcpyHostToDevice, c->st));
      c->mir_cnt = c->dalloc<unsigned long long>(1 + 2 * P);
    }
  }
  const int64_t pv = c->sharded ? c->pk : c->p;   // variables held in Xt
  c->xrows_pad = c->sharded ? c->pk_pad : c->p_pad;

  phase("init+comm");
  // ---- X -> Xt (variable-major, padded), finiteness check ----
  const size_t T = c->tsz;
  c->Xt = c->dalloc_bytes((size_t)c->xrows_pad * c->ldk * T);
  const int64_t rows_src = prm->layout == ACCORD_LAYOUT_SAMPLES_ROW_MAJOR ? c->n : pv;
  const int64_t cols_src = prm->layout == ACCORD_LAYOUT_SAMPLES_ROW_MAJOR ? pv : c->n;
  const int64_t ldx = prm->ldx ? prm->ldx : cols_src;
  const void* Xsrc = prm->X;
  void* staging = nullptr;
  phase("X^T alloc");
  if (!prm->x_on_device) {
    staging = c->dalloc_bytes((size_t)rows_src * cols_src * T);
    phase("staging alloc");
    if (ldx == cols_src)   // dense: one linear copy (a 2-D copy of 4 KB rows is ~8x slower)
      CK(cudaMemcpyAsync(staging, prm->X, (size_t)rows_src * cols_src * T,
                         cudaMemcpyHostToDevice, c->st));
    else
      CK(cudaMemcpy2DAsync(staging, cols_src * T, prm->X, ldx * T, cols_src * T, rows_src,
                           cudaMemcpyHostToDevice, c->st));
    Xsrc = staging;
    phase("H2D copy");
  }
  unsigned long long* badidx = c->dalloc<unsigned long long>(1);
  CK(cudaMemsetAsync(badidx, 0xff, 8, c->st));
  c->launches += launch_load_xt(c->dtype, Xsrc, prm->x_on_device ? ldx : cols_src, prm->layout,
                                c->n, pv, c->Xt, c->ldk, c->xrows_pad, badidx, c->st);
  unsigned long long hb = 0;
  CK(cudaMemcpyAsync(&hb, badidx, 8, cudaMemcpyDeviceToHost, c->st));
  csync(c, c->st);
  if (staging) c->dfree(staging, (size_t)rows_src * cols_src * T);
  if (hb != ~0ull) {
    char m[160];
    std::snprintf(m, sizeof m, "non-finite X at (row %lld, col %lld) of the given layout",
                  (long long)(hb / cols_src), (long long)(hb % cols_src));
    throw Fail{ACCORD_E_INVALID, m};
  }

  phase("X^T (alloc, copy, transpose, check)");
  // ---- L ----
  if (prm->inv_L > 0) {
    c->inv_L = prm->inv_L;
    c->L = 1.0 / prm->inv_L;
  } else {
    // L = sigma_max(S) by Lanczos on the samples' Gram operator
    // (SPEC.md:85 suggests power iteration; the top eigenvalues of the
    // block-diagonal configs are clustered, so power iteration needs ~600
    // passes over X at c5, Lanczos ~50), then a safety inflation: a Ritz value
    // approaches L from below, and overestimating L is safe.
    c->L = lanczos_lmax(c, pv) * (1.0 + 2e-3);
    // L = 0 only for X = 0 (S = 0); any other non-positive or non-finite
    // estimate would silently disable the tau <= 1/L floor of Alg. 1
    if (!(c->L > 0) || !std::isfinite(c->L))
      throw Fail{ACCORD_E_NUMERIC, "sigma_max(S) estimate is not positive (X = 0?); pass inv_L"};
    c->inv_L = 1.0 / c->L;
  }

  if (ctrace) std::fprintf(stderr, "[accord create] Lanczos steps %d\n", c->lanczos_steps);
  phase("L (Lanczos)");
  // ---- operands ----
  const bool x3 = c->gemm == ACCORD_GEMM_BF16X3, filt = c->gemm == ACCORD_GEMM_BF16_FILTER;
  for (int b = 0; b < 2; ++b) {
    c->Y[b] = c->dalloc_bytes((size_t)c->pk_pad * c->ldk * T);
    CK(cudaMemsetAsync(c->Y[b], 0, (size_t)c->pk_pad * c->ldk * T, c->st));
  }
  if (tc) {
    c->Xhi = c->dalloc<__nv_bfloat16>((size_t)c->xrows_pad * c->ldk);
    if (x3) c->Xlo = c->dalloc<__nv_bfloat16>((size_t)c->xrows_pad * c->ldk);
    c->launches += launch_split_bf16((const float*)c->Xt, c->xrows_pad * c->ldk, c->Xhi, c->Xlo,
                                     c->st);
    for (int b = 0; b < 2; ++b) {
      c->Yhi[b] = c->dalloc<__nv_bfloat16>((size_t)c->pk_pad * c->ldk);
      CK(cudaMemsetAsync(c->Yhi[b], 0, (size_t)c->pk_pad * c->ldk * 2, c->st));
      if (x3) {
        c->Ylo[b] = c->dalloc<__nv_bfloat16>((size_t)c->pk_pad * c->ldk);
        CK(cudaMemsetAsync(c->Ylo[b], 0, (size_t)c->pk_pad * c->ldk * 2, c->st));
      }
      c->row_A[b] = c->dalloc<float>(c->pk);
      c->row_B[b] = c->dalloc<float>(c->pk);
    }
    if (filt) {
      // per-column constants of the filter bound for all p columns (the
      // sharded mode computes its slab's and gathers the rest)
      c->col_sd = c->dalloc<float2>(c->p);
      const int64_t off = c->sharded ? c->r0 : 0;
      c->launches += launch_col_norms(pv, c->ldk, (const float*)c->Xt, c->col_sd + off, c->st);
      if (c->i8) {
        // int8 X^T (block scale per 256 variables, variables permuted so that
        // a block holds nearly equal max |x|: quant_i8.cu) and the bound's
        // column constants of that quantisation
        c->xperm = c->dalloc<int32_t>(c->p_pad);
        {
          float* mx = c->dalloc<float>(c->p);
          c->launches += launch_row_absmax(c->p, c->n, c->ldk, (const float*)c->Xt, mx, c->st);
          std::vector<float> hm(c->p);
          CK(cudaMemcpyAsync(hm.data(), mx, c->p * 4, cudaMemcpyDeviceToHost, c->st));
          csync(c, c->st);
          c->dfree(mx, c->p * 4);
          const std::vector<int32_t> perm = scale_permutation(hm, c->p_pad);
          CK(cudaMemcpyAsync(c->xperm, perm.data(), c->p_pad * 4, cudaMemcpyHostToDevice, c->st));
          csync(c, c->st);   // perm is a local vector
        }
        c->col_sd_q = c->dalloc<float2>(c->p);
        c->blk_q = c->dalloc<float2>(c->p_pad / kRowPad);
        CK(cudaMemsetAsync(c->blk_q, 0, (c->p_pad / kRowPad) * sizeof(float2), c->st));
        c->Xq = c->dalloc<int8_t>((size_t)c->xrows_pad * c->ldk);
        CK(cudaMemsetAsync(c->Xq, 0, (size_t)c->xrows_pad * c->ldk, c->st));
        c->xq_scale = c->dalloc<float>(c->p_pad / kRowPad);
        c->launches += launch_quant_x_i8(pv, c->n, c->ldk, (const float*)c->Xt, c->xperm, c->Xq,
                                         c->xq_scale, c->col_sd_q, c->st);
        for (int b = 0; b < 2; ++b) {
          c->Yq[b] = c->dalloc<int8_t>((size_t)c->pk_pad * c->ldk);
          CK(cudaMemsetAsync(c->Yq[b], 0, (size_t)c->pk_pad * c->ldk, c->st));
          c->yq_s[b] = c->dalloc<float>(c->pk);
          c->yq_A[b] = c->dalloc<float>(c->pk);
          c->yq_B[b] = c->dalloc<float>(c->pk);
        }
      }
      if (c->sharded) gather_col_sd(c);
    }
    std::string e;
    float2* bsd = c->dalloc<float2>(c->p_pad / kRowPad);
    CK(cudaMemsetAsync(bsd, 0, (c->p_pad / kRowPad) * sizeof(float2), c->st));
    c->plan = tc_plan_create(c->Yhi[0], x3 ? c->Ylo[0] : c->Yhi[0], c->Yhi[1],
                             x3 ? c->Ylo[1] : c->Yhi[1], c->pk_pad, c->Xhi,
                             x3 ? c->Xlo : c->Xhi, c->xrows_pad, c->p_pad, c->n, c->ldk, bsd, &e);
    if (!c->plan) throw Fail{ACCORD_E_CUDA, "tensor map: " + e};
    if (c->i8 && !tc_plan_set_i8(c->plan, c->Yq[0], c->Yq[1], c->Xq, c->xrows_pad, c->blk_q, &e))
      throw Fail{ACCORD_E_CUDA, "tensor map (int8): " + e};
    if (filt) c->launches += tc_plan_set_col_norms(c->plan, c->col_sd, c->p, c->st);
    if (c->i8)
      c->launches += tc_plan_set_col_norms(c->plan, c->col_sd_q, c->p, c->st, true, c->xperm);
  }

  phase("operands (Y, bf16 copies, column norms, tensor maps)");
  // ---- ring buffers of the sharded mode ----
  if (c->sharded) {
    for (int q = 0; q < c->world; ++q)
      c->rrows_pad = std::max(c->rrows_pad, round_up(slab_rows(c, q), kRowPad));
    const size_t rb = (size_t)c->rrows_pad * c->ldk;
    for (int b = 0; b < 2; ++b) {
      c->rbuf[b] = c->dalloc_bytes(rb * T);
      CK(cudaMemsetAsync(c->rbuf[b], 0, rb * T, c->st));
      if (tc) {
        c->rhi[b] = c->dalloc<__nv_bfloat16>(rb);
        CK(cudaMemsetAsync(c->rhi[b], 0, rb * 2, c->st));
        if (x3) {
          c->rlo[b] = c->dalloc<__nv_bfloat16>(rb);
          CK(cudaMemsetAsync(c->rlo[b], 0, rb * 2, c->st));
        }
        std::string e;
        if (!tc_plan_set_b(c->plan, 1 + b, c->rhi[b], x3 ? c->rlo[b] : c->rhi[b], c->rrows_pad, &e))
          throw Fail{ACCORD_E_CUDA, "tensor map: " + e};
      }
    }
    c->yacc = c->dalloc<double>((size_t)c->pk_pad * c->ldk);
    c->dacc = c->dalloc<double>((size_t)c->pk_pad * c->ldk);
    if (c->comm == ACCORD_COMM_HOST) {
      CK(cudaMallocHost(&c->h_send, rb * T));
      CK(cudaMallocHost(&c->h_recv, rb * T));
    }
  }

  // ---- per-row and entry-indexed state ----
  c->om_ptr = c->dalloc<int64_t>(c->pk + 1);
  c->c_ptr = c->dalloc<int64_t>(c->pk + 1);
  c->c_ptr2 = c->dalloc<int64_t>(c->pk + 1);
  c->row_cnt = c->dalloc<int32_t>(c->pk);
  c->rcur = c->dalloc<int32_t>(c->pk);
  c->long_rows = c->dalloc<int32_t>(c->pk + 1);
  c->chunk_next = c->dalloc<unsigned int>(1);
  c->gemm_warps = c->plan ? 4 * tc_grid_size(c->plan, c->sm_count) : 0;
  c->row_D2 = c->dalloc<double>(c->pk);
  c->row_Y2 = c->dalloc<double>(c->pk);
  c->row_dd = c->dalloc<double>(c->pk);
  c->row_l1 = c->dalloc<double>(c->pk);
  c->row_logd = c->dalloc<double>(c->pk);
  c->row_nnz = c->dalloc<int32_t>(c->pk);
  c->row_dd2 = c->dalloc<double>(c->pk);
  c->row_l1_2 = c->dalloc<double>(c->pk);
  c->row_logd2 = c->dalloc<double>(c->pk);
  c->row_D2b = c->dalloc<double>(c->pk);
  c->diag_xx = c->dalloc<double>(c->pk);   // line search from Omega = I
  c->diag_xz = c->dalloc<double>(c->pk);
  c->diag_zz = c->dalloc<double>(c->pk);
  c->diag_a = c->dalloc<double>(c->pk);
  c->row_nnz2 = c->dalloc<int32_t>(c->pk);
  {
    const char* e = std::getenv("ACCORD_LS_PAIRS");   // A-B switch
    c->pair_ls = !(e && e[0] == '0');
    const char* r = std::getenv("ACCORD_REFINE");     // A-B: ff = float-float refine
    c->refine_ff = (r && r[0] == 'f' && r[1] == 'f') ? 1 : 0;
    if (const char* x = std::getenv("ACCORD_XDROP")) c->x_drop_target = std::clamp(std::atoi(x), 0, 4);
    if (const char* x = std::getenv("ACCORD_YDROP")) c->y_drop_target = std::clamp(std::atoi(x), 0, 4);
    if (const char* x = std::getenv("ACCORD_XDROP_AT")) c->x_drop_at = std::atof(x);
  }
  c->bad_diag = c->dalloc<int32_t>(1);
  c->scan_tmp_sz = scan_tmp_bytes(c->pk + 1);
  c->scan_tmp = c->dalloc_bytes(c->scan_tmp_sz);
  // TMA-staged SpMM for large row blocks; below ~6.5e4 rows the persistent
  // producer/consumer pipeline has too few items per block to hide its
  // per-item latency and the block-per-row kernel is faster (config 3:
  // 0.8 vs 0.4 ms per trial; config 4: 1.8 vs 3.4 ms)
  // ... and only when every consumer warp is full (ldk a multiple of 256): with
  // lanes past the row end the row finalize diverges, and at config 6 (n = 365,
  // one candidate per row) the block-per-row kernel is twice as fast (0.58 vs
  // 1.15 ms per step, profiles/r02c/c6ab)
  c->tma_spmm = !c->sharded && spmm_tma_supported(c->dtype, c->ldk) && c->pk >= 65536 &&
                c->ldk % 256 == 0 &&
                std::getenv("ACCORD_SPMM_PLAIN") == nullptr;   // env: A-B diagnostic
  if (std::getenv("ACCORD_SPMM_TMA"))   // env: force (tests of the TMA path at small sizes)
    c->tma_spmm = !c->sharded && spmm_tma_supported(c->dtype, c->ldk);
  if (c->world > 1 && !c->sharded && spmm_tma_supported(c->dtype, c->ldk)) {
    // the paired line-search pass exists for the TMA SpMM only, and every
    // rank must run the same passes (each ends in an allreduce of 8 or 16
    // sums): one SpMM kind for all ranks, TMA if any rank's block is large
    const double flag = c->tma_spmm ? 1.0 : 0.0;
    CK(cudaMemcpyAsync(c->red_d + 8, &flag, 8, cudaMemcpyHostToDevice, c->st));
    c->tma_spmm = allreduce_max(c, c->red_d + 8) > 0.5;
  }
  c->itm_n = c->dalloc<int32_t>(c->pk);
  c->itm_s = c->dalloc<int32_t>(c->pk);
  c->itm_ptr = c->dalloc<int64_t>(c->pk + 1);
  c->slot_ptr = c->dalloc<int64_t>(c->pk + 1);
  c->row_done = c->dalloc<int32_t>(c->pk);
  CK(cudaMemsetAsync(c->row_done, 0, c->pk * 4, c->st));
  int64_t cap = prm->cand_capacity;
  if (cap <= 0) {
    // The first iteration (G = S) has the most candidates (config 5: ~365 per
    // row); size for it so that it is not recomputed (~52 B per entry across
    // pool, C, keys and Omega arrays): within 40% of the free device memory,
    // or exactly the default the workspace query assumed.
    cap = default_capacity(c->pk, c->p);
    if (!c->arena.base) {
      size_t fr = 0, tot = 0;
      cudaMemGetInfo(&fr, &tot);
      const int64_t mem_cap = (int64_t)(0.4 * (double)fr / 52.0);
      cap = std::max<int64_t>(std::min(cap, mem_cap),
                              std::min<int64_t>(c->pk * c->p, c->pk * 16));
    }
  }
  cap = std::max<int64_t>(cap, c->pk);
  phase("per-row state");
  grow(c, std::min<int64_t>(cap, (int64_t)UINT32_MAX), 0);
  phase("candidate pool");

  // ---- Omega^{(0)} = I, Y^{(0)} = rows of X^T, f^{(0)} ----
  c->launches += launch_identity(c->dtype, c->pk, c->r0, c->om_ptr, c->om_col, c->om_val, c->st);
  recompute_y(c);
  c->omega_identity = true;
  refresh_objective(c);
  phase("Omega = I, Y, f");
}

template <typename F>
accord_status guard(accord_ctx* c, F&& fn) {
  try {
    fn();
    return ACCORD_OK;
  } catch (const Fail& f) {
    if (c) c->err = f.msg;
    return f.s;
  } catch (const std::bad_alloc&) {
    if (c) c->err = "host allocation failed";
    return ACCORD_E_NOMEM;
  } catch (...) {
    if (c) c->err = "unknown internal error";
    return ACCORD_E_CUDA;
  }
}

void TR(accord_ctx* c, const char* name) {
  if (!c->trace) return;
  if (c->tr_marks.size() >= c->tr_pool.size()) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    c->tr_pool.push_back(e);
  }
  cudaEvent_t e = c->tr_pool[c->tr_marks.size()];
  CK(cudaEventRecord(e, c->st));
  c->tr_marks.emplace_back(name, e);
}

void TR_flush(accord_ctx* c) {
  if (!c->trace || c->tr_marks.empty()) return;
  CK(cudaEventSynchronize(c->tr_marks.back().second));
  std::fprintf(stderr, "[accord trace] it=%lld maxrow=%.0f ncand=%.0f nnz=%lld i8=%d",
               (long long)c->iters, c->h_red[7], c->h_red[6], (long long)c->nnz_global,
               c->i8_last ? 1 : 0);
  for (size_t i = 1; i < c->tr_marks.size(); ++i) {
    float ms = 0;
    cudaEventElapsedTime(&ms, c->tr_marks[i - 1].second, c->tr_marks[i].second);
    std::fprintf(stderr, " %s=%.3f", c->tr_marks[i].first, ms);
  }
  std::fprintf(stderr, "\n");
  c->tr_marks.clear();
}

float ev_ms(accord_ctx* c, int a, int b) {
  float ms = 0;
  cudaEventElapsedTime(&ms, c->ev[a], c->ev[b]);
  return ms;
}

double lam_eff(const accord_ctx* c) { return c->refit ? c->phi * c->lam : c->lam; }

// ---- symmetric first GEMM across ranks: the mirrored entries' exchange ----
void grow_mirror(accord_ctx* c, int64_t need) {
  const int64_t cap = need + need / 4 + (1 << 20);
  c->dfree(c->mir_row, c->mir_cap * 4);
  c->dfree(c->mir_col, c->mir_cap * 4);
  c->dfree(c->mir_send, c->mir_cap * 8);
  c->mir_row = c->dalloc<int32_t>(cap);
  c->mir_col = c->dalloc<int32_t>(cap);
  c->mir_send = c->dalloc<int32_t>(2 * cap);
  c->mir_cap = cap;
}

// Send every mirrored entry (global row k, column i) to the rank owning row
// k and receive this rank's into mir_recv (mir_recv_n entries). Collective.
void mirror_exchange(accord_ctx* c, int64_t n_out) {
  const int P = c->world;
  cudaStream_t S = c->st;
  unsigned long long* dcnt = c->mir_cnt + 1;
  unsigned long long* dcur = c->mir_cnt + 1 + P;
  CK(cudaMemsetAsync(dcnt, 0, P * 8, S));
  c->launches += launch_mirror_count(n_out, c->mir_row, c->rb_dev, P, dcnt, S);
  std::vector<unsigned long long> cnt(P), off(P, 0);
  CK(cudaMemcpyAsync(cnt.data(), dcnt, P * 8, cudaMemcpyDeviceToHost, S));
  csync(c, S);
  for (int q = 1; q < P; ++q) off[q] = off[q - 1] + cnt[q - 1];
  CK(cudaMemcpyAsync(dcur, off.data(), P * 8, cudaMemcpyHostToDevice, S));
  c->launches += launch_mirror_scatter(n_out, c->mir_row, c->mir_col, c->rb_dev, P, dcur,
                                       c->mir_send, S);
  // counts[src][dst] on every rank
  std::vector<double> m(P * P, 0.0);
  for (int q = 0; q < P; ++q) m[c->rank * P + q] = (double)cnt[q];
  for (int q = 0; q < P * P; q += 16) {
    const int k = std::min(16, P * P - q);
    CK(cudaMemcpyAsync(c->red_d, m.data() + q, k * 8, cudaMemcpyHostToDevice, S));
    allreduce(c, c->red_d, c->h_red, k);
    std::memcpy(m.data() + q, c->h_red, k * 8);
  }
  std::vector<int64_t> rc(P), roff(P, 0);
  int64_t R = 0;
  for (int q = 0; q < P; ++q) {
    rc[q] = (int64_t)m[q * P + c->rank];
    roff[q] = R;
    R += rc[q];
  }
  if (R > c->mir_recv_cap) {
    c->dfree(c->mir_recv, c->mir_recv_cap * 8);
    c->mir_recv_cap = R + R / 4 + 1024;
    c->mir_recv = c->dalloc<int32_t>(2 * c->mir_recv_cap);
  }
  c->mir_recv_n = R;
  for (int q = 0; q < P; ++q) c->mirrored_sent += (int64_t)cnt[q];
  if (c->comm == ACCORD_COMM_NCCL) {
    NcclApi* api = nccl_api();
    if (!api->Send || !api->Recv) throw Fail{ACCORD_E_NCCL, "NCCL without send/recv"};
    NK(api->GroupStart());
    for (int q = 0; q < P; ++q) {
      if (q == c->rank) continue;
      if (cnt[q])
        NK(api->Send(c->mir_send + 2 * off[q], cnt[q] * 8, ncclChar, q, c->nccl, S));
      if (rc[q])
        NK(api->Recv(c->mir_recv + 2 * roff[q], (size_t)rc[q] * 8, ncclChar, q, c->nccl, S));
    }
    NK(api->GroupEnd());
    csync(c, S);
    return;
  }
  // host transport (tests): every rank gathers [counts | pairs] of all ranks
  if (!c->agv) throw Fail{ACCORD_E_INVALID, "multi-rank host comm needs allgatherv"};
  std::vector<char> mineb(P * 8 + n_out * 8);
  for (int q = 0; q < P; ++q) {
    const int64_t v = (int64_t)cnt[q];
    std::memcpy(mineb.data() + q * 8, &v, 8);
  }
  if (n_out)
    CK(cudaMemcpyAsync(mineb.data() + P * 8, c->mir_send, n_out * 8, cudaMemcpyDeviceToHost, S));
  csync(c, S);
  std::vector<int64_t> counts(P, 0);
  if (c->agv(c->cu, mineb.data(), (int64_t)mineb.size(), nullptr, counts.data()) != 0)
    throw Fail{ACCORD_E_COMM, "allgatherv (sizes) failed"};
  int64_t all = 0;
  for (auto x : counts) all += x;
  std::vector<char> buf(all);
  if (c->agv(c->cu, mineb.data(), (int64_t)mineb.size(), buf.data(), counts.data()) != 0)
    throw Fail{ACCORD_E_COMM, "allgatherv failed"};
  std::vector<int32_t> recv(2 * std::max<int64_t>(R, 1));
  const char* rd = buf.data();
  for (int q = 0; q < P; ++q) {
    std::vector<int64_t> cq(P);
    std::memcpy(cq.data(), rd, P * 8);
    int64_t o = 0;
    for (int d = 0; d < c->rank; ++d) o += cq[d];
    if (q != c->rank && cq[c->rank])
      std::memcpy(recv.data() + 2 * roff[q], rd + P * 8 + o * 8, cq[c->rank] * 8);
    rd += counts[q];
  }
  if (R) CK(cudaMemcpyAsync(c->mir_recv, recv.data(), R * 8, cudaMemcpyHostToDevice, S));
  csync(c, S);
}

// Mark `count` entries written from chunk `used` on as pool chunks [used,
// used + needc) (fill counts and the chunk counter the finalize reads).
void pool_claim(accord_ctx* c, int64_t used, int64_t needc, int64_t count) {
  cudaStream_t S = c->st;
  if (needc > 0) {
    std::vector<unsigned long long> fill(needc, (unsigned long long)c->chunk);
    fill.back() = (unsigned long long)(count - (needc - 1) * c->chunk);
    CK(cudaMemcpyAsync(c->chunk_fill + used, fill.data(), needc * 8, cudaMemcpyHostToDevice, S));
    const unsigned int nx = (unsigned int)(used + needc);
    CK(cudaMemcpyAsync(c->chunk_next, &nx, 4, cudaMemcpyHostToDevice, S));
    csync(c, S);   // the host vectors go out of scope
  }
  c->h_seg[1] = used + needc;
}

// Append the received mirrored entries to the pool as chunks [used, used+needc).
void mirror_append(accord_ctx* c, int64_t used, int64_t needc) {
  c->launches += launch_mirror_append(c->mir_recv_n, c->mir_recv, c->r0, c->pool_row,
                                      c->pool_col, used * c->chunk, c->row_cnt, c->st);
  pool_claim(c, used, needc, c->mir_recv_n);
}

// Operands of a gradient pass other than the current iterate's (lambda_max:
// A = the rank's rows of X^T, i.e. Omega = I, with an empty support).
struct GradOverride {
  int ybuf;                 // plan A map
  const float *row_A, *row_B;
  const float* row_scale;   // I8_FILTER: per-row scale of the A operand
  OmegaView om;
  double lam_cand;
  unsigned int* max_out;    // != NULL: max-reduce pass only (no candidates)
  bool sym;
};

// Candidate set C with exact gradient values G on it and the current omega:
// either the GEMM + fused epilogue + finalize (+ refine) of a plain iteration,
// or, for the bias-correction refit (Eq. 3.8), the fixed support S_hat with G
// from the SDDMM (entries off S_hat carry an infinite penalty and stay 0).
void build_candidates(accord_ctx* c, accord_iter_stats& st, const GradOverride* ov = nullptr) {
  cudaStream_t S = c->st;
  if (c->refit && !ov) {
    CK(cudaEventRecord(c->ev[1], S));
    CK(cudaEventRecord(c->ev[2], S));
    CK(cudaMemcpyAsync(c->c_ptr, c->refit_ptr, (c->pk + 1) * 8, cudaMemcpyDeviceToDevice, S));
    c->items_of = nullptr;
    c->c_sym = false;
    CK(cudaMemcpyAsync(c->c_col, c->refit_col, c->refit_nnz * 4, cudaMemcpyDeviceToDevice, S));
    c->launches += launch_lookup(c->dtype, c->pk, c->c_ptr, c->c_col, c->om_ptr, c->om_col,
                                 c->om_val, c->c_w, S);
    CK(cudaEventRecord(c->ev[3], S));
    refine_all(c);
    CK(cudaEventRecord(c->ev[4], S));
    TR(c, "refit_sddmm");
    CK(cudaEventSynchronize(c->ev[4]));
    st.ms_finalize = ev_ms(c, 2, 3);
    st.ms_refine = ev_ms(c, 3, 4);
    return;
  }
  // ---------------- a2 + a3: gradient GEMM with the fused epilogue --------
  // several ranks at Omega = I: the cyclic half of the symmetric GEMM, with
  // the mirrored entries of other ranks' rows exchanged after it
  // (not under the filter audit: another rank's mirrored accumulators would
  // be missing from this rank's dump)
  // int8 GEMM (I8_FILTER, or AUTO once |C| is small; an override pass --
  // lambda_max at Omega = I -- whenever int8 operands exist): the int8 copy of
  // the current Y and its bound constants (a read of Y per GEMM: ~1 ms at c5)
  const bool use_i8 = c->i8 && (ov ? true : c->i8_on);
  if (!use_i8 && !ov) ensure_yhi(c, c->cur);   // a bf16 GEMM after int8 ones
  const bool sym2 = !use_i8 && !ov && !c->audit_acc && c->sym2_ok && c->omega_identity &&
                    c->gemm == ACCORD_GEMM_BF16_FILTER && !std::getenv("ACCORD_GEMM_NOSYM");
  bool exchanged = false;
  if (sym2 && !c->mir_row) grow_mirror(c, std::max<int64_t>(c->pk * 64, 1 << 20));
  c->i8_last = use_i8;
  st.gemm_i8 = use_i8 ? 1 : 0;
  if (use_i8 && !ov)
    c->launches += launch_quant_y_i8(c->pk, c->n, c->ldk, (const float*)c->Y[c->cur],
                                     c->Yq[c->cur], c->yq_s[c->cur], c->yq_A[c->cur],
                                     c->yq_B[c->cur], S);
  for (;;) {
    CK(cudaMemsetAsync(c->row_cnt, 0, c->pk * 4, S));
    CK(cudaMemsetAsync(c->chunk_fill, 0, c->nchunks * 8, S));
    if (c->gemm_warps == 0) {   // SIMT: one chunk, handed out up front
      static const unsigned int one = 1;
      CK(cudaMemcpyAsync(c->chunk_next, &one, 4, cudaMemcpyHostToDevice, S));
    } else {
      CK(cudaMemsetAsync(c->chunk_next, 0, 4, S));
    }
    // supp Omega joins C in the finalize (filter path); none for an override
    // pass (lambda_max: empty support)
    const int64_t n_sup = (c->gemm == ACCORD_GEMM_BF16_FILTER && !ov) ? c->nnz_local : 0;
    EpiParams ep{};
    ep.pk = c->pk;
    ep.p = c->p;
    ep.r0 = c->r0;
    ep.col_base = 0;
    ep.col_end = c->p;
    ep.inv_n = 1.0 / (double)c->n;
    ep.lam_cand = c->dtype == ACCORD_F64 ? c->lam : c->lam * (1.0 - 4e-6);
    ep.row_A = c->row_A[c->cur];
    ep.row_B = c->row_B[c->cur];
    ep.col_sd = c->col_sd;
    // fp32-accumulation term of the filter bound: (n/16 + 17) * 2^-22 * sum|y^ x^|
    ep.gamma = (float)(((double)c->ldk / 16.0 + 17.0) * std::ldexp(1.0, -22));
    if (use_i8) {   // exact s32 accumulation: no accumulation term
      ep.gamma = 0.f;
      ep.row_A = c->yq_A[c->cur];
      ep.row_B = c->yq_B[c->cur];
      ep.row_scale = c->yq_s[c->cur];
    }
    if (use_i8) {
      ep.blk_scale = c->xq_scale;
      ep.col_perm = c->xperm;
    }
    ep.exact_cols = std::getenv("ACCORD_FILTER_EXACT") != nullptr;   // A-B diagnostic
    // Omega = I on one rank: G = S is symmetric, half the tiles (ACCORD_GEMM_NOSYM: off)
    // (not on the int8 operands: their columns are permuted variables)
    ep.sym = !use_i8 && c->omega_identity && c->gemm == ACCORD_GEMM_BF16_FILTER && c->world == 1 &&
             !c->sharded && c->r0 == 0 && c->pk == c->p && !std::getenv("ACCORD_GEMM_NOSYM");
    if (sym2) {
      ep.sym = 2;
      ep.mt0 = (int)(c->r0 / kRowPad);
      ep.nt = (int)(c->p_pad / kRowPad);
      ep.mir_row = c->mir_row;
      ep.mir_col = c->mir_col;
      ep.mir_cnt = c->mir_cnt;
      ep.mir_cap = c->mir_cap;
      CK(cudaMemsetAsync(c->mir_cnt, 0, 8, S));
    }
    ep.audit_acc = c->audit_acc;
    ep.audit_ld = c->audit_ld;
    OmegaView omv = omega_view(c);
    int ybuf = c->cur;
    if (ov) {
      ybuf = ov->ybuf;
      ep.row_A = ov->row_A;
      ep.row_B = ov->row_B;
      ep.row_scale = ov->row_scale;
      ep.lam_cand = ov->lam_cand;
      ep.max_out = ov->max_out;
      ep.sym = ov->sym;
      ep.audit_acc = nullptr;
      omv = ov->om;
    }
    c->c_sym = !ov && ep.sym == 1;
    CK(cudaEventRecord(c->ev[1], S));
    const bool tc = c->gemm == ACCORD_GEMM_BF16X3 || c->gemm == ACCORD_GEMM_BF16_FILTER;
    auto gemm = [&](const void* xt, int bsel, int64_t v0, int64_t v1) {
      ep.col_base = v0;
      ep.col_end = v1;
      if (tc) {
        const int l = launch_gemm_tc(c->plan, use_i8 ? (int)ACCORD_GEMM_I8_FILTER : c->gemm, ybuf,
                                     bsel, c->sm_count, ep, omv, pool_view(c), S);
        if (use_i8) c->gemm_launches_i8++;
        if (l < 0) throw Fail{ACCORD_E_CUDA, "tcgen05 GEMM launch failed"};
        c->launches += l;
      } else {
        c->launches += launch_gemm_simt(c->dtype, c->Y[c->cur], xt, c->ldk, c->ldk, ep, omv,
                                        pool_view(c), S);
      }
      c->gemm_launches++;
    };
    if (c->sharded)   // G_k[:, slab j] for every slab j, the pool filling across the ring
      ring_pass(c, tc, [&](const void* xt, int bsel, int64_t v0, int64_t v1, bool, bool) {
        gemm(xt, bsel, v0, v1);
      });
    else
      gemm(c->Xt, 0, 0, c->p);
    CK(cudaGetLastError());
    CK(cudaEventRecord(c->ev[2], S));
    TR(c, "gemm");
    unsigned long long h_mir = 0;
    {
      unsigned int used = 0;
      CK(cudaMemcpyAsync(&used, c->chunk_next, 4, cudaMemcpyDeviceToHost, S));
      CK(cudaMemcpyAsync(c->h_seg, c->chunk_fill, 8, cudaMemcpyDeviceToHost, S));
      if (sym2) CK(cudaMemcpyAsync(&h_mir, c->mir_cnt, 8, cudaMemcpyDeviceToHost, S));
      csync(c, S);
      c->h_seg[1] = used;
    }
    st.ms_gemm += ev_ms(c, 1, 2);
    if (ov && ov->max_out) return;   // max-reduce pass: no candidates
    // overflow: SIMT counts entries in chunk_fill[0]; tcgen05 counts chunks
    const int64_t need = c->gemm_warps == 0 ? (int64_t)c->h_seg[0]
                                            : (int64_t)c->h_seg[1] * c->chunk;
    const bool ovf = c->gemm_warps == 0 ? need > c->chunk : (int64_t)c->h_seg[1] > c->nchunks;
    bool ovf_any = ovf;
    if (c->sharded) {   // the ring is collective: redo it together if any rank overflowed
      c->h_red[0] = ovf ? 1.0 : 0.0;
      CK(cudaMemcpyAsync(c->red_d, c->h_red, 8, cudaMemcpyHostToDevice, S));
      allreduce(c, c->red_d, c->h_red, 1);
      ovf_any = c->h_red[0] > 0;
    }
    if (sym2 && (int64_t)h_mir > c->mir_cap) {   // mirror buffer overflow: grow, redo locally
      grow_mirror(c, (int64_t)h_mir);
      if (!ovf) continue;
    }
    if (!ovf_any) {
      // the mirrored positions received from other ranks (sym 2) join the pool
      if (sym2 && !exchanged) {   // collective, once (a local redo regenerates the same entries)
        mirror_exchange(c, (int64_t)h_mir);
        exchanged = true;
      }
      const int64_t used = (int64_t)c->h_seg[1];
      const int64_t need_m = sym2 ? (c->mir_recv_n + c->chunk - 1) / c->chunk : 0;
      if (used + need_m > c->nchunks) {
        const int64_t want = (used + need_m) * c->chunk;   // room for the received entries
        grow(c, want + want / 4 + (1 << 20), c->nnz_local);
        continue;
      }
      if (sym2) mirror_append(c, used, need_m);
      // supp Omega with its diagonal joins C in the finalize (the filter's
      // epilogue emits only its |acc| survivors): the key arrays must hold
      // both before the dedupe
      if (n_sup) c->launches += launch_support_count(c->pk, omv.ptr, c->row_cnt, S);
      c->launches += launch_scan_i32(c->row_cnt, c->c_ptr, c->pk, c->scan_tmp, c->scan_tmp_sz, S);
      // the pool's chunks bound the GEMM's entries: read the exact total
      // (one more host sync) only when that bound does not already fit
      if (n_sup && (int64_t)c->h_seg[1] * c->chunk + n_sup > c->cap) {
        int64_t tot = 0;
        CK(cudaMemcpyAsync(&tot, c->c_ptr + c->pk, 8, cudaMemcpyDeviceToHost, S));
        csync(c, S);
        if (tot > c->cap) {
          grow(c, tot + tot / 4 + (1 << 20), c->nnz_local);
          continue;
        }
      }
      break;
    }
    if (!ovf) continue;
    const int64_t want = need + need / 4 + (1 << 20);
    if (want >= (int64_t)UINT32_MAX)
      throw Fail{ACCORD_E_NOMEM, "candidate pool exceeds 2^32 entries"};
    grow(c, want, c->nnz_local);
  }
  // ---------------- a4: finalize C (row counts scanned into c_ptr above) ----
  TR(c, "host_gap+scan");
  CK(cudaMemsetAsync(c->rcur, 0, c->pk * 4, S));
  CK(cudaMemsetAsync(c->long_rows, 0, 4, S));
  TR(c, "memset");
  PoolView pv = pool_view(c);
  const bool filt = c->gemm == ACCORD_GEMM_BF16_FILTER;
  if (filt) {          // the epilogue emits positions only
    pv.g = nullptr;    // values come from the refine
    pv.w = nullptr;    // omega_ik from a lookup in Omega's sorted rows
  }
  c->launches += launch_finalize(c->dtype, c->pk, pv, c->c_ptr, c->rcur, c->keys,
                                 c->keys_tmp, c->c_col, c->c_g, c->c_w, c->long_rows, S,
                                 filt && !ov ? c->om_ptr : nullptr,
                                 filt && !ov ? c->om_col : nullptr);
  if (filt && !ov) {
    // the support entries the filter also emitted sit next to their twin after
    // the row sort: keep one of each (C's new row pointers in c_ptr2, swapped in)
    c->launches += launch_dedupe(c->pk, c->c_ptr, c->keys, c->row_cnt, c->c_ptr2, c->c_col,
                                 c->scan_tmp, c->scan_tmp_sz, S);
    std::swap(c->c_ptr, c->c_ptr2);
  }
  c->items_of = nullptr;   // C changed
  if (filt) {
    const ProxItems* pit = nullptr;
    ProxItems pitems{};
    if (!c->sharded) {   // work items of C (also used by the refine and the trials)
      build_items(c, c->c_ptr);
      pitems = ProxItems{c->itm_ptr, c->item_row, c->n_items, kItemEntries, nullptr, nullptr,
                         nullptr, nullptr};
      pit = &pitems;
    }
    if (!ov)
      c->launches += launch_lookup(c->dtype, c->pk, c->c_ptr, c->c_col, c->om_ptr, c->om_col,
                                   c->om_val, c->c_w, S, pit);
  }
  CK(cudaEventRecord(c->ev[3], S));
  TR(c, "finalize");
  if (c->gemm == ACCORD_GEMM_BF16_FILTER && !ov) {
    // exact values of the filtered candidates: G_ik = <Y_i, X_k> / n (f64 accumulation)
    refine_all(c);
  }
  CK(cudaEventRecord(c->ev[4], S));
  TR(c, "refine");
  CK(cudaEventSynchronize(c->ev[4]));
  st.ms_finalize = ev_ms(c, 2, 3);
  st.ms_refine = ev_ms(c, 3, 4);
}

// X^T_hi rounded to 7 - drop mantissa bits (filter path, X replicated): the
// bf16 copy, the per-column bound constants and the tile maxima are rebuilt
// from the f32 X^T, so the filter stays certified. The
// candidate set only grows (the bound widens), never loses an entry.
void set_x_width(accord_ctx* c, int drop) {
  c->launches += launch_split_bf16((const float*)c->Xt, c->xrows_pad * c->ldk, c->Xhi, nullptr,
                                   c->st, drop);
  c->launches += launch_col_norms(c->p, c->ldk, (const float*)c->Xt, c->col_sd, c->st, drop);
  c->launches += tc_plan_set_col_norms(c->plan, c->col_sd, c->p, c->st);
  c->x_drop = drop;
}

void step_one(accord_ctx* c, accord_iter_stats* s) {
  accord_iter_stats st{};
  cudaStream_t S = c->st;
  CK(cudaEventRecord(c->ev[0], S));
  TR(c, "start");
  build_candidates(c, st);
  const double lam = lam_eff(c);
  // ---------------- a5-a7: line search ----------------
  const int nb = c->cur ^ 1;
  double tau = c->tau0;
  double r[8];
  // From Omega = I every trial's Y+ is a_i(tau) x_i + tau z_i (kernels.cu,
  // diag_t_kernel): one SpMM of T = S_lam(-G) off the diagonal, then O(p)
  // per trial. Needs power-of-two tau (tau0, beta), where omega+ = tau t is
  // exact. ACCORD_LS_NODIAG=1: plain trials.
  auto pow2 = [](double v) { int e; return v > 0 && std::frexp(v, &e) == 0.5; };
  const bool diag_ls = c->omega_identity && c->gemm == ACCORD_GEMM_BF16_FILTER && !c->refit &&
                       c->beta < 1.0 && pow2(c->tau0) && pow2(c->beta) &&
                       !std::getenv("ACCORD_LS_NODIAG");
  const int64_t xrow0 = c->sharded ? 0 : c->r0;   // X^T row of local row 0
  if (diag_ls) {
    CK(cudaEventRecord(c->ev[4], S));
    c->launches += launch_diag_t(c->pk, c->r0, c->c_ptr, c->c_col, (const float*)c->c_g, lam,
                                 (float*)c->c_wn2, S);
    spmm_all(c, c->c_ptr, c->c_col, c->c_wn2, nullptr, nb, nullptr, c->row_Y2);   // Z -> Y[nb]
    c->launches += launch_diag_dots(c->pk, c->ldk, xrow0, (const float*)c->Xt,
                                    (const float*)c->Y[nb], c->diag_xx, c->diag_xz, c->diag_zz, S);
    CK(cudaEventRecord(c->ev[5], S));
    CK(cudaEventSynchronize(c->ev[5]));
    st.ms_spmm += ev_ms(c, 4, 5);
    TR(c, "diag_z");
  }
  // One line-search pass: prox at ta (and at beta*ta when paired), SpMM, the
  // per-trial sums reduced and all-reduced into h_red[0..7] (and [8..15]).
  // Paired: the same gather pass also accumulates D' for beta*ta, so a
  // rejected first step costs no second pass (the sums of the second step are
  // bitwise those of its own pass: the extra entries carry Delta' = 0).
  auto run_trial = [&](double ta, bool paired) {
    CK(cudaEventRecord(c->ev[4], S));
    const ProxItems pitems{c->itm_ptr, c->item_row, c->n_items, kItemEntries, c->itm_dd,
                           c->itm_l1, c->itm_logd, c->itm_nnz};
    const ProxItems* pit = c->items_of == c->c_ptr ? &pitems : nullptr;
    c->launches += launch_prox(c->dtype, c->pk, c->r0, c->c_ptr, c->c_col, c->c_g, c->c_w,
                               c->c_wn, ta, lam, c->row_dd, c->row_l1, c->row_logd,
                               c->row_nnz, S, pit);
    if (paired)
      c->launches += launch_prox(c->dtype, c->pk, c->r0, c->c_ptr, c->c_col, c->c_g, c->c_w,
                                 c->c_wn2, ta * c->beta, lam, c->row_dd2, c->row_l1_2,
                                 c->row_logd2, c->row_nnz2, S, pit);
    CK(cudaEventRecord(c->ev[5], S));
    TR(c, "prox");
    if (diag_ls) {
      c->launches += launch_diag_trial(c->pk, c->r0, c->c_ptr, c->c_col, (const float*)c->c_w,
                                       (const float*)c->c_wn, ta, c->diag_xx, c->diag_xz,
                                       c->diag_zz, c->row_Y2, c->row_D2, c->diag_a, S);
    } else if (paired) {
      if (c->items_of != c->c_ptr) build_items(c, c->c_ptr);
      const bool hi = want_yhi(c) && c->Yhi[nb];
      c->yhi_ok[nb] = hi || !c->Yhi[nb];
      c->launches += launch_spmm_tma(c->pk, c->ldk, c->c_ptr, c->c_col, (const float*)c->c_wn,
                                     (const float*)c->c_w, (const float*)c->Xt, (float*)c->Y[nb],
                                     hi ? c->Yhi[nb] : nullptr, hi ? c->Ylo[nb] : nullptr, c->row_A[nb],
                                     c->row_B[nb], c->row_D2, c->row_Y2, items_view(c),
                                     c->sm_count, S, (const float*)c->c_wn2, c->row_D2b,
                                     c->y_drop);
    } else {
      spmm_all(c, c->c_ptr, c->c_col, c->c_wn, c->c_w, nb, c->row_D2, c->row_Y2);
    }
    CK(cudaEventRecord(c->ev[6], S));
    TR(c, "spmm");
    c->launches += launch_reduce_rows(c->pk, c->row_D2, c->row_dd, c->row_logd, c->row_Y2,
                                      c->row_l1, c->row_nnz, c->c_ptr, c->red_d, S);
    if (paired)
      c->launches += launch_reduce_rows(c->pk, c->row_D2b, c->row_dd2, c->row_logd2, nullptr,
                                        c->row_l1_2, c->row_nnz2, c->c_ptr, c->red_d + 8, S);
    CK(cudaGetLastError());
    allreduce(c, c->red_d, c->h_red, paired ? 16 : 8);
    CK(cudaEventRecord(c->ev[7], S));
    TR(c, "reduce+decide");
    CK(cudaEventSynchronize(c->ev[7]));
    st.ms_prox += ev_ms(c, 4, 5);
    st.ms_spmm += ev_ms(c, 5, 6);
    st.ms_reduce += ev_ms(c, 6, 7);
    for (int k = 0; k < (paired ? 15 : 7); ++k)
      if (k != 7 && !std::isfinite(c->h_red[k])) {
        char m[128];
        std::snprintf(m, sizeof m, "non-finite line-search sum at iteration %lld",
                      (long long)c->iters);
        throw Fail{ACCORD_E_NUMERIC, m};
      }
  };
  const bool pair_ok = c->pair_ls && c->tma_spmm && !c->sharded && c->beta < 1.0 &&
                       c->ldk <= 8 * kSpmmPairMaxConsumers && !diag_ls;
  for (;;) {
    // a trial at or below the 1/L floor is accepted whatever the test says
    const bool paired = pair_ok && !(tau <= c->inv_L);
    run_trial(tau, paired);
    std::memcpy(r, c->h_red, sizeof(r));
    st.trials++;
    // Sufficient decrease in the exact-quadratic form (reading R8):
    // ||Delta X^T||^2 / n <= ||Delta||^2 / tau, or tau <= 1/L.
    double lhs = r[0] / (double)c->n, rhs = r[1] / tau;
    st.ls_lhs = lhs;
    st.ls_rhs = rhs;
    bool floor_hit = tau <= c->inv_L;
    if (c->beta >= 1.0 || lhs <= rhs || floor_hit) {
      st.floor_hit = (!(lhs <= rhs) && floor_hit) ? 1 : 0;
      break;
    }
    if (paired) {   // the second step of the pair, from the same pass
      const double tb = tau * c->beta;
      st.trials++;
      const double lb = c->h_red[8] / (double)c->n, rb = c->h_red[9] / tb;
      if (lb <= rb || tb <= c->inv_L) {
        // accepted: its Y+ (and the committed sums) from a pass of its own
        tau = tb;
        run_trial(tau, false);
        std::memcpy(r, c->h_red, sizeof(r));
        lhs = r[0] / (double)c->n;
        rhs = r[1] / tau;
        st.ls_lhs = lhs;
        st.ls_rhs = rhs;
        floor_hit = tau <= c->inv_L;
        st.floor_hit = (!(lhs <= rhs) && floor_hit) ? 1 : 0;
        break;
      }
      tau = tb * c->beta;
      continue;
    }
    tau *= c->beta;
  }
  // ---------------- accept: Omega <- Omega+, Y <- Y+ ----------------
  if (diag_ls) {
    c->launches += launch_diag_apply(c->pk, c->ldk, xrow0, (const float*)c->Xt, (float*)c->Y[nb],
                                     c->Yhi[nb], c->diag_a, tau, c->row_A[nb], c->row_B[nb], S,
                                     c->y_drop);
    c->yhi_ok[nb] = true;
  }
  c->launches += launch_scan_i32(c->row_nnz, c->om_ptr, c->pk, c->scan_tmp, c->scan_tmp_sz, S);
  c->launches += launch_compact(c->dtype, c->pk, c->r0, c->c_ptr, c->c_col, c->c_wn, c->om_ptr,
                                c->om_col, c->om_val, S);
  if (c->items_of == c->om_ptr) c->items_of = nullptr;   // Omega changed
  c->omega_identity = false;
  TR(c, "compact");
  c->cur = nb;
  int64_t nnz_loc = 0;
  CK(cudaMemcpyAsync(&nnz_loc, c->om_ptr + c->pk, 8, cudaMemcpyDeviceToHost, S));
  CK(cudaGetLastError());
  CK(cudaEventRecord(c->ev[7], S));
  CK(cudaEventSynchronize(c->ev[7]));
  c->nnz_local = nnz_loc;
  const int64_t nnz_before = c->nnz_global;   // the support the GEMM ran at
  c->nnz_global = (int64_t)r[5];
  c->parts[0] = -r[2];
  c->parts[1] = r[3] / (2.0 * (double)c->n);
  c->parts[2] = lam * r[4];
  c->f = c->parts[0] + c->parts[1] + c->parts[2];
  c->iters++;
  st.tau = tau;
  st.f = c->f;
  st.logdet_part = c->parts[0];
  st.g_part = c->parts[1];
  st.l1_part = c->parts[2];
  st.delta_fro = std::sqrt(r[1]);
  st.nnz = (int64_t)r[5];
  st.n_cand = (int64_t)r[6];
  st.max_row_cand = (int64_t)r[7];
  st.ms_total = ev_ms(c, 0, 7);
  TR_flush(c);
  if (!std::isfinite(c->f)) throw Fail{ACCORD_E_NUMERIC, "non-finite objective"};
  // AUTO's operand switch (global |C| and nnz, so every rank takes the same
  // decision): int8 once the bf16 filter's |C| / p is small, or once the new
  // iterate's support is (nnz / p <= i8_nnz = 256: the next C is mostly
  // supp Omega plus the filter's slack; c5: |C| / p = 385, 243, 36 at
  // iterations 1-3, nnz / p = 242, 35, 10 after them), provided
  // |C| / p <= i8_ccap = 512 (not from Omega = I's G = S, whose int8 C is
  // ~5x the bf16 one); back to bf16 if the int8 filter's |C| / p exceeds
  // i8_off
  //
  // Cost check after every int8 GEMM: int8 saves ~40 % of a GEMM pass, i.e.
  // ~0.8 p n / peak per row, and each candidate beyond the support costs a
  // 4n-byte gather in the refine, so the break-even is ~1e-3 p candidates
  // per row beyond supp Omega (c5: ~1000; c3, p = 20,000: ~20). If the int8
  // C held more than i8_excess p^2 entries beyond the support it was computed
  // at, int8 stays off for the solve (c3: 227 - 43 per row; c5: 60 - 9; c4:
  // 41 - 5; c5 iteration 2: 357 - 242). Counts only, so the decision is
  // deterministic and the same on every rank.
  if (c->i8 && !c->i8_force && !c->refit) {
    const double pp = (double)c->p;
    if (st.gemm_i8 && !c->i8_banned &&
        (double)(st.n_cand - nnz_before) > c->i8_excess * pp * pp)
      c->i8_banned = true;
    c->i8_on = !c->i8_banned &&
               (c->i8_on ? (double)st.n_cand <= c->i8_off * pp
                         : ((double)st.n_cand <= c->i8_at * pp ||
                            ((double)st.nnz <= c->i8_nnz * pp &&
                             (double)st.n_cand <= c->i8_ccap * pp)));
  }
  if (c->plan && c->col_sd && !c->sharded && !c->i8 &&
      (double)st.n_cand <= c->x_drop_at * (double)c->p) {
    if (c->x_drop != c->x_drop_target) set_x_width(c, c->x_drop_target);
    c->y_drop = c->y_drop_target;   // from the next Y on (each Y carries its own row norms)
  }
  if (s) *s = st;
}

// lambda_max = max_{i != k} |S_ik| (SPEC.md
// lambda_grid), global (collective). BF16_FILTER: the gradient GEMM at
// Omega = I (A = the rank's rows of X^T_hi) in max-reduce mode gives a
// certified lower bound m on n lambda_max (max over entries of |acc| minus the
// filter bound), then a candidate pass at threshold m / n (1 - 1e-6) holds the
// maximiser, and the refine recomputes the candidates exactly (float64): the
// result is the exact maximum of the f32 data's S. Other GEMM kinds: direct
// float64 dot products on the CUDA cores. The iterate is not changed.
double lambda_max_impl(accord_ctx* c) {
  cudaStream_t S = c->st;
  const int64_t xrow0 = c->sharded ? 0 : c->r0;   // X^T row of local row 0
  const size_t T = c->tsz;
  const char* xrows = (const char*)c->Xt + (size_t)xrow0 * c->ldk * T;
  double* rmax = c->dalloc<double>(std::max<int64_t>(c->pk, 1));
  double* dout = c->dalloc<double>(1);
  struct Tmp {
    accord_ctx* c;
    std::vector<std::pair<void*, size_t>> v;
    ~Tmp() { for (auto& q : v) c->dfree(q.first, q.second); }
  } tmp{c, {{rmax, std::max<int64_t>(c->pk, 1) * 8}, {dout, 8}}};
  const bool filt = c->gemm == ACCORD_GEMM_BF16_FILTER &&
                    (c->sharded || c->r0 + c->pk_pad <= c->xrows_pad);
  if (!filt) {
    if (!c->sharded) {
      c->launches += launch_gram_offdiag_max(c->dtype, c->pk, c->r0, c->n, c->ldk, xrows, c->Xt, 0,
                                             c->p, 0, rmax, dout, S);
    } else {
      ring_pass(c, false, [&](const void* slab, int, int64_t v0, int64_t v1, bool first, bool last) {
        c->launches += launch_gram_offdiag_max(c->dtype, c->pk, c->r0, c->n, c->ldk, xrows, slab,
                                               v0, v1, first ? 0 : 1, rmax, last ? dout : nullptr,
                                               S);
      });
    }
    CK(cudaGetLastError());
    return allreduce_max(c, dout);
  }
  // ---- tensor-core filter path ----
  if (!c->plan_a_x) {
    std::string e;
    const __nv_bfloat16* xh = c->Xhi + (size_t)xrow0 * c->ldk;
    if (!tc_plan_set_a(c->plan, 2, xh, c->pk_pad, &e)) throw Fail{ACCORD_E_CUDA, "tensor map: " + e};
    c->plan_a_x = true;
  }
  float* rA = c->dalloc<float>(std::max<int64_t>(c->pk, 1));
  float* rB = c->dalloc<float>(std::max<int64_t>(c->pk, 1));
  int64_t* eptr = c->dalloc<int64_t>(c->pk + 1);   // empty support (diagonal is emitted anyway)
  unsigned int* dmax = c->dalloc<unsigned int>(1);
  tmp.v.push_back({rA, std::max<int64_t>(c->pk, 1) * 4});
  tmp.v.push_back({rB, std::max<int64_t>(c->pk, 1) * 4});
  tmp.v.push_back({eptr, (c->pk + 1) * 8});
  tmp.v.push_back({dmax, 4});
  CK(cudaMemsetAsync(eptr, 0, (c->pk + 1) * 8, S));
  CK(cudaMemsetAsync(dmax, 0, 4, S));
  c->launches += launch_row_ab(c->pk, c->ldk, (const float*)xrows, rA, rB, S, c->x_drop);
  // int8 operands: the rank's X^T rows quantised per row into the spare int8
  // Y buffer (the int8 buffers are re-quantised before every GEMM); the
  // columns are the permuted int8 X^T, so no symmetric schedule
  const int qb = 1 - c->cur;
  if (c->i8)
    c->launches += launch_quant_y_i8(c->pk, c->n, c->ldk, (const float*)xrows, c->Yq[qb],
                                     c->yq_s[qb], c->yq_A[qb], c->yq_B[qb], S);
  GradOverride ov{c->i8 ? qb : 2, c->i8 ? c->yq_A[qb] : rA, c->i8 ? c->yq_B[qb] : rB,
                  c->i8 ? c->yq_s[qb] : nullptr, OmegaView{eptr, c->om_col, c->om_val}, 0.0, dmax,
                  !c->i8 && c->world == 1 && !c->sharded && c->r0 == 0 && c->pk == c->p &&
                      !std::getenv("ACCORD_GEMM_NOSYM")};
  accord_iter_stats st{};
  build_candidates(c, st, &ov);                      // pass 1: certified lower bound
  unsigned int hm = 0;
  CK(cudaMemcpyAsync(&hm, dmax, 4, cudaMemcpyDeviceToHost, S));
  csync(c, S);
  float lb = 0.f;
  std::memcpy(&lb, &hm, 4);
  double lbd = (double)lb;
  {   // the global lower bound (every rank's maximiser must be kept)
    double* d = c->red_d + 8;
    CK(cudaMemcpyAsync(d, &lbd, 8, cudaMemcpyHostToDevice, S));
    lbd = allreduce_max(c, d);
  }
  ov.max_out = nullptr;
  ov.lam_cand = std::max(0.0, lbd / (double)c->n * (1.0 - 1e-6));
  build_candidates(c, st, &ov);                      // pass 2: the candidates near the max
  c->items_of = nullptr;
  // their values exactly (float64 dots of the f32 data)
  if (!c->sharded) {
    c->launches += launch_cand_dot_max(c->dtype, c->pk, c->r0, c->n, c->ldk, c->c_ptr, c->c_col,
                                       xrows, c->Xt, 0, c->p, 0, rmax, dout, S);
  } else {
    ring_pass(c, false, [&](const void* slab, int, int64_t v0, int64_t v1, bool first, bool last) {
      c->launches += launch_cand_dot_max(c->dtype, c->pk, c->r0, c->n, c->ldk, c->c_ptr, c->c_col,
                                         xrows, slab, v0, v1, first ? 0 : 1, rmax,
                                         last ? dout : nullptr, S);
    });
  }
  CK(cudaGetLastError());
  return allreduce_max(c, dout);
}

// Gather every rank's row block of Omega into one global host CSR (collective).
// fetch = false: only the global nnz.
void gather_host(accord_ctx* c, bool fetch, int64_t* total_out, std::vector<int64_t>* gp_out,
                 std::vector<int32_t>* gc_out, std::vector<char>* gv_out) {
    const size_t T = c->tsz;
    // ---- gather all ranks' row blocks (collective) ----
    // 1) per-rank (rows, nnz)
    std::vector<double> h(2 * c->world, 0.0);
    double* d = c->red_d;
    std::vector<double> mine(2 * c->world, 0.0);
    mine[2 * c->rank] = (double)c->pk;
    mine[2 * c->rank + 1] = (double)c->nnz_local;
    std::vector<double> tot(2 * c->world);
    for (int q = 0; q < 2 * c->world; q += 8) {
      const int cnt = std::min(8, 2 * c->world - q);
      CK(cudaMemcpyAsync(d, mine.data() + q, cnt * 8, cudaMemcpyHostToDevice, c->st));
      allreduce(c, d, c->h_red, cnt);
      std::memcpy(tot.data() + q, c->h_red, cnt * 8);
    }
    int64_t total = 0, rows_total = 0;
    for (int q = 0; q < c->world; ++q) {
      rows_total += (int64_t)tot[2 * q];
      total += (int64_t)tot[2 * q + 1];
    }
    *total_out = total;
    if (!fetch) return;
    if (rows_total != c->p) throw Fail{ACCORD_E_INVALID, "row blocks do not cover p rows"};
    // local block to host
    std::vector<int64_t> lp(c->pk + 1);
    std::vector<int32_t> lc(c->nnz_local);
    std::vector<char> lv(c->nnz_local * T);
    CK(cudaMemcpyAsync(lp.data(), c->om_ptr, (c->pk + 1) * 8, cudaMemcpyDeviceToHost, c->st));
    CK(cudaMemcpyAsync(lc.data(), c->om_col, c->nnz_local * 4, cudaMemcpyDeviceToHost, c->st));
    CK(cudaMemcpyAsync(lv.data(), c->om_val, c->nnz_local * T, cudaMemcpyDeviceToHost, c->st));
    csync(c, c->st);
    std::vector<int64_t>& gp = *gp_out;
    std::vector<int32_t>& gc = *gc_out;
    std::vector<char>& gv = *gv_out;
    gp.assign(c->p + 1, 0);
    gc.resize(total);
    gv.resize(total * T);
    if (c->comm == ACCORD_COMM_NCCL) {
      NcclApi* api = nccl_api();
      int64_t* dptr = nullptr;
      int32_t* dcol = nullptr;
      char* dval = nullptr;
      dptr = c->dalloc<int64_t>(rows_total + c->world);
      dcol = c->dalloc<int32_t>(std::max<int64_t>(total, 1));
      dval = c->dalloc<char>(std::max<int64_t>(total, 1) * T);
      int64_t ro = 0, eo = 0;
      NK(api->GroupStart());
      for (int q = 0; q < c->world; ++q) {
        const int64_t rq = (int64_t)tot[2 * q], nq = (int64_t)tot[2 * q + 1];
        const bool me = q == c->rank;
        NK(api->Broadcast(me ? (const void*)c->om_ptr : nullptr, dptr + ro + q, (rq + 1) * 8,
                          ncclChar, q, c->nccl, c->st));
        if (nq > 0) {
          NK(api->Broadcast(me ? (const void*)c->om_col : nullptr, dcol + eo, nq * 4, ncclChar, q,
                            c->nccl, c->st));
          NK(api->Broadcast(me ? (const void*)c->om_val : nullptr, dval + eo * T, nq * T,
                            ncclChar, q, c->nccl, c->st));
        }
        ro += rq;
        eo += nq;
      }
      NK(api->GroupEnd());
      std::vector<int64_t> hp(rows_total + c->world);
      CK(cudaMemcpyAsync(hp.data(), dptr, hp.size() * 8, cudaMemcpyDeviceToHost, c->st));
      CK(cudaMemcpyAsync(gc.data(), dcol, total * 4, cudaMemcpyDeviceToHost, c->st));
      CK(cudaMemcpyAsync(gv.data(), dval, total * T, cudaMemcpyDeviceToHost, c->st));
      csync(c, c->st);
      c->dfree(dptr, (rows_total + c->world) * 8);
      c->dfree(dcol, std::max<int64_t>(total, 1) * 4);
      c->dfree(dval, std::max<int64_t>(total, 1) * T);
      ro = 0;
      eo = 0;
      for (int q = 0; q < c->world; ++q) {
        const int64_t rq = (int64_t)tot[2 * q];
        for (int64_t i = 0; i <= rq; ++i) gp[ro + i] = eo + hp[ro + q + i];
        ro += rq;
        eo += (int64_t)tot[2 * q + 1];
      }
    } else {
      if (!c->agv) throw Fail{ACCORD_E_INVALID, "GATHER with host comm needs allgatherv"};
      // pack [rows][nnz][row_ptr][col][val]
      std::vector<char> blob(16 + lp.size() * 8 + lc.size() * 4 + lv.size());
      int64_t hdr[2] = {c->pk, c->nnz_local};
      char* w = blob.data();
      std::memcpy(w, hdr, 16); w += 16;
      std::memcpy(w, lp.data(), lp.size() * 8); w += lp.size() * 8;
      std::memcpy(w, lc.data(), lc.size() * 4); w += lc.size() * 4;
      std::memcpy(w, lv.data(), lv.size());
      std::vector<int64_t> counts(c->world, 0);
      if (c->agv(c->cu, blob.data(), (int64_t)blob.size(), nullptr, counts.data()) != 0)
        throw Fail{ACCORD_E_COMM, "allgatherv (sizes) failed"};
      int64_t all = 0;
      for (auto x : counts) all += x;
      std::vector<char> buf(all);
      if (c->agv(c->cu, blob.data(), (int64_t)blob.size(), buf.data(), counts.data()) != 0)
        throw Fail{ACCORD_E_COMM, "allgatherv failed"};
      const char* rd = buf.data();
      int64_t ro = 0, eo = 0;
      for (int q = 0; q < c->world; ++q) {
        int64_t hq[2];
        std::memcpy(hq, rd, 16);
        const int64_t* qp = (const int64_t*)(rd + 16);
        for (int64_t i = 0; i <= hq[0]; ++i) gp[ro + i] = eo + qp[i];
        std::memcpy(gc.data() + eo, rd + 16 + (hq[0] + 1) * 8, hq[1] * 4);
        std::memcpy(gv.data() + eo * T, rd + 16 + (hq[0] + 1) * 8 + hq[1] * 4, hq[1] * T);
        rd += counts[q];
        ro += hq[0];
        eo += hq[1];
      }
    }
}

}  // namespace

// ============================================================================
// C ABI
// ============================================================================
extern "C" {

void accord_default_params(accord_init_params* prm) {
  if (!prm) return;
  std::memset(prm, 0, sizeof(*prm));
  prm->abi_version = ACCORD_ABI_VERSION;
  prm->device = -1;
  prm->layout = ACCORD_LAYOUT_SAMPLES_ROW_MAJOR;
  prm->dtype = ACCORD_F32;
  prm->gemm = ACCORD_GEMM_AUTO;
  prm->tau0 = 0.5;
  prm->beta = 0.5;
  prm->world = 1;
  prm->comm = ACCORD_COMM_NONE;
}

accord_status accord_workspace_size(const accord_init_params* prm, size_t* bytes) {
  g_create_err.clear();
  if (!bytes) {
    g_create_err = "bytes is NULL";
    return ACCORD_E_INVALID;
  }
  try {
    validate(prm);
    *bytes = footprint(prm).total + 4096;   // + the arena's alignment slack
    return ACCORD_OK;
  } catch (const Fail& f) {
    g_create_err = f.msg;
    return f.s;
  } catch (...) {
    g_create_err = "internal error";
    return ACCORD_E_INVALID;
  }
}

accord_status accord_create(accord_ctx** out, const accord_init_params* prm) {
  g_create_err.clear();
  if (!out) {
    g_create_err = "out is NULL";
    return ACCORD_E_INVALID;
  }
  *out = nullptr;
  accord_ctx* c = new (std::nothrow) accord_ctx();
  if (!c) return ACCORD_E_NOMEM;
  accord_status s = guard(c, [&] { create_impl(c, prm); });
  if (s != ACCORD_OK) {
    g_create_err = c->err;
    accord_destroy(c);
    return s;
  }
  *out = c;
  return ACCORD_OK;
}

accord_status accord_step(accord_ctx* c, int32_t iters, accord_iter_stats* stats) {
  if (!c) return ACCORD_E_INVALID;
  if (iters < 0) {
    c->err = "iters < 0";
    return ACCORD_E_INVALID;
  }
  return guard(c, [&] {
    for (int32_t i = 0; i < iters; ++i) step_one(c, stats ? stats + i : nullptr);
  });
}

accord_status accord_objective(accord_ctx* c, double* f, double* parts) {
  if (!c) return ACCORD_E_INVALID;
  if (f) *f = c->f;
  if (parts) std::memcpy(parts, c->parts, sizeof(c->parts));
  return ACCORD_OK;
}

accord_status accord_export_csr(accord_ctx* c, int32_t scope, int64_t* row_ptr, int32_t* col,
                                void* val, int64_t capacity, int64_t* nnz_out,
                                int32_t on_device) {
  if (!c || !nnz_out) return ACCORD_E_INVALID;
  return guard(c, [&] {
    const size_t T = c->tsz;
    const cudaMemcpyKind k = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    if (scope == ACCORD_SCOPE_LOCAL || (c->world == 1 && c->comm != ACCORD_COMM_NCCL)) {
      *nnz_out = c->nnz_local;
      if (!row_ptr) return;
      if (capacity < c->nnz_local) throw Fail{ACCORD_E_CAPACITY, "capacity too small"};
      CK(cudaMemcpyAsync(row_ptr, c->om_ptr, (c->pk + 1) * 8, k, c->st));
      CK(cudaMemcpyAsync(col, c->om_col, c->nnz_local * 4, k, c->st));
      CK(cudaMemcpyAsync(val, c->om_val, c->nnz_local * T, k, c->st));
      csync(c, c->st);
      return;
    }
    if (scope != ACCORD_SCOPE_GATHER) throw Fail{ACCORD_E_INVALID, "bad scope"};
    std::vector<int64_t> gp;
    std::vector<int32_t> gc;
    std::vector<char> gv;
    int64_t total = 0;
    gather_host(c, !!row_ptr, &total, &gp, &gc, &gv);
    *nnz_out = total;
    if (!row_ptr) return;
    if (capacity < total) throw Fail{ACCORD_E_CAPACITY, "capacity too small"};
    const cudaMemcpyKind hk = on_device ? cudaMemcpyHostToDevice : cudaMemcpyHostToHost;
    CK(cudaMemcpy(row_ptr, gp.data(), gp.size() * 8, hk));
    CK(cudaMemcpy(col, gc.data(), gc.size() * 4, hk));
    CK(cudaMemcpy(val, gv.data(), gv.size(), hk));
  });
}

// NEXT(4): Theta-hat = Omega_D Omega and the partial correlations rho-hat
// computed on the device (postproc.cu).
accord_status accord_export_transformed(accord_ctx* c, int32_t kind, int32_t scope,
                                        int64_t* row_ptr, int32_t* col, void* val,
                                        int64_t capacity, int64_t* nnz_out, int32_t on_device) {
  if (!c || !nnz_out) return ACCORD_E_INVALID;
  if (kind == ACCORD_EXPORT_OMEGA)
    return accord_export_csr(c, scope, row_ptr, col, val, capacity, nnz_out, on_device);
  return guard(c, [&] {
    if (kind != ACCORD_EXPORT_THETA && kind != ACCORD_EXPORT_PCORR)
      throw Fail{ACCORD_E_INVALID, "bad export kind"};
    if (scope != ACCORD_SCOPE_LOCAL && scope != ACCORD_SCOPE_GATHER)
      throw Fail{ACCORD_E_INVALID, "bad scope"};
    const size_t T = c->tsz;
    cudaStream_t S = c->st;
    // temporaries of this call only
    std::vector<std::pair<void*, size_t>> tmp;
    struct Free {
      accord_ctx* c;
      std::vector<std::pair<void*, size_t>>& v;
      ~Free() {
        if (c->st) cudaStreamSynchronize(c->st);
        for (auto& q : v) c->dfree(q.first, q.second);
      }
    } fr{c, tmp};
    auto talloc = [&](size_t b) {
      void* q = c->dalloc_bytes(b);
      tmp.push_back({q, b});
      return q;
    };
    // The input CSR: this rank's block (THETA of the local rows, or P = 1) or the
    // gathered global Omega (collective) uploaded to the device.
    const bool local_in = c->world == 1 || (kind == ACCORD_EXPORT_THETA && scope == ACCORD_SCOPE_LOCAL);
    const int64_t* iptr = c->om_ptr;
    const int32_t* icol = c->om_col;
    const void* ival = c->om_val;
    int64_t irows = c->pk, ioff = c->r0;
    if (!local_in) {
      std::vector<int64_t> gp;
      std::vector<int32_t> gc;
      std::vector<char> gv;
      int64_t total = 0;
      gather_host(c, true, &total, &gp, &gc, &gv);
      int64_t* dp = (int64_t*)talloc(gp.size() * 8);
      int32_t* dc = (int32_t*)talloc(gc.size() * 4);
      void* dv = talloc(gv.size());
      CK(cudaMemcpyAsync(dp, gp.data(), gp.size() * 8, cudaMemcpyHostToDevice, S));
      CK(cudaMemcpyAsync(dc, gc.data(), gc.size() * 4, cudaMemcpyHostToDevice, S));
      CK(cudaMemcpyAsync(dv, gv.data(), gv.size(), cudaMemcpyHostToDevice, S));
      csync(c, S);   // the host vectors go out of scope
      iptr = dp;
      icol = dc;
      ival = dv;
      irows = c->p;
      ioff = 0;
    }
    // output rows [a, b) of the input CSR
    const bool all = scope == ACCORD_SCOPE_GATHER || c->world == 1;
    const int64_t a = all || local_in ? 0 : c->r0, b = all ? irows : (local_in ? irows : c->r1);
    const int64_t rows = b - a;
    double* d = (double*)talloc(irows * 8);
    int32_t* bad = (int32_t*)talloc(4);
    CK(cudaMemsetAsync(bad, 0, 4, S));
    c->launches += launch_diag(c->dtype, irows, ioff, iptr, icol, ival, d, bad, S);
    int64_t* optr = nullptr;
    int32_t* ocol = nullptr;
    void* oval = nullptr;
    int64_t h_ab[2] = {0, 0};
    CK(cudaMemcpyAsync(h_ab, iptr + a, 8, cudaMemcpyDeviceToHost, S));
    CK(cudaMemcpyAsync(h_ab + 1, iptr + b, 8, cudaMemcpyDeviceToHost, S));
    int32_t hbad = 0;
    CK(cudaMemcpyAsync(&hbad, bad, 4, cudaMemcpyDeviceToHost, S));
    csync(c, S);
    if (hbad) throw Fail{ACCORD_E_DOMAIN, "Omega has a missing or nonpositive diagonal entry"};
    int64_t nnz = 0;
    if (kind == ACCORD_EXPORT_THETA) {
      nnz = h_ab[1] - h_ab[0];
      oval = talloc(nnz * T);
      c->launches += launch_theta(c->dtype, a, b, iptr, icol, ival, d, oval, S);
      // structure = Omega's rows [a, b), rebased to 0
      optr = (int64_t*)talloc((rows + 1) * 8);
      std::vector<int64_t> hp(rows + 1);
      CK(cudaMemcpyAsync(hp.data(), iptr + a, (rows + 1) * 8, cudaMemcpyDeviceToHost, S));
      csync(c, S);
      for (auto& x : hp) x -= h_ab[0];
      CK(cudaMemcpyAsync(optr, hp.data(), (rows + 1) * 8, cudaMemcpyHostToDevice, S));
      ocol = const_cast<int32_t*>(icol) + h_ab[0];
      csync(c, S);
    } else {
      int32_t* own = (int32_t*)talloc(rows * 4);
      int32_t* cnt = (int32_t*)talloc(rows * 4);
      int32_t* ext = (int32_t*)talloc(rows * 4);
      int32_t* long_rows = (int32_t*)talloc((rows + 1) * 4);
      optr = (int64_t*)talloc((rows + 1) * 8);
      CK(cudaMemsetAsync(own, 0, rows * 4, S));
      CK(cudaMemsetAsync(cnt, 0, rows * 4, S));
      CK(cudaMemsetAsync(ext, 0, rows * 4, S));
      CK(cudaMemsetAsync(long_rows, 0, 4, S));
      c->launches += launch_pcorr_count(c->dtype, irows, a, b, iptr, icol, ival, own, cnt, S);
      void* stmp = talloc(scan_tmp_bytes(rows + 1));
      c->launches += launch_scan_i32(cnt, optr, rows, stmp, scan_tmp_bytes(rows + 1), S);
      CK(cudaMemcpyAsync(&nnz, optr + rows, 8, cudaMemcpyDeviceToHost, S));
      csync(c, S);
      uint64_t* keys = (uint64_t*)talloc(nnz * 8);
      uint64_t* ktmp = (uint64_t*)talloc(nnz * 8);
      c->launches += launch_pcorr_fill(c->dtype, irows, a, b, iptr, icol, ival, own, optr, ext,
                                       keys, S);
      c->launches += launch_rowsort(rows, optr, keys, ktmp, long_rows, S);
      ocol = (int32_t*)talloc(nnz * 4);
      oval = talloc(nnz * T);
      c->launches += launch_pcorr_value(c->dtype, a, b, iptr, icol, ival, d, optr, keys, ocol,
                                        oval, S);
    }
    CK(cudaGetLastError());
    *nnz_out = nnz;
    if (!row_ptr) {
      csync(c, S);
      return;
    }
    if (capacity < nnz) throw Fail{ACCORD_E_CAPACITY, "capacity too small"};
    const cudaMemcpyKind k = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    CK(cudaMemcpyAsync(row_ptr, optr, (rows + 1) * 8, k, S));
    CK(cudaMemcpyAsync(col, ocol, nnz * 4, k, S));
    CK(cudaMemcpyAsync(val, oval, nnz * T, k, S));
    csync(c, S);
  });
}

accord_status accord_set_omega_csr(accord_ctx* c, const int64_t* row_ptr, const int32_t* col,
                                   const void* val, int64_t nnz) {
  if (!c || !row_ptr || (nnz > 0 && (!col || !val))) return ACCORD_E_INVALID;
  return guard(c, [&] {
    if (row_ptr[0] != 0 || row_ptr[c->pk] != nnz) throw Fail{ACCORD_E_INVALID, "bad row_ptr"};
    for (int64_t i = 0; i < c->pk; ++i) {
      if (row_ptr[i + 1] < row_ptr[i]) throw Fail{ACCORD_E_INVALID, "row_ptr not monotone"};
      for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
        if (col[e] < 0 || col[e] >= c->p) throw Fail{ACCORD_E_INVALID, "column out of range"};
        if (e > row_ptr[i] && col[e] <= col[e - 1])
          throw Fail{ACCORD_E_INVALID, "columns not strictly increasing"};
      }
    }
    if (nnz > c->cap) grow(c, nnz + nnz / 4 + 1024, 0);
    CK(cudaMemcpyAsync(c->om_ptr, row_ptr, (c->pk + 1) * 8, cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(c->om_col, col, nnz * 4, cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(c->om_val, val, nnz * c->tsz, cudaMemcpyHostToDevice, c->st));
    c->nnz_local = nnz;
    recompute_y(c);
    refresh_objective(c);
  });
}

accord_status accord_set_lambda(accord_ctx* c, double lambda) {
  if (!c) return ACCORD_E_INVALID;
  if (!(lambda >= 0) || !std::isfinite(lambda)) {
    c->err = "lambda must be finite and >= 0";
    return ACCORD_E_INVALID;
  }
  return guard(c, [&] {
    c->lam = lambda;
    // AUTO's int8 cost check starts over (the candidate density depends on lambda)
    c->i8_banned = false;
    refresh_objective(c);
  });
}

accord_status accord_refit(accord_ctx* c, double phi) {
  if (!c) return ACCORD_E_INVALID;
  if (!(phi >= 0 && phi <= 1)) {
    c->err = "phi must be in [0, 1] (Eq. 3.8)";
    return ACCORD_E_INVALID;
  }
  return guard(c, [&] {
    // S_hat = support of the current estimate (diagonal always stored)
    c->dfree(c->refit_ptr, (c->pk + 1) * 8);
    c->dfree(c->refit_col, c->refit_nnz * 4);
    c->refit_nnz = c->nnz_local;
    c->refit_ptr = c->dalloc<int64_t>(c->pk + 1);
    c->refit_col = c->dalloc<int32_t>(std::max<int64_t>(c->refit_nnz, 1));
    CK(cudaMemcpyAsync(c->refit_ptr, c->om_ptr, (c->pk + 1) * 8, cudaMemcpyDeviceToDevice,
                       c->st));
    CK(cudaMemcpyAsync(c->refit_col, c->om_col, c->refit_nnz * 4, cudaMemcpyDeviceToDevice,
                       c->st));
    c->refit = true;
    c->phi = phi;
    refresh_objective(c);
  });
}

accord_status accord_solve(accord_ctx* c, int32_t max_iter, double tol, int32_t* iters_done,
                           accord_iter_stats* last) {
  if (!c || max_iter < 0 || !(tol >= 0)) return ACCORD_E_INVALID;
  return guard(c, [&] {
    accord_iter_stats st{};
    int32_t it = 0;
    while (it < max_iter) {
      step_one(c, &st);
      ++it;
      if (st.delta_fro < tol) break;   // ||Omega^(t+1) - Omega^(t)||_F < tol (reading R13)
    }
    if (iters_done) *iters_done = it;
    if (last) *last = st;
  });
}

accord_status accord_kkt_residual(accord_ctx* c, double* kkt) {
  if (!c || !kkt) return ACCORD_E_INVALID;
  return guard(c, [&] {
    accord_iter_stats st{};
    build_candidates(c, st);
    c->launches += launch_kkt(c->dtype, c->pk, c->r0, c->c_ptr, c->c_col, c->c_g, c->c_w,
                              lam_eff(c), c->row_dd, c->red_d + 8, c->st);
    CK(cudaGetLastError());
    *kkt = allreduce_max(c, c->red_d + 8);
  });
}

accord_status accord_path(accord_ctx* c, const double* lambdas, int32_t k, int32_t max_iter,
                          double tol, double gamma, double* epbic, int64_t* nnz_off,
                          int32_t* iters, int32_t* best) {
  if (!c || !lambdas || k < 1 || max_iter < 1 || !(gamma >= 0)) return ACCORD_E_INVALID;
  return guard(c, [&] {
    const size_t T = c->tsz;
    int64_t* bptr = c->dalloc<int64_t>(c->pk + 1);
    int32_t* bcol = nullptr;
    void* bval = nullptr;
    int64_t bcap = 0, bnnz = 0;
    double best_e = INFINITY, best_lam = c->lam;
    int32_t bi = 0;
    for (int32_t j = 0; j < k; ++j) {
      if (!(lambdas[j] >= 0) || !std::isfinite(lambdas[j]))
        throw Fail{ACCORD_E_INVALID, "bad lambda in the path"};
      c->lam = lambdas[j];
      refresh_objective(c);                       // warm start from the previous estimate
      accord_iter_stats st{};
      int32_t it = 0;
      while (it < max_iter) {
        step_one(c, &st);
        ++it;
        if (st.delta_fro < tol) break;
      }
      // epBIC, Eq. (3.7): 2n (loss) + ||Omega||_0 (log n + 4 gamma log p), off-diagonal count
      const double loss = c->parts[0] + c->parts[1];
      const int64_t koff = c->nnz_global - c->p;
      const double e = 2.0 * (double)c->n * loss +
                       (double)koff * (std::log((double)c->n) + 4.0 * gamma * std::log((double)c->p));
      if (epbic) epbic[j] = e;
      if (nnz_off) nnz_off[j] = koff;
      if (iters) iters[j] = it;
      if (e < best_e) {
        best_e = e;
        best_lam = lambdas[j];
        bi = j;
        if (c->nnz_local > bcap) {
          c->dfree(bcol, bcap * 4);
          c->dfree(bval, bcap * T);
          bcap = c->nnz_local + c->nnz_local / 4 + 16;
          bcol = c->dalloc<int32_t>(bcap);
          bval = c->dalloc_bytes(bcap * T);
        }
        bnnz = c->nnz_local;
        CK(cudaMemcpyAsync(bptr, c->om_ptr, (c->pk + 1) * 8, cudaMemcpyDeviceToDevice, c->st));
        CK(cudaMemcpyAsync(bcol, c->om_col, bnnz * 4, cudaMemcpyDeviceToDevice, c->st));
        CK(cudaMemcpyAsync(bval, c->om_val, bnnz * T, cudaMemcpyDeviceToDevice, c->st));
      }
    }
    // restore the epBIC-selected estimate (and its lambda)
    CK(cudaMemcpyAsync(c->om_ptr, bptr, (c->pk + 1) * 8, cudaMemcpyDeviceToDevice, c->st));
    CK(cudaMemcpyAsync(c->om_col, bcol, bnnz * 4, cudaMemcpyDeviceToDevice, c->st));
    CK(cudaMemcpyAsync(c->om_val, bval, bnnz * T, cudaMemcpyDeviceToDevice, c->st));
    csync(c, c->st);
    c->dfree(bptr, (c->pk + 1) * 8);
    c->dfree(bcol, bcap * 4);
    c->dfree(bval, bcap * T);
    c->nnz_local = bnnz;
    c->lam = best_lam;
    recompute_y(c);
    refresh_objective(c);
    if (best) *best = bi;
  });
}

accord_status accord_lambda_max(accord_ctx* c, double* lmax) {
  if (!c || !lmax) return ACCORD_E_INVALID;
  return guard(c, [&] {
    const double v = lambda_max_impl(c);
    if (!(v > 0) || !std::isfinite(v))
      throw Fail{ACCORD_E_NUMERIC, "lambda_max is not positive (all-zero or uncorrelated data)"};
    *lmax = v;
  });
}

accord_status accord_lambda_grid(accord_ctx* c, int32_t k, double ratio, double* lambdas) {
  if (!c || !lambdas || k < 1 || !(ratio > 0 && ratio < 1)) {
    if (c) c->err = "need k >= 1 and 0 < ratio < 1";
    return ACCORD_E_INVALID;
  }
  double lm = 0;
  const accord_status s = accord_lambda_max(c, &lm);
  if (s != ACCORD_OK) return s;
  // k log-evenly spaced points from lambda_max down to ratio * lambda_max
  for (int32_t j = 0; j < k; ++j)
    lambdas[j] = k == 1 ? lm : lm * std::pow(ratio, (double)j / (double)(k - 1));
  return ACCORD_OK;
}

accord_status accord_filter_audit(accord_ctx* c, float* acc, int64_t ld, float* y, int64_t ldy,
                                  float* row_ab, float* col_sd, double* gamma, int64_t* c_ptr,
                                  int32_t* c_col, int64_t capacity, int64_t* n_cand) {
  if (!c || !acc || !n_cand) return ACCORD_E_INVALID;
  return guard(c, [&] {
    if (c->gemm != ACCORD_GEMM_BF16_FILTER)
      throw Fail{ACCORD_E_UNSUPPORTED, "filter audit needs the BF16_FILTER GEMM"};
    if (ld < c->p) throw Fail{ACCORD_E_INVALID, "ld < p"};
    if (y && ldy < c->n) throw Fail{ACCORD_E_INVALID, "ldy < n"};
    c->audit_acc = acc;
    c->audit_ld = ld;
    accord_iter_stats st{};
    try {
      build_candidates(c, st);
    } catch (...) {
      c->audit_acc = nullptr;
      throw;
    }
    c->audit_acc = nullptr;
    cudaStream_t S = c->st;
    if (y)
      CK(cudaMemcpy2DAsync(y, ldy * 4, c->Y[c->cur], c->ldk * 4, c->n * 4, c->pk,
                           cudaMemcpyDeviceToDevice, S));
    const bool q = c->i8_last;   // the audited GEMM ran in int8: its constants, gamma = 0
    if (row_ab) {
      CK(cudaMemcpyAsync(row_ab, q ? c->yq_A[c->cur] : c->row_A[c->cur], c->pk * 4,
                         cudaMemcpyDeviceToHost, S));
      CK(cudaMemcpyAsync(row_ab + c->pk, q ? c->yq_B[c->cur] : c->row_B[c->cur], c->pk * 4,
                         cudaMemcpyDeviceToHost, S));
    }
    if (col_sd)
      CK(cudaMemcpyAsync(col_sd, q ? c->col_sd_q : c->col_sd, c->p * 8, cudaMemcpyDeviceToHost, S));
    if (gamma)
      *gamma = q ? 0.0
                     : (double)(float)(((double)c->ldk / 16.0 + 17.0) * std::ldexp(1.0, -22));
    int64_t nc = 0;
    CK(cudaMemcpyAsync(&nc, c->c_ptr + c->pk, 8, cudaMemcpyDeviceToHost, S));
    csync(c, S);
    *n_cand = nc;
    if (!c_ptr) return;
    if (capacity < nc) throw Fail{ACCORD_E_CAPACITY, "capacity too small"};
    CK(cudaMemcpyAsync(c_ptr, c->c_ptr, (c->pk + 1) * 8, cudaMemcpyDeviceToHost, S));
    CK(cudaMemcpyAsync(c_col, c->c_col, nc * 4, cudaMemcpyDeviceToHost, S));
    csync(c, S);
  });
}

accord_status accord_row_stats(accord_ctx* c, const int64_t* rows, int64_t count, double* d2,
                               double* delta2) {
  if (!c || (count > 0 && !rows)) return ACCORD_E_INVALID;
  return guard(c, [&] {
    std::vector<double> a(c->pk), b(c->pk);
    CK(cudaMemcpyAsync(a.data(), c->row_D2, c->pk * 8, cudaMemcpyDeviceToHost, c->st));
    CK(cudaMemcpyAsync(b.data(), c->row_dd, c->pk * 8, cudaMemcpyDeviceToHost, c->st));
    csync(c, c->st);
    for (int64_t q = 0; q < count; ++q) {
      if (rows[q] < 0 || rows[q] >= c->pk) throw Fail{ACCORD_E_INVALID, "row out of range"};
      if (d2) d2[q] = a[rows[q]];
      if (delta2) delta2[q] = b[rows[q]];
    }
  });
}

accord_status accord_get_info(accord_ctx* c, accord_info* info) {
  if (!c || !info) return ACCORD_E_INVALID;
  std::memset(info, 0, sizeof(*info));
  info->n = c->n;
  info->p = c->p;
  info->row_begin = c->r0;
  info->row_end = c->r1;
  info->ldk = c->ldk;
  info->L = c->L;
  info->inv_L = c->inv_L;
  info->lambda = c->lam;
  info->tau0 = c->tau0;
  info->beta = c->beta;
  info->dtype = c->dtype;
  info->gemm = (c->i8_force || c->gemm_launches_i8 > 0) ? (int)ACCORD_GEMM_I8_FILTER : c->gemm;
  info->gemm_launches_i8 = c->gemm_launches_i8;
  info->sm_count = c->sm_count;
  info->cc_major = c->cc_major;
  info->cc_minor = c->cc_minor;
  info->iterations = c->iters;
  info->nnz_local = c->nnz_local;
  info->cand_capacity = c->cap;
  info->kernel_launches = c->launches;
  info->gemm_launches = c->gemm_launches;
  info->f = c->f;
  info->device_bytes = c->bytes;
  info->workspace_bytes = c->arena.size;
  info->workspace_high = c->arena.high;
  info->mirrored_sent = c->mirrored_sent;
  return ACCORD_OK;
}

accord_status accord_nccl_unique_id(uint8_t id[128]) {
  NcclApi* api = nccl_api();
  if (!api || !id) return ACCORD_E_NCCL;
  ncclUniqueId u;
  if (api->GetUniqueId(&u) != ncclSuccess) return ACCORD_E_NCCL;
  std::memcpy(id, &u, 128);
  return ACCORD_OK;
}

void accord_destroy(accord_ctx* c) {
  if (!c) return;
  if (c->st) cudaStreamSynchronize(c->st);
  else cudaDeviceSynchronize();
  if (c->plan) tc_plan_destroy(c->plan);
  // (buffers carved out of a caller workspace belong to the caller's allocation)
  if (!c->arena.base)
    for (void* ptr : c->allocs) cudaFree(ptr);
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : c->tr_pool) cudaEventDestroy(e);
  if (c->h_red) cudaFreeHost(c->h_red);
  if (c->h_seg) cudaFreeHost(c->h_seg);
  if (c->h_send) cudaFreeHost(c->h_send);
  if (c->h_recv) cudaFreeHost(c->h_recv);
  if (c->cs) {
    cudaStreamSynchronize(c->cs);
    cudaStreamDestroy(c->cs);
  }
  for (int b = 0; b < 2; ++b) {
    if (c->ev_comp[b]) cudaEventDestroy(c->ev_comp[b]);
    if (c->ev_recv[b]) cudaEventDestroy(c->ev_recv[b]);
  }
  if (c->nccl_ring && nccl_api()) nccl_api()->CommDestroy(c->nccl_ring);
  if (c->nccl && nccl_api()) nccl_api()->CommDestroy(c->nccl);
  delete c;
}

const char* accord_status_string(accord_status s) {
  switch (s) {
    case ACCORD_OK: return "ok";
    case ACCORD_E_INVALID: return "invalid argument";
    case ACCORD_E_CUDA: return "CUDA error";
    case ACCORD_E_NCCL: return "NCCL error";
    case ACCORD_E_CAPACITY: return "buffer capacity too small";
    case ACCORD_E_NUMERIC: return "non-finite value";
    case ACCORD_E_DOMAIN: return "nonpositive diagonal";
    case ACCORD_E_NOMEM: return "out of memory";
    case ACCORD_E_UNSUPPORTED: return "unsupported";
    case ACCORD_E_COMM: return "communicator callback failed";
  }
  return "unknown status";
}

const char* accord_last_error(const accord_ctx* c) {
  return c ? c->err.c_str() : g_create_err.c_str();
}

int32_t accord_abi_version(void) { return ACCORD_ABI_VERSION; }

}  // extern "C"
