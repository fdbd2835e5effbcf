// Host orchestration and C ABI of lazypca_b200.
//
// The reducers below mirror proj/core/src/reducer.cpp step for step — config
// resolution (:137-161), Omega regeneration (:128-130), sketch (:163-169),
// F formation (:216-234 Lazy, :192-214 SPCA), finish_spectral (:75-90) with
// truncated_svd_via_gram (truncated_svd.cpp:13-82), apply_map (:348-353) —
// with every numeric phase a device kernel on the context's stream and the
// row-sharded exchange (q+1 fp64 allreduces of n x l) done with NCCL.
#include <cuda_runtime.h>
#include <nccl.h>

#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <functional>
#include <memory>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "../../include/lazypca_b200.h"
#include "common.cuh"
#include "kernels.cuh"
#include "rng.cuh"

using lpca::Error;
using lpca::index_t;

namespace {

thread_local std::string g_err_msg;
thread_local std::int64_t g_err_index = -1;
thread_local double g_err_gap = 0.0;

}  // namespace

// lpca_last_error* state for the host-only translation units (mapio.cpp).
namespace {
thread_local std::unique_ptr<lpca::Error> g_callback_error;
}
void lpca::set_callback_error(const Error& e) { g_callback_error = std::make_unique<Error>(e); }
bool lpca::take_callback_error(Error* out) {
  if (!g_callback_error) return false;
  *out = *g_callback_error;
  g_callback_error.reset();
  return true;
}

void lpca::set_last_error(const std::string& msg, std::int64_t index, double gap) {
  g_err_msg = msg;
  g_err_index = index;
  g_err_gap = gap;
}

namespace {

template <typename F>
lpca_status guarded(F&& fn) {
  try {
    fn();
    return LPCA_OK;
  } catch (const Error& e) {
    g_err_msg = e.what();
    g_err_index = e.index;
    g_err_gap = e.gap;
    return static_cast<lpca_status>(e.code);
  } catch (const std::exception& e) {
    g_err_msg = e.what();
    g_err_index = -1;
    return LPCA_ERR_INTERNAL;
  }
}

// NCCL is resolved at run time, only when a context spans more than one rank:
// the process may already hold torch's bundled libnccl.so.2 (same soname,
// newer symbols), which must win over the system copy. Types come from nccl.h.
struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static bool loaded = false;
  if (loaded) return api;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h && std::getenv("LPCA_NCCL_PATH")) h = dlopen(std::getenv("LPCA_NCCL_PATH"), RTLD_NOW);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
  if (!h) throw Error(lpca::kNccl, std::string("cannot load libnccl.so.2: ") + dlerror());
  api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
  api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
  api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
  api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
  api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
  if (!api.get_unique_id || !api.comm_init_rank || !api.all_reduce || !api.comm_destroy || !api.error_string)
    throw Error(lpca::kNccl, "libnccl.so.2 lacks a required symbol");
  loaded = true;
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Error(lpca::kNccl, std::string(what) + ": " + nccl().error_string(r));
}

std::string S(index_t v) { return std::to_string(v); }

}  // namespace

struct lpca_ctx {
  int device = 0;
  int rank = 0, world = 1;
  cudaStream_t stream = nullptr;
  cudaStream_t own_stream = nullptr;
  ncclComm_t comm = nullptr;
  lpca_allreduce_fn hook = nullptr;  // caller's collective in place of NCCL
  void* hook_user = nullptr;
  int num_sms = 148;
  int gemm_path = 0;  // 0 = tcgen05 split-TF32 for fp32 data, 1 = SIMT
  int exact = 0;      // fp64 reference summation order (tests)
  std::int64_t launches = 0;
  int last_sweeps = 0;
  int eigensolver = 0;  // 0: tridiagonal route (tridiag_eigh), 1: parallel Jacobi (jacobi_eigh)
  std::unordered_map<std::string, std::pair<void*, std::size_t>> ws;
  // phase events [0, 18); power-step pass events [18, 18 + 4 * kPowerEvSteps)
  static constexpr int kPowerEvSteps = 8;
  cudaEvent_t ev[18 + 4 * kPowerEvSteps] = {};
  std::unordered_set<lpca_map*> live_maps;  // maps whose V was allocated on this context's stream
  int pass_slot = -1;  // >= 0: the next X pass records ev[pass_slot] / ev[pass_slot + 1] around its kernel
  bool force_scan = false;  // fit_dev retry: per-run scales by the full scan
  // the last transform's fp16 range flag (pinned host copy) and its scanned redo
  const int* tr_flag = nullptr;
  std::function<void()> tr_redo;

  void note_launch(int n = 1) { launches += n; }

  // Host X crossing PCIe in row chunks on copy_stream (lpca_fit,
  // lpca_fit_transform): (end row, landed event) per chunk, in order. The
  // fp16 sketch consumes the chunks as they land (xw_pass); every other reader
  // of X waits for all of them first (wait_arrivals). The transform's Y comes
  // back the same way, chunk by chunk behind the transform's launches.
  // the row-gather schedule of the last very sparse Omega (sparse_omega.cu),
  // keyed by what determines Omega; steps < 0: infeasible for that Omega
  std::string row_sched_key;
  int row_sched_steps = -1, row_sched_smax = 0, row_sched_splits = 1;
  cudaStream_t copy_stream = nullptr;
  std::vector<std::pair<index_t, cudaEvent_t>> arrivals;
  std::vector<cudaEvent_t> chunk_ev[2];  // [0] H2D chunks, [1] D2H chunks
  cudaStream_t copies() {
    if (!copy_stream) LPCA_CUDA(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking));
    return copy_stream;
  }
  cudaEvent_t chunk_event(int pool, std::size_t i) {
    auto& v = chunk_ev[pool];
    while (v.size() <= i) {
      cudaEvent_t e = nullptr;
      LPCA_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      v.push_back(e);
    }
    return v[i];
  }
  void wait_arrivals() {
    if (!arrivals.empty()) LPCA_CUDA(cudaStreamWaitEvent(stream, arrivals.back().second, 0));
    arrivals.clear();
  }

  // Pinned host block for the small device->host reads of one call (status
  // words, eigenvalues, R diagonals): cudaMemcpyAsync into pageable memory
  // would block the host at the copy, before the work queued behind it.
  char* pin = nullptr;
  std::size_t pin_used = 0;
  static constexpr std::size_t kPinBytes = 1 << 20;
  void pin_reset() { pin_used = 0; }
  template <typename T>
  T* stage_read(const T* dev, index_t count) {
    const std::size_t bytes = sizeof(T) * static_cast<std::size_t>(count > 0 ? count : 1);
    if (!pin) LPCA_CUDA(cudaMallocHost(reinterpret_cast<void**>(&pin), kPinBytes));
    const std::size_t off = (pin_used + 15) & ~std::size_t(15);
    if (off + bytes > kPinBytes) throw Error(lpca::kInternal, "pinned readback block exhausted");
    pin_used = off + bytes;
    T* h = reinterpret_cast<T*>(pin + off);
    if (count > 0) LPCA_CUDA(cudaMemcpyAsync(h, dev, sizeof(T) * count, cudaMemcpyDeviceToHost, stream));
    return h;
  }

  void* buf(const std::string& name, std::size_t bytes) {
    auto it = ws.find(name);
    if (it != ws.end() && it->second.second >= bytes) return it->second.first;
    if (it != ws.end()) {
      LPCA_CUDA(cudaStreamSynchronize(stream));
      LPCA_CUDA(cudaFree(it->second.first));
      ws.erase(it);
    }
    void* p = nullptr;
    const std::size_t guard = guards() ? kGuardBytes : 0;
    LPCA_CUDA(cudaMalloc(&p, (bytes < 256 ? 256 : bytes) + guard));
    if (std::getenv("LPCA_WS_POISON"))  // debugging aid: NaN-fill new workspaces
      LPCA_CUDA(cudaMemsetAsync(p, 0xff, bytes < 256 ? 256 : bytes, stream));
    if (guard)  // debugging aid (lpca_debug_check_guards): a pattern band right after the workspace
      LPCA_CUDA(cudaMemsetAsync(static_cast<char*>(p) + bytes, kGuardByte, guard, stream));
    ws[name] = {p, bytes};
    return p;
  }
  // LPCA_WS_GUARD=1: every workspace is followed by a guard band whose pattern
  // lpca_debug_check_guards verifies (out-of-bounds writes of any kernel into
  // the library's own buffers; compute-sanitizer is unavailable on the pool).
  static constexpr std::size_t kGuardBytes = 1 << 20;
  static constexpr int kGuardByte = 0xA5;
  static bool guards() {
    static const bool on = [] {
      const char* e = std::getenv("LPCA_WS_GUARD");
      return e && e[0] == '1';
    }();
    return on;
  }
  template <typename T>
  T* get(const std::string& name, std::size_t count) {
    return static_cast<T*>(buf(name, count * sizeof(T)));
  }
  std::size_t cached(const std::string& name) const {
    auto it = ws.find(name);
    return it == ws.end() ? 0 : it->second.second;
  }
  void release(const std::string& name) {
    auto it = ws.find(name);
    if (it == ws.end()) return;
    LPCA_CUDA(cudaStreamSynchronize(stream));
    LPCA_CUDA(cudaFree(it->second.first));
    ws.erase(it);
  }
  void allreduce(double* p, index_t count) {
    if (world <= 1 && !comm) return;  // (a one-rank communicator still runs: the NCCL path on one GPU)
    if (hook) {
      if (hook(hook_user, p, count, stream) != 0) throw Error(lpca::kNccl, "allreduce hook failed");
      return;
    }
    nccl_check(nccl().all_reduce(p, p, static_cast<std::size_t>(count), ncclDouble, ncclSum, comm, stream),
               "ncclAllReduce");
  }
  // Every rank's `k` host values: rank r's go to slots [r k, r k + k) of a zeroed
  // world x k vector summed over ranks (an allgather through the sum
  // collective). Synchronises the stream; world == 1 returns the input.
  std::vector<double> gather_host(const std::vector<double>& mine) {
    if (world <= 1) return mine;
    const std::size_t k = mine.size(), total = k * static_cast<std::size_t>(world);
    std::vector<double> all(total, 0.0);
    std::copy(mine.begin(), mine.end(), all.begin() + static_cast<std::ptrdiff_t>(k * rank));
    double* d = static_cast<double*>(buf("agree", total * sizeof(double)));
    LPCA_CUDA(cudaMemcpyAsync(d, all.data(), total * sizeof(double), cudaMemcpyHostToDevice, stream));
    allreduce(d, static_cast<index_t>(total));
    LPCA_CUDA(cudaMemcpyAsync(all.data(), d, total * sizeof(double), cudaMemcpyDeviceToHost, stream));
    LPCA_CUDA(cudaStreamSynchronize(stream));
    return all;
  }
};

struct lpca_map {
  int device = 0;
  int method = LPCA_LAZY_SPCA;
  index_t k = 0, l = 0, n = 0;
  std::uint64_t seed = 0;
  double density = 1.0, scale = 1.0;
  double* v = nullptr;  // device, n x k column-major fp64
  std::vector<double> sigma;
  float xmax = 0.0f;    // max|X| of the fitted rows (scale of the fp16 transform; 0 = unknown)
  // V comes from the stream-ordered allocator on the creating context's stream:
  // no device-wide synchronisation per fit (cudaMalloc/cudaFree would stall the
  // pipeline). A map must be destroyed before its context.
  cudaStream_t stream = nullptr;
  lpca_ctx* owner = nullptr;  // cleared if the context goes first (then V frees on the legacy stream)
  void alloc_v(lpca_ctx& c, std::size_t bytes) {
    owner = &c;
    stream = c.stream;
    c.live_maps.insert(this);
    LPCA_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&v), bytes, stream));
  }
  ~lpca_map() {
    if (owner) owner->live_maps.erase(this);
    if (v) cudaFreeAsync(v, stream);
  }
};

namespace {

using namespace lpca;

// ---- configuration (ReducerConfig::resolved, reducer.cpp:137-161;
//      ProjectionSpec::validate, projection.cpp:52-60) ----------------------
lpca_config resolve(const lpca_config& in, index_t data_cols) {
  lpca_config out = in;
  if (out.k < 1) throw Error(kInvalidArgument, "reducer: k must be at least 1, got " + S(out.k));
  if (out.l == 0) out.l = out.k;
  if (out.k > out.l)
    throw Error(kInvalidArgument,
                "reducer: k = " + S(out.k) + " exceeds sketch width l = " + S(out.l));
  if (out.method == LPCA_RP && out.k != out.l)
    throw Error(kInvalidArgument,
                "reducer: random projection reduces straight to k dimensions; l must equal k");
  if (out.block_rows > 0) out.streaming = 1;
  if (out.streaming && out.block_rows < 1)
    throw Error(kInvalidArgument, "reducer: streaming mode needs block_rows >= 1");
  if (out.proj_n == 0) out.proj_n = data_cols;
  if (out.proj_l == 0) out.proj_l = out.l;
  if (out.proj_n != data_cols)
    throw Error(kDimension, "reducer: projection is built for n = " + S(out.proj_n) +
                                " but the data has " + S(data_cols) + " columns");
  if (out.proj_l != out.l)
    throw Error(kDimension, "reducer: projection width " + S(out.proj_l) +
                                " does not match l = " + S(out.l));
  if (out.proj_l < 2)
    throw Error(kInvalidArgument,
                "projection: sketch width l must be at least 2, got " + S(out.proj_l));
  if (out.proj_l > out.proj_n)
    throw Error(kInvalidArgument, "projection: sketch width l = " + S(out.proj_l) +
                                      " exceeds data dimensionality n = " + S(out.proj_n));
  if (!(out.density > 0.0) || out.density > 1.0)
    throw Error(kInvalidArgument,
                "projection: density must lie in (0, 1], got " + std::to_string(out.density));
  if (out.power_iters < 0) throw Error(kInvalidArgument, "reducer: power_iters must be >= 0");
  if (out.method != LPCA_RP && out.method != LPCA_SPCA && out.method != LPCA_LAZY_SPCA)
    throw Error(kInvalidArgument, "unknown method");
  return out;
}

double projection_scale(const lpca_config& c) {
  return c.projection_kind == LPCA_GAUSSIAN ? std::sqrt(static_cast<double>(c.proj_l))
                                            : std::sqrt(static_cast<double>(c.proj_l) * c.density);
}

void check_ctx(lpca_ctx* ctx) {
  if (!ctx) throw Error(kInvalidArgument, "null context");
  LPCA_CUDA(cudaSetDevice(ctx->device));
  ctx->pin_reset();  // every entry point starts with an empty readback block
}

// ---- device-resident X ------------------------------------------------------
struct DevX {
  const void* p = nullptr;
  int dtype = 8;
  index_t m = 0, n = 0, ld = 0;
  // sparse path (csrc/sparse.cu): X as CSR (row gathers) and CSC (column
  // gathers) on the device, fp64 values, 32-bit indices; p is null
  const std::int64_t* rp = nullptr;
  const std::int32_t* ci = nullptr;
  const double* rv = nullptr;
  const std::int64_t* cp = nullptr;
  const std::int32_t* ri = nullptr;
  const double* cv = nullptr;
  index_t nnz = 0;
  bool sparse() const { return rp != nullptr; }
};

// CSC inputs stay sparse on the device below this density (LPCA_SPARSE=1/0
// forces the choice); denser ones are densified for the tensor-core passes.
bool keep_sparse(index_t nnz, index_t m, index_t n) {
  const char* e = std::getenv("LPCA_SPARSE");
  if (e && e[0]) return e[0] == '1';
  return static_cast<double>(nnz) < 0.25 * static_cast<double>(m) * static_cast<double>(n) &&
         m < (index_t(1) << 31) && n < (index_t(1) << 31);
}

std::size_t dsize(int dtype) { return dtype == 4 ? 4 : 8; }

void check_view(const lpca_matrix_view* x) {
  if (!x) throw Error(kInvalidArgument, "null matrix view");
  if (x->dtype != LPCA_F32 && x->dtype != LPCA_F64)
    throw Error(kInvalidArgument, "matrix view: dtype must be LPCA_F32 or LPCA_F64");
  if (x->rows < 0 || x->cols < 0)
    throw Error(kInvalidArgument, "sparse matrix dimensions must be non-negative");
  if (x->layout == LPCA_CSC) {
    if (x->location != LPCA_HOST) throw Error(kInvalidArgument, "CSC views must be host memory");
    if (!x->col_ptr || (x->nnz > 0 && (!x->row_idx || !x->data)))
      throw Error(kInvalidArgument, "CSC view: missing arrays");
  } else if (x->layout != LPCA_ROW_MAJOR && x->layout != LPCA_COL_MAJOR) {
    throw Error(kInvalidArgument, "matrix view: unknown layout");
  } else if (!x->data && x->rows * x->cols > 0) {
    throw Error(kInvalidArgument, "matrix view: null data");
  } else if (x->ld != 0 && x->rows * x->cols > 0) {
    const index_t inner = x->layout == LPCA_ROW_MAJOR ? x->cols : x->rows;
    if (x->ld < inner)
      throw Error(kInvalidArgument, "matrix view: ld = " + S(x->ld) + " is smaller than the " +
                                        (x->layout == LPCA_ROW_MAJOR ? "row" : "column") + " length " + S(inner));
  }
}

// A CSC view staged on the device (csrc/sparse.cu): col_ptr, row_idx and the
// values cross PCIe as the caller holds them; the entries are checked and the
// indices narrowed by a kernel, then either the CSR copy is built (the sparse
// path) or X is densified into a row-major matrix of its own dtype (denser
// inputs, for the tensor-core passes). Errors are the host loop's, in its
// order: the first column whose col_ptr decreases is found here, and an entry
// error in an earlier column wins over it (the device checks exactly those
// columns).
// Returns false (nothing staged) when the device scratch (~24 B per entry)
// does not fit the free memory: the host path below then does the same work.
bool stage_csc_device(lpca_ctx& ctx, const lpca_matrix_view* x, const char* slot, double* h2d_bytes,
                      bool densify, DevX& out) {
  const index_t m = x->rows, n = x->cols, nnz = x->nnz;
  const std::size_t es = dsize(x->dtype), nz = static_cast<std::size_t>(nnz > 0 ? nnz : 1);
  // the first column whose col_ptr decreases (or runs past nnz, which a later
  // column must then undo: the entries before it stay inside the arrays)
  index_t bad_col = -1;
  for (index_t j = 0; j < n && bad_col < 0; ++j)
    if (x->col_ptr[j + 1] < x->col_ptr[j] || x->col_ptr[j + 1] > nnz) bad_col = j;
  const index_t ncheck = bad_col >= 0 ? bad_col : n;
  const std::string sl(slot);
  auto* cp = ctx.get<std::int64_t>(sl + ".cp", n + 1);
  auto* ri = ctx.get<std::int32_t>(sl + ".ri", nz);
  auto* cv = ctx.get<double>(sl + ".cv", nz);
  auto* first = ctx.get<unsigned long long>(sl + ".first", 1);
  // scratch (one cached workspace, reused by later calls of the same shape):
  // the caller's 64-bit rows and values, each entry's column, the sorts' keys,
  // the row counts, CUB's temp. (A stream-ordered allocation
  // returned its tens of GB to the driver at every call: 2-6 s of remapping.)
  const index_t nin = bad_col >= 0 ? x->col_ptr[bad_col] : nnz;  // entries of the checked columns
  const std::size_t tb = densify ? 0 : csc_stage_temp_bytes(m, nnz);
  auto a16 = [](std::size_t b) { return (b + 15) & ~std::size_t(15); };
  const std::size_t off_v = a16(nz * 8), off_c = off_v + a16(nz * es), off_k = off_c + a16(nz * 4),
                    off_n = off_k + a16(nz * 4), off_t = off_n + a16(8 * static_cast<std::size_t>(m + 1)),
                    total = densify ? off_k : off_t + tb;  // densify: the caller's arrays and colof only
  if (ctx.cached(sl + ".stage") < total) {
    ctx.release(sl + ".stage");
    std::size_t free_b = 0, total_b = 0;
    LPCA_CUDA(cudaMemGetInfo(&free_b, &total_b));
    const std::size_t outputs = densify ? dsize(x->dtype) * static_cast<std::size_t>(m) * static_cast<std::size_t>(n)
                                        : nz * 12 + 8 * static_cast<std::size_t>(m + 1);
    if (total + outputs + (std::size_t(1) << 30) > free_b) return false;
  }
  char* tmp = ctx.get<char>(sl + ".stage", total);
  auto* ri64 = reinterpret_cast<std::int64_t*>(tmp);
  void* vin = tmp + off_v;
  auto* colof = reinterpret_cast<std::int32_t*>(tmp + off_c);
  auto* keys = reinterpret_cast<std::int32_t*>(tmp + off_k);
  auto* cnt = reinterpret_cast<std::int64_t*>(tmp + off_n);
  LPCA_CUDA(cudaMemcpyAsync(cp, x->col_ptr, sizeof(std::int64_t) * (n + 1), cudaMemcpyHostToDevice, ctx.stream));
  if (nin > 0) {
    LPCA_CUDA(cudaMemcpyAsync(ri64, x->row_idx, sizeof(std::int64_t) * nin, cudaMemcpyHostToDevice, ctx.stream));
    LPCA_CUDA(cudaMemcpyAsync(vin, x->data, es * nin, cudaMemcpyHostToDevice, ctx.stream));
  }
  launch_csc_check(ctx.stream, ncheck, m, cp, ri64, vin, x->dtype, ri, colof, cv, first);
  LPCA_LAUNCHED(ctx);
  const unsigned long long* fh = ctx.stage_read(first, 1);
  LPCA_CUDA(cudaStreamSynchronize(ctx.stream));
  if (*fh != ~0ull || bad_col >= 0) {
    if (*fh == ~0ull) throw Error(kInvalidArgument, "csc: col_ptr must be non-decreasing");
    const index_t p = static_cast<index_t>(*fh / 4);
    const int code = static_cast<int>(*fh % 4);
    const index_t j = static_cast<index_t>(std::upper_bound(x->col_ptr, x->col_ptr + ncheck + 1, p) - x->col_ptr) - 1;
    if (code == 0) throw Error(kDimension, "csc: row index out of range in column " + S(j));
    if (code == 1) throw Error(kInvalidArgument, "csc: row indices must be strictly increasing in column " + S(j));
    if (code == 2) throw Error(kInvalidArgument, "csc: explicit zero stored in column " + S(j));
    throw Error(kInvalidArgument, "csc: non-finite value in column " + S(j));
  }
  if (h2d_bytes) *h2d_bytes += static_cast<double>(nnz) * static_cast<double>(8 + es) + static_cast<double>(n + 1) * 8;
  // the scratch stays cached for the next call unless memory is tight
  auto keep_or_release_scratch = [&]() {
    std::size_t free_b = 0, total_b = 0;
    LPCA_CUDA(cudaMemGetInfo(&free_b, &total_b));
    if (free_b < total_b / 4) ctx.release(sl + ".stage");
  };
  if (densify) {
    DevX d;
    d.m = m;
    d.n = n;
    d.dtype = x->dtype;
    void* dst = ctx.buf(slot, es * m * n);
    launch_zero(ctx.stream, dst, es * m * n);
    launch_csc_to_dense(ctx.stream, m, n, cp, ri64, cv, d.dtype, dst, n);
    LPCA_LAUNCHED(ctx);
    d.p = dst;
    d.ld = n;
    keep_or_release_scratch();
    out = d;
    return true;
  }
  auto* rp = ctx.get<std::int64_t>(sl + ".rp", m + 1);
  auto* ci = ctx.get<std::int32_t>(sl + ".ci", nz);
  auto* rv = ctx.get<double>(sl + ".rv", nz);
  launch_csr_from_csc(ctx.stream, m, nnz, ri, colof, cv, rp, ci, rv, cnt, keys, tmp + off_t, tb);
  ctx.note_launch(1);  // row counts (+ CUB's scan and two radix sorts)
  LPCA_CUDA(cudaGetLastError());
  keep_or_release_scratch();
  DevX d;
  d.m = m;
  d.n = n;
  d.dtype = 8;
  d.ld = n;
  d.rp = rp;
  d.ci = ci;
  d.rv = rv;
  d.cp = cp;
  d.ri = ri;
  d.cv = cv;
  d.nnz = nnz;
  out = d;
  return true;
}

// Brings any view to a row-major device matrix of its own dtype. Host data is
// copied with one cudaMemcpyAsync per contiguous range; a column-major or CSC
// view is transposed / densified by a kernel after upload.
DevX stage_x(lpca_ctx& ctx, const lpca_matrix_view* x, const char* slot, double* h2d_bytes) {
  check_view(x);
  DevX d;
  d.m = x->rows;
  d.n = x->cols;
  d.dtype = x->dtype;
  const std::size_t es = dsize(x->dtype);
  if (d.m == 0 || d.n == 0) {
    d.p = ctx.buf(slot, es);
    d.ld = d.n > 0 ? d.n : 1;
    return d;
  }
  if (x->layout == LPCA_CSC) {
    const index_t nnz = x->nnz;
    // canonical-form checks of SparseMatrix::from_csc (sparse_matrix.cpp:50-80)
    if (x->col_ptr[0] != 0) throw Error(kInvalidArgument, "csc: col_ptr[0] must be 0");
    if (x->col_ptr[x->cols] != nnz) throw Error(kDimension, "csc: col_ptr[cols] must equal nnz");
    DevX dd;
    const char* host_env = std::getenv("LPCA_CSC_HOST");  // tests: force the host staging below
    if (nnz < (index_t(1) << 31) && !(host_env && host_env[0] == '1') &&
        stage_csc_device(ctx, x, slot, h2d_bytes, !keep_sparse(nnz, x->rows, x->cols), dd))
      return dd;
    std::vector<double> vals(static_cast<std::size_t>(nnz));
    for (index_t j = 0; j < x->cols; ++j) {
      const index_t lo = x->col_ptr[j], hi = x->col_ptr[j + 1];
      // (hi > nnz: a later column must decrease; stop before reading past the arrays)
      if (hi < lo || hi > nnz) throw Error(kInvalidArgument, "csc: col_ptr must be non-decreasing");
      for (index_t p = lo; p < hi; ++p) {
        const index_t r = x->row_idx[p];
        if (r < 0 || r >= x->rows)
          throw Error(kDimension, "csc: row index out of range in column " + S(j));
        if (p > lo && r <= x->row_idx[p - 1])
          throw Error(kInvalidArgument, "csc: row indices must be strictly increasing in column " + S(j));
        const double v = x->dtype == 4 ? static_cast<const float*>(x->data)[p]
                                       : static_cast<const double*>(x->data)[p];
        if (v == 0.0) throw Error(kInvalidArgument, "csc: explicit zero stored in column " + S(j));
        if (!std::isfinite(v)) throw Error(kInvalidArgument, "csc: non-finite value in column " + S(j));
        vals[static_cast<std::size_t>(p)] = v;
      }
    }
    if (keep_sparse(nnz, x->rows, x->cols)) {
      // CSR by a stable counting sort of the CSC entries: within a row the
      // columns stay ascending (the reference's accumulation order)
      const index_t m = x->rows, n = x->cols;
      std::vector<std::int64_t> rptr(static_cast<std::size_t>(m + 1), 0);
      for (index_t p = 0; p < nnz; ++p) ++rptr[static_cast<std::size_t>(x->row_idx[p] + 1)];
      for (index_t i = 0; i < m; ++i) rptr[static_cast<std::size_t>(i + 1)] += rptr[static_cast<std::size_t>(i)];
      std::vector<std::int64_t> fill(rptr.begin(), rptr.end() - 1);
      std::vector<std::int32_t> ccol(static_cast<std::size_t>(nnz)), crow(static_cast<std::size_t>(nnz));
      std::vector<double> cval(static_cast<std::size_t>(nnz));
      for (index_t j = 0; j < n; ++j)
        for (index_t p = x->col_ptr[j]; p < x->col_ptr[j + 1]; ++p) {
          const index_t r = x->row_idx[p];
          const std::int64_t q = fill[static_cast<std::size_t>(r)]++;
          ccol[static_cast<std::size_t>(q)] = static_cast<std::int32_t>(j);
          cval[static_cast<std::size_t>(q)] = vals[static_cast<std::size_t>(p)];
          crow[static_cast<std::size_t>(p)] = static_cast<std::int32_t>(r);
        }
      const std::string sl(slot);
      const std::size_t nz = static_cast<std::size_t>(nnz > 0 ? nnz : 1);
      auto* rp = ctx.get<std::int64_t>(sl + ".rp", m + 1);
      auto* ci = ctx.get<std::int32_t>(sl + ".ci", nz);
      auto* rv = ctx.get<double>(sl + ".rv", nz);
      auto* cp = ctx.get<std::int64_t>(sl + ".cp", n + 1);
      auto* ri = ctx.get<std::int32_t>(sl + ".ri", nz);
      auto* cv = ctx.get<double>(sl + ".cv", nz);
      LPCA_CUDA(cudaMemcpyAsync(rp, rptr.data(), sizeof(std::int64_t) * (m + 1), cudaMemcpyHostToDevice, ctx.stream));
      LPCA_CUDA(cudaMemcpyAsync(cp, x->col_ptr, sizeof(std::int64_t) * (n + 1), cudaMemcpyHostToDevice, ctx.stream));
      if (nnz > 0) {
        LPCA_CUDA(cudaMemcpyAsync(ci, ccol.data(), sizeof(std::int32_t) * nnz, cudaMemcpyHostToDevice, ctx.stream));
        LPCA_CUDA(cudaMemcpyAsync(rv, cval.data(), sizeof(double) * nnz, cudaMemcpyHostToDevice, ctx.stream));
        LPCA_CUDA(cudaMemcpyAsync(ri, crow.data(), sizeof(std::int32_t) * nnz, cudaMemcpyHostToDevice, ctx.stream));
        LPCA_CUDA(cudaMemcpyAsync(cv, vals.data(), sizeof(double) * nnz, cudaMemcpyHostToDevice, ctx.stream));
      }
      LPCA_CUDA(cudaStreamSynchronize(ctx.stream));  // the host vectors die here
      if (h2d_bytes) *h2d_bytes += static_cast<double>(nnz * 24 + (m + n + 2) * 8);
      d.dtype = 8;
      d.ld = n;
      d.rp = rp;
      d.ci = ci;
      d.rv = rv;
      d.cp = cp;
      d.ri = ri;
      d.cv = cv;
      d.nnz = nnz;
      return d;
    }
    auto* cp = ctx.get<std::int64_t>(std::string(slot) + ".ptr", x->cols + 1);
    auto* ri = ctx.get<std::int64_t>(std::string(slot) + ".idx", nnz > 0 ? nnz : 1);
    auto* vv = ctx.get<double>(std::string(slot) + ".val", nnz > 0 ? nnz : 1);
    LPCA_CUDA(cudaMemcpyAsync(cp, x->col_ptr, sizeof(std::int64_t) * (x->cols + 1),
                              cudaMemcpyHostToDevice, ctx.stream));
    if (nnz > 0) {
      LPCA_CUDA(cudaMemcpyAsync(ri, x->row_idx, sizeof(std::int64_t) * nnz, cudaMemcpyHostToDevice, ctx.stream));
      LPCA_CUDA(cudaMemcpyAsync(vv, vals.data(), sizeof(double) * nnz, cudaMemcpyHostToDevice, ctx.stream));
    }
    void* dst = ctx.buf(slot, es * d.m * d.n);
    launch_zero(ctx.stream, dst, es * d.m * d.n);
    launch_csc_to_dense(ctx.stream, d.m, d.n, cp, ri, vv, d.dtype, dst, d.n);
    LPCA_LAUNCHED(ctx);
    // the staged host vectors must outlive the async copies
    LPCA_CUDA(cudaStreamSynchronize(ctx.stream));
    if (h2d_bytes) *h2d_bytes += static_cast<double>(nnz * (8 + 8) + (x->cols + 1) * 8);
    d.p = dst;
    d.ld = d.n;
    return d;
  }
  const bool row = x->layout == LPCA_ROW_MAJOR;
  const index_t ld = x->ld > 0 ? x->ld : (row ? x->cols : x->rows);
  if (x->location == LPCA_DEVICE && row) {
    d.p = x->data;
    d.ld = ld;
    return d;
  }
  const void* src_dev = x->data;
  index_t src_ld = ld;
  if (x->location == LPCA_HOST) {
    const index_t outer = row ? x->rows : x->cols, inner = row ? x->cols : x->rows;
    void* dst = ctx.buf(row ? std::string(slot) : std::string(slot) + ".cm", es * outer * inner);
    LPCA_CUDA(cudaMemcpy2DAsync(dst, es * inner, x->data, es * ld, es * inner, outer,
                                cudaMemcpyHostToDevice, ctx.stream));
    if (h2d_bytes) *h2d_bytes += static_cast<double>(es * outer * inner);
    if (row) {
      d.p = dst;
      d.ld = inner;
      return d;
    }
    src_dev = dst;
    src_ld = inner;
  }
  void* dst = ctx.buf(slot, es * d.m * d.n);
  launch_transpose(ctx.stream, d.dtype, src_dev, src_ld, d.m, d.n, dst, d.n);
  LPCA_LAUNCHED(ctx);
  d.p = dst;
  d.ld = d.n;
  return d;
}

// Rows per PCIe chunk of a host X (about 1 GiB, a multiple of the U^T scale
// block so every chunk starts a new block), or 0: one copy (LPCA_H2D_CHUNKS=0,
// or fewer than two chunks' worth of rows).
// (LPCA_H2D_CHUNKS and LPCA_H2D_CHUNK_MB are read per call: tests switch them)
bool copy_chunks_enabled() {
  const char* e = std::getenv("LPCA_H2D_CHUNKS");
  return !(e && e[0] == '0');
}

index_t h2d_chunk_rows(index_t rows, index_t row_bytes) {
  if (!copy_chunks_enabled() || row_bytes <= 0) return 0;
  const char* mb = std::getenv("LPCA_H2D_CHUNK_MB");
  const index_t bytes = (mb && std::atoll(mb) > 0 ? std::atoll(mb) : 1024) << 20;
  index_t r = bytes / row_bytes / kUScaleRows * kUScaleRows;
  if (r < kUScaleRows) r = kUScaleRows;
  return rows >= 2 * r ? r : 0;
}

// Rows per chunk of a transform whose Y goes to the host: 16 chunks on
// whole U^T-scale-sized blocks, or 0 (one copy) for small m.
index_t d2h_chunk_rows(index_t rows) {
  if (!copy_chunks_enabled()) return 0;  // LPCA_H2D_CHUNKS=0
  const index_t r = round_up(ceil_div(rows, index_t(16)), kUScaleRows);
  return rows >= 4 * r && rows >= 16 * kUScaleRows ? r : 0;
}

// stage_x for the fits: a host row-major X of at least two chunks crosses PCIe
// in chunks on the copy stream (after `start`, recorded on the compute stream
// once the buffer's previous readers are queued), each chunk's landing in
// ctx.arrivals and the last one also in `done`. Other inputs: stage_x.
DevX stage_x_arriving(lpca_ctx& ctx, const lpca_matrix_view* x, const char* slot, double* h2d_bytes,
                      cudaEvent_t start, cudaEvent_t done) {
  if (x && x->layout == LPCA_ROW_MAJOR && x->location == LPCA_HOST && x->rows > 0 && x->cols > 0) {
    check_view(x);
    const std::size_t es = dsize(x->dtype);
    const index_t chunk = h2d_chunk_rows(x->rows, static_cast<index_t>(es) * x->cols);
    if (chunk > 0) {
      DevX d;
      d.m = x->rows;
      d.n = x->cols;
      d.dtype = x->dtype;
      d.ld = x->cols;
      const index_t ld = x->ld > 0 ? x->ld : x->cols;
      void* dst = ctx.buf(slot, es * d.m * d.n);
      cudaStream_t cs = ctx.copies();
      LPCA_CUDA(cudaStreamWaitEvent(cs, start, 0));
      ctx.arrivals.clear();
      std::size_t i = 0;
      for (index_t r0 = 0; r0 < d.m; r0 += chunk, ++i) {
        const index_t r1 = r0 + chunk < d.m ? r0 + chunk : d.m;
        LPCA_CUDA(cudaMemcpy2DAsync(static_cast<char*>(dst) + es * r0 * d.n, es * d.n,
                                    static_cast<const char*>(x->data) + es * r0 * ld, es * ld, es * d.n, r1 - r0,
                                    cudaMemcpyHostToDevice, cs));
        // the last chunk's event is `done` itself: whoever waits for all of X
        // has also waited for the event the h2d timing reads
        const cudaEvent_t e = r1 == d.m ? done : ctx.chunk_event(0, i);
        LPCA_CUDA(cudaEventRecord(e, cs));
        ctx.arrivals.emplace_back(r1, e);
      }
      if (h2d_bytes) *h2d_bytes += static_cast<double>(es * d.m * d.n);
      d.p = dst;
      return d;
    }
  }
  DevX d = stage_x(ctx, x, slot, h2d_bytes);
  LPCA_CUDA(cudaEventRecord(done, ctx.stream));
  return d;
}

// Ends a fit's use of the copy stream: nothing still waits on a chunk, and no
// copy still reads the caller's host buffers when the call returns (also on
// the error paths).
struct CopyScope {
  lpca_ctx& ctx;
  explicit CopyScope(lpca_ctx& c) : ctx(c) {}
  ~CopyScope() {
    ctx.arrivals.clear();
    if (ctx.copy_stream) cudaStreamSynchronize(ctx.copy_stream);
  }
};

// ---- GEMM dispatch ------------------------------------------------------------
// Which engine runs an fp32 X-pass: tcgen05 split-TF32 when the path is
// selected and the shape is supported, SIMT FFMA otherwise (fp64: DFMA).
bool use_tc(const lpca_ctx& ctx, const DevX& x, index_t w) {
  return ctx.gemm_path == 0 && x.dtype == 4 && tc_xw_supported(x.n, round_up(w, 16)) &&
         x.ld % 4 == 0 && tc_utx_supported(w, x.n);
}

// A sketch-shaped operand (m x l): the plain row-major matrix (dtype of X, ld
// `ld`) and, on the tensor-core path, the tf32 hi/lo planes of its transpose
// (round_up(l,16) rows of length m, ld `ldt`) — the K-major A operand of U^T X.
struct Panel {
  void* plain = nullptr;
  float* hi = nullptr;
  float* lo = nullptr;
  index_t ld = 0;
  index_t ldt = 0;
  // pair fp16 path: U^T as fp16 hi/lo planes [ld][ldt16] scaled per (column,
  // kUScaleRows-row block), inverse scales uinv[block][ld] (tc_pair.cuh)
  __half* h16hi = nullptr;
  __half* h16lo = nullptr;
  float* uinv = nullptr;
  index_t ldt16 = 0;
};

// fp16 operand encoding of the X passes (tc_pair.cuh): the first pass over X
// (tf32) records max|X| on the device; later passes scale X by it. A transform
// gets the fitted data's max by value and re-checks the data it actually reads.
struct XScale {
  uint32_t* dev = nullptr;    // max|X| bits on the device
  float host = 0.0f;          // or by value (dev null)
  bool record = false;        // tf32 pass that records max|X| into dev
  bool use = false;           // fp16 pass
  uint32_t* check = nullptr;  // fp16 X W: max|X| of the rows read
  int* ovf = nullptr;         // scanless per-run scales: flags runs that need the scan
};

// Very sparse Omega on dense X: 0 = always the dense passes, 1 = always a
// gather sketch (fp32: the row gather when its schedule fits), default: the
// row gather for fp32 rows longer than 8192 (configs[3]: 3.9 vs 5.4 ms per
// 200k rows unthrottled, 58-61 vs 71-73 ms at full size power-capped; shorter
// rows pay its per-row overhead: n = 4096, l = 110 at 400k rows 4.7 vs 1.2 ms
// for the HBM-bound dense pass) and off the tcgen05 path; the chunk gather
// for fp64 X and the SIMT path otherwise.
int sparse_omega_mode() {  // read per fit (tests switch it)
  const char* e = getenv("LPCA_SPARSE_OMEGA");
  return e && e[0] == '0' ? 0 : (e && e[0] == '1' ? 1 : 2);
}

bool f16_enabled() {
  static const bool on = [] {
    const char* e = getenv("LPCA_TC_F16");
    return !(e && e[0] == '0');
  }();
  return on;
}

// LPCA_BLO_SKIP=0 keeps the a_hi w_lo MMAs when W is exact in fp16 (A/B)
bool blo_skip_enabled() {
  static const bool on = [] {
    const char* e = getenv("LPCA_BLO_SKIP");
    return !(e && e[0] == '0');
  }();
  return on;
}

index_t planes_ld(index_t m) { return round_up(m > 0 ? m : 1, 4); }

// Brackets the X-pass kernel itself (not its operand preparation) with the
// context's pass events, for the per-kernel times in lpca_timings.
void pass_mark(lpca_ctx& ctx, int which) {
  if (ctx.pass_slot >= 0) LPCA_CUDA(cudaEventRecord(ctx.ev[ctx.pass_slot + which], ctx.stream));
}

// out = X W, W fp64 column-major (n x wc, ld ldw). For fp32 X the operand is
// prepared once per call (rounded to fp32, or split into tf32 hi/lo planes).
void xw_pass(lpca_ctx& ctx, const DevX& x, const double* w, index_t wc, index_t ldw, const Panel& out,
             bool exact, const XScale* xs = nullptr) {
  const index_t m = x.m, n = x.n;
  // only the 2-SM pass takes X chunk by chunk as it lands (ctx.arrivals)
  const bool pair = !x.sparse() && x.dtype == 4 && use_tc(ctx, x, wc) && tc_pair_mode();
  if (!pair) ctx.wait_arrivals();
  if (m == 0) return;
  if (x.sparse()) {  // row gathers over CSR in the reference's order (kernels.cpp:30-47)
    double* wt = ctx.get<double>("w.rows", n * wc);
    launch_transpose(ctx.stream, 8, w, ldw, n, wc, wt, wc);
    LPCA_LAUNCHED(ctx);
    pass_mark(ctx, 0);
    launch_spmm_csr(ctx.stream, m, x.rp, x.ci, x.rv, wt, wc, wc, out.plain, 8, out.ld, 1);
    LPCA_LAUNCHED(ctx);
    pass_mark(ctx, 1);
    return;
  }
  if (x.dtype == 8) {
    pass_mark(ctx, 0);
    launch_xw_simt<double, double>(ctx.stream, static_cast<const double*>(x.p), m, n, x.ld, w, wc,
                                   ldw, static_cast<double*>(out.plain), out.ld, 1, exact);
    LPCA_LAUNCHED(ctx);
    pass_mark(ctx, 1);
    return;
  }
  if (use_tc(ctx, x, wc) && tc_pair_mode()) {
    XwPairArgs p;
    p.x = static_cast<const float*>(x.p);
    p.m = m;
    p.n = n;
    p.ldx = x.ld;
    p.wpad = round_up(wc, 16);
    if (xs && xs->use) {
      p.ldw = round_up(n, 8);
      __half* hi = ctx.get<__half>("w.h16hi", p.wpad * p.ldw);
      __half* lo = ctx.get<__half>("w.h16lo", p.wpad * p.ldw);
      float* winv = ctx.get<float>("w.inv", p.wpad);
      int* lo_nz = blo_skip_enabled() ? ctx.get<int>("w.lonz", 1) : nullptr;
      launch_split_f16_w(ctx.stream, w, ldw, n, wc, p.wpad, hi, lo, p.ldw, winv, lo_nz);
      LPCA_LAUNCHED(ctx);
      p.wlo_nz = lo_nz;
      if (lo_nz && std::getenv("LPCA_VERBOSE")) {
        int h = -1;
        LPCA_CUDA(cudaMemcpyAsync(&h, lo_nz, sizeof(int), cudaMemcpyDeviceToHost, ctx.stream));
        LPCA_CUDA(cudaStreamSynchronize(ctx.stream));
        std::fprintf(stderr, "lazypca_b200: x w pass n=%lld wc=%d w lo plane %s\n", (long long)n, (int)wc,
                     h ? "nonzero" : "zero (a_hi w_lo MMAs skipped)");
      }
      p.half = true;
      p.w_hi = hi;
      p.w_lo = lo;
      p.winv = winv;
      p.xmax_in = xs->dev;
      p.xmax_val = xs->host;
      p.xmax_out = xs->check;
      p.ovf = xs->ovf;
    } else {
      p.ldw = round_up(n, 4);
      float* hi = ctx.get<float>("w.hi", p.wpad * p.ldw);
      float* lo = ctx.get<float>("w.lo", p.wpad * p.ldw);
      launch_split_tf32_w(ctx.stream, w, ldw, n, wc, p.wpad, hi, lo, p.ldw);
      LPCA_LAUNCHED(ctx);
      p.w_hi = hi;
      p.w_lo = lo;
      p.xmax_out = xs && xs->record ? xs->dev : nullptr;
    }
    p.out = static_cast<float*>(out.plain);
    p.ldo = out.ld;
    p.wstore = wc;
    if (out.h16hi) {
      p.uh = out.h16hi;
      p.ul = out.h16lo;
      p.uinv = out.uinv;
      p.ldh = out.ldt16;
    } else {
      p.out_hi = out.hi;
      p.out_lo = out.lo;
      p.ldh = out.ldt;
    }
    if (ctx.pass_slot >= 0) {  // the launcher records them around the kernel itself
      p.ev_pre = ctx.ev[ctx.pass_slot];
      p.ev_post = ctx.ev[ctx.pass_slot + 1];
    }
    if (ctx.arrivals.empty()) {
      launch_xw_pair(ctx.stream, p, ctx.num_sms);
      LPCA_LAUNCHED(ctx);
      return;
    }
    // X still crossing PCIe: one launch per landed chunk (chunks start on
    // U^T scale blocks, so each launch owns whole blocks of the planes)
    const auto chunks = std::move(ctx.arrivals);
    ctx.arrivals.clear();
    if (chunks.back().first != m) throw Error(kInternal, "xw_pass: arriving chunks do not cover X");
    index_t r0 = 0;
    for (std::size_t i = 0; i < chunks.size(); ++i) {
      const index_t r1 = chunks[i].first;
      if (r0 % kUScaleRows) throw Error(kInternal, "xw_pass: chunk not on a scale block");
      LPCA_CUDA(cudaStreamWaitEvent(ctx.stream, chunks[i].second, 0));
      XwPairArgs q = p;
      q.x = p.x + r0 * p.ldx;
      q.m = r1 - r0;
      if (q.out) q.out += r0 * p.ldo;
      if (q.uh) {
        q.uh += r0;
        q.ul += r0;
        q.uinv += (r0 / kUScaleRows) * p.wpad;
      }
      if (q.out_hi) {
        q.out_hi += r0;
        q.out_lo += r0;
      }
      q.ev_pre = i == 0 ? p.ev_pre : nullptr;
      q.ev_post = i + 1 == chunks.size() ? p.ev_post : nullptr;
      launch_xw_pair(ctx.stream, q, ctx.num_sms);
      LPCA_LAUNCHED(ctx);
      r0 = r1;
    }
    return;
  }
  if (use_tc(ctx, x, wc)) {
    const index_t wpad = round_up(wc, 16);
    float* hi = ctx.get<float>("w.hi", wpad * n);
    float* lo = ctx.get<float>("w.lo", wpad * n);
    launch_split_tf32_w(ctx.stream, w, ldw, n, wc, wpad, hi, lo, n);
    LPCA_LAUNCHED(ctx);
    pass_mark(ctx, 0);
    launch_xw_tc_planes(ctx.stream, static_cast<const float*>(x.p), m, n, x.ld, hi, lo, wpad, n,
                        static_cast<float*>(out.plain), out.ld, wc, out.hi, out.lo, out.ldt,
                        ctx.num_sms);
    LPCA_LAUNCHED(ctx);
    pass_mark(ctx, 1);
    return;
  }
  float* w32 = ctx.get<float>("w.f32", wc * n);
  launch_convert_f64_to_f32(ctx.stream, w, ldw, w32, n, n, wc, 1.0);
  LPCA_LAUNCHED(ctx);
  pass_mark(ctx, 0);
  launch_xw_simt<float, float>(ctx.stream, static_cast<const float*>(x.p), m, n, x.ld, w32, wc, n,
                               static_cast<float*>(out.plain), out.ld, 1, false);
  LPCA_LAUNCHED(ctx);
  pass_mark(ctx, 1);
}

index_t pick_chunks(const lpca_ctx& ctx, index_t m, index_t tiles, bool exact) {
  if (exact || m <= 0) return 1;
  index_t chunks = ceil_div(4 * ctx.num_sms, tiles > 0 ? tiles : 1);
  const index_t max_chunks = ceil_div(m, 2048);
  if (chunks > max_chunks) chunks = max_chunks;
  if (chunks < 1) chunks = 1;
  return chunks;
}

// F (l x n column-major fp64) = U^T X summed over this rank's rows, then
// allreduced over ranks.
void utx_pass(lpca_ctx& ctx, const DevX& x, const Panel& u, index_t l, double* f, bool exact,
              const XScale* xs = nullptr, bool over_ranks = true) {
  const index_t m = x.m, n = x.n;
  if (m == 0) {
    launch_zero(ctx.stream, f, sizeof(double) * l * n);
    if (over_ranks) ctx.allreduce(f, l * n);
    return;
  }
  index_t chunks;
  double* part;
  if (x.sparse()) {  // column gathers over CSC in the reference's order (kernels.cpp:70-113)
    pass_mark(ctx, 0);
    launch_gemm_t_csc(ctx.stream, n, x.cp, x.ri, x.cv, static_cast<const double*>(u.plain), u.ld, l, f, false);
    LPCA_LAUNCHED(ctx);
    pass_mark(ctx, 1);
    if (over_ranks) ctx.allreduce(f, l * n);
    return;
  }
  if (u.h16hi && x.dtype == 4) {
    index_t rps = 0;
    chunks = utx_pair_splits(m, n, ctx.num_sms, &rps);
    part = chunks == 1 ? f : ctx.get<double>("f.part", chunks * l * n);
    UtxPairArgs p;
    p.half = true;
    p.u_hi = u.h16hi;
    p.u_lo = u.h16lo;
    p.ldt = u.ldt16;
    p.uinv = u.uinv;
    p.xmax_in = xs ? xs->dev : nullptr;
    p.x = static_cast<const float*>(x.p);
    p.ldx = x.ld;
    p.m = m;
    p.l = l;
    p.n = n;
    p.part = part;
    if (ctx.pass_slot >= 0) {
      p.ev_pre = ctx.ev[ctx.pass_slot];
      p.ev_post = ctx.ev[ctx.pass_slot + 1];
    }
    launch_utx_pair(ctx.stream, p, ctx.num_sms);
  } else if (u.hi && x.dtype == 4) {
    index_t rps = 0;
    chunks = utx_tc_splits(m, l, n, ctx.num_sms, &rps);
    part = chunks == 1 ? f : ctx.get<double>("f.part", chunks * l * n);
    pass_mark(ctx, 0);
    launch_utx_tc_planes(ctx.stream, u.hi, u.lo, u.ldt, static_cast<const float*>(x.p), x.ld, m, l, n, part,
                         ctx.num_sms);
  } else {
    // the fp64 fast kernel runs 128 x 128 tiles, one CTA per SM (gemm_simt.cu)
    const bool fast64 = x.dtype == 8 && !exact && l > 64 && n > 64;
    chunks = fast64 ? pick_chunks(ctx, m, ceil_div(n, 128) * ceil_div(l, 128) / 2, exact)
                    : pick_chunks(ctx, m, ceil_div(n, 64) * ceil_div(l, 64), exact);
    const index_t chunk_rows = round_up(ceil_div(m, chunks), 128);
    chunks = ceil_div(m, chunk_rows);
    part = chunks == 1 ? f : ctx.get<double>("f.part", chunks * l * n);
    pass_mark(ctx, 0);
    if (x.dtype == 4)
      launch_utx_simt<float>(ctx.stream, static_cast<const float*>(u.plain), u.ld,
                             static_cast<const float*>(x.p), x.ld, m, l, n, chunk_rows, part, false);
    else
      launch_utx_simt<double>(ctx.stream, static_cast<const double*>(u.plain), u.ld,
                              static_cast<const double*>(x.p), x.ld, m, l, n, chunk_rows, part, exact);
  }
  LPCA_LAUNCHED(ctx);
  pass_mark(ctx, 1);
  if (chunks > 1) {
    launch_reduce_partials(ctx.stream, part, chunks, l * n, f);
    LPCA_LAUNCHED(ctx);
  }
  if (over_ranks) ctx.allreduce(f, l * n);
}

// Orthonormalises the power step's Z (n x l, held as F = Z^T, l x n) by
// shifted CholeskyQR3 (Fukaya et al. 2020): a first Cholesky of ZᵀZ + s·I with
// s = 11 (n l + l (l + 1)) u ||Z||_F^2 survives condition numbers up to ~1/u
// (q >= 2 makes Z's columns that close: plain CholeskyQR2 fails there, as the
// survey's naive-power probe did), then two plain CholeskyQR passes
// restore orthogonality. Each pass: F <- L^{-1} F with L L^T = F F^T.
// The power step's Cholesky statuses (pivot + 1 of a failed pass, else 0).
void check_orth_status(const int* h3) {
  for (int p = 0; p < 3; ++p)
    if (h3[p] != 0)
      throw Error(kRankDeficiency, "power iteration: cholesky pivot " + S(h3[p] - 1) + " is not positive definite",
                  h3[p] - 1);
}

// Shifted CholeskyQR3 (Fukaya, Kannan, Nakatsukasa, Yamamoto, Yanagisawa 2020)
// of the tall matrix A = [top; body]: top an optional l x l fp64 block (the
// streaming reducer's running R, on this rank), body `rows` x l row-major
// (dtype, ld) on this rank, rows of all ranks stacked when over_ranks (the
// Gram matrices are summed). The first Cholesky factors G + s I with
// s = 11 (M l + l (l + 1)) u ||A||_F^2 (M = global rows), which succeeds up
// to cond(A) ~ 1/u; two plain passes restore orthogonality. Q overwrites top
// and body. Left on the device for one deferred host check (qr_check): the
// diagonal of R = R3 R2 R1 (the remaining column norms the reference's
// Householder QR tests, qr.cpp:37-58), ||A||_F^2 and each pass's Cholesky
// failure (pivot + 1). With r_out, R itself (upper, column-major l x l).
struct QrDev {
  double* rdiag = nullptr;
  double* fro2 = nullptr;
  int* st = nullptr;
};

QrDev cholqr3(lpca_ctx& ctx, double* top, void* body, int dtype, index_t rows, index_t ld, index_t l,
              double global_rows, bool over_ranks, bool exact, double* r_out, const std::string& tag) {
  QrDev q;
  q.rdiag = ctx.get<double>(tag + ".rdiag", l);
  q.fro2 = ctx.get<double>(tag + ".fro2", 1);
  q.st = ctx.get<int>(tag + ".st", 3);
  double* g = ctx.get<double>(tag + ".g", l * l);
  double* w = ctx.get<double>(tag + ".w", l * l);
  double* lm = ctx.get<double>(tag + ".lm", l * l);
  double* tmp = ctx.get<double>(tag + ".tmp", l * l);
  const double shift = 11.0 * (global_rows * static_cast<double>(l) + static_cast<double>(l) * (l + 1)) * 0x1p-53;
  for (int p = 0; p < 3; ++p) {
    // G = A^T A (this rank's rows, then summed over ranks)
    if (rows > 0) {
      index_t chunks = pick_chunks(ctx, rows, ceil_div(l, 64) * ceil_div(l, 64), exact);
      const index_t chunk_rows = round_up(ceil_div(rows, chunks), 128);
      chunks = ceil_div(rows, chunk_rows);
      double* gpart = chunks == 1 ? g : ctx.get<double>(tag + ".gpart", chunks * l * l);
      if (dtype == 4)
        launch_syrk_partials<float>(ctx.stream, static_cast<const float*>(body), ld, rows, l, chunk_rows, gpart);
      else
        launch_syrk_partials<double>(ctx.stream, static_cast<const double*>(body), ld, rows, l, chunk_rows, gpart);
      LPCA_LAUNCHED(ctx);
      if (chunks > 1) {
        launch_reduce_partials(ctx.stream, gpart, chunks, l * l, g);
        LPCA_LAUNCHED(ctx);
      }
    } else {
      launch_zero(ctx.stream, g, sizeof(double) * l * l);
    }
    if (top) {
      launch_small_gemm(ctx.stream, 1, 0, l, top, top, g, 1.0);
      LPCA_LAUNCHED(ctx);
    }
    if (over_ranks) ctx.allreduce(g, l * l);
    if (p == 0) {
      launch_trace(ctx.stream, g, l, q.fro2);
      launch_add_trace_shift(ctx.stream, g, l, shift);
      ctx.note_launch(2);
    }
    launch_chol_inverse(ctx.stream, g, l, w, lm, q.st + p, 0.0);
    launch_rdiag_update(ctx.stream, w, l, q.rdiag, p == 0);
    ctx.note_launch(2);
    if (r_out) {  // R <- R_p R with R_p = L_p^T
      launch_small_gemm(ctx.stream, 1, 0, l, lm, p == 0 ? nullptr : r_out, tmp, 0.0);
      LPCA_CUDA(cudaMemcpyAsync(r_out, tmp, sizeof(double) * l * l, cudaMemcpyDeviceToDevice, ctx.stream));
      LPCA_LAUNCHED(ctx);
    }
    // Q <- Q W_p
    if (rows > 0) {
      void* qb = ctx.buf(tag + ".q", dsize(dtype) * rows * ld);
      if (dtype == 8) {
        launch_xw_simt<double, double>(ctx.stream, static_cast<const double*>(body), rows, l, ld, w, l, l,
                                       static_cast<double*>(qb), ld, 1, exact);
      } else {
        float* w32 = ctx.get<float>(tag + ".w32", l * l);
        launch_convert_f64_to_f32(ctx.stream, w, l, w32, l, l, l, 1.0);
        LPCA_LAUNCHED(ctx);
        launch_zero(ctx.stream, qb, sizeof(float) * rows * ld);
        launch_xw_simt<float, float>(ctx.stream, static_cast<const float*>(body), rows, l, ld, w32, l, l,
                                     static_cast<float*>(qb), ld, 1, false);
      }
      LPCA_LAUNCHED(ctx);
      LPCA_CUDA(cudaMemcpyAsync(body, qb, dsize(dtype) * rows * ld, cudaMemcpyDeviceToDevice, ctx.stream));
    }
    if (top) {
      launch_small_gemm(ctx.stream, 0, 0, l, top, w, tmp, 0.0);
      LPCA_CUDA(cudaMemcpyAsync(top, tmp, sizeof(double) * l * l, cudaMemcpyDeviceToDevice, ctx.stream));
      LPCA_LAUNCHED(ctx);
    }
  }
  return q;
}

// Host copies of a QrDev, valid after the stream has been synchronised.
struct QrHost {
  const double* rdiag = nullptr;
  const double* fro2 = nullptr;
  const int* st = nullptr;
  index_t l = 0;
};
QrHost qr_stage(lpca_ctx& ctx, const QrDev& d, index_t l) {
  return QrHost{ctx.stage_read(d.rdiag, l), ctx.stage_read(d.fro2, 1), ctx.stage_read(d.st, 3), l};
}

// householder_qr's rank test (qr.cpp:37-58): the first column whose remaining
// norm |R_jj| is at most 1e-12 ||A||_F (or whose Cholesky pivot failed) is
// numerically dependent. Returns -1 or the column; *norm gets |R_jj|.
index_t qr_first_dependent(const QrHost& h, double* norm) {
  const double tol = 1e-12 * std::sqrt(h.fro2[0] > 0.0 ? h.fro2[0] : 0.0);
  for (int p = 0; p < 3; ++p)
    if (h.st[p] != 0) {  // a pass's pivot was not positive: that column has no remaining norm
      *norm = 0.0;
      return h.st[p] - 1;
    }
  for (index_t j = 0; j < h.l; ++j) {
    const double r = std::fabs(h.rdiag[j]);
    if (!(r > tol)) {
      *norm = r;
      return j;
    }
  }
  return -1;
}

void orth_rows(lpca_ctx& ctx, double* f, index_t l, index_t n, int* st3 = nullptr) {
  double* g = ctx.get<double>("orth.g", l * l);
  double* w = ctx.get<double>("orth.w", l * l);
  double* lm = ctx.get<double>("orth.l", l * l);
  double* tmp = ctx.get<double>("orth.tmp", l * n);
  const bool deferred = st3 != nullptr;
  if (!deferred) st3 = ctx.get<int>("orth.status", 3);
  double* gpart = ctx.get<double>("gram.part", gram_fast_chunks(l, n) * l * l);
  const double shift = 11.0 * (static_cast<double>(n) * l + static_cast<double>(l) * (l + 1)) * 0x1p-53;
  for (int pass = 0; pass < 3; ++pass) {
    launch_gram_fast(ctx.stream, f, l, n, g, gpart);
    LPCA_LAUNCHED(ctx);
    if (pass == 0) {
      launch_add_trace_shift(ctx.stream, g, l, shift);
      LPCA_LAUNCHED(ctx);
    }
    launch_chol_inverse(ctx.stream, g, l, w, lm, st3 + pass);
    LPCA_LAUNCHED(ctx);
    launch_apply_rinv_t(ctx.stream, w, l, f, n, tmp);
    LPCA_LAUNCHED(ctx);
  }
  if (!deferred) {
    const int* h = ctx.stage_read(st3, 3);
    LPCA_CUDA(cudaStreamSynchronize(ctx.stream));
    check_orth_status(h);
    ctx.pin_reset();
  }
}

struct PhaseEvents {
  lpca_ctx& ctx;
  explicit PhaseEvents(lpca_ctx& c) : ctx(c) {
    for (auto& e : ctx.ev)
      if (!e) LPCA_CUDA(cudaEventCreate(&e));
  }
  void mark(int i) { LPCA_CUDA(cudaEventRecord(ctx.ev[i], ctx.stream)); }
  double secs(int a, int b) {
    float ms = 0.f;
    LPCA_CUDA(cudaEventElapsedTime(&ms, ctx.ev[a], ctx.ev[b]));
    return ms * 1e-3;
  }
};

void regenerate_dev(lpca_ctx& ctx, const lpca_config& c, double* omega) {
  if (c.projection_kind == LPCA_GAUSSIAN)
    launch_omega_gaussian(ctx.stream, c.proj_n, c.proj_l, c.seed, omega, c.proj_n);
  else
    launch_omega_very_sparse(ctx.stream, c.proj_n, c.proj_l, c.density, c.seed, omega, c.proj_n);
  LPCA_LAUNCHED(ctx);
}

// Symmetric eigensolve of a device l x l matrix (overwritten for Jacobi).
// method 0: tridiagonal route (Householder + multisection + inverse iteration),
// method 1: parallel cyclic Jacobi (the cross-check solver).
void eigh_dev(lpca_ctx& ctx, double* a, index_t l, double* evals, double* evecs, int* st, double* gap,
              int method) {
  if (method == 1) {
    double* work = ctx.get<double>("eig.jwork", 2 * l * l);
    launch_jacobi_eigh(ctx.stream, a, l, evals, evecs, work, st, gap);
    LPCA_LAUNCHED(ctx);
    return;
  }
  void* work = ctx.buf("eig.twork", eigh_tridiag_workspace(l));
  launch_eigh_tridiag(ctx.stream, a, l, evals, evecs, work, st, gap);
  ctx.note_launch(12);
  LPCA_CUDA(cudaGetLastError());
}

// truncated_svd_via_gram on a device F (l x n). Fills v (n x k), sigma (host),
// and optionally u~ (device, l x k). Throws the reference's errors.
void finish_spectral(lpca_ctx& ctx, const double* f, index_t l, index_t n, index_t k, double* v,
                     std::vector<double>& sigma, double* ut_out,
                     const std::function<void()>& before_sync = std::function<void()>(),
                     const std::function<void()>& pre_check = std::function<void()>()) {
  if (l > n)
    throw Error(kDimension, "truncated_svd_via_gram: F must be wide (l <= n), got " + S(l) + "x" + S(n));
  if (k < 1 || k > l)
    throw Error(kInvalidArgument, "truncated_svd_via_gram: need 1 <= k <= l, got k = " + S(k));
  double* g = ctx.get<double>("svd.g", l * l);
  double* evals = ctx.get<double>("svd.evals", l);
  double* evecs = ctx.get<double>("svd.evecs", l * l);
  int* st = ctx.get<int>("svd.status", 2);
  double* gap = ctx.get<double>("svd.gap", 1);
  if (ctx.exact) {
    launch_gram(ctx.stream, f, l, n, g);  // the reference's rounding sequence
  } else {
    launch_gram_fast(ctx.stream, f, l, n, g, ctx.get<double>("gram.part", gram_fast_chunks(l, n) * l * l));
  }
  LPCA_LAUNCHED(ctx);
  eigh_dev(ctx, g, l, evals, evecs, st, gap, ctx.eigensolver);
  launch_vform(ctx.stream, f, l, n, evecs, evals, k, nullptr, v);
  LPCA_LAUNCHED(ctx);
  launch_sign_canon(ctx.stream, v, n, k, evecs, l);
  LPCA_LAUNCHED(ctx);
  if (ut_out) {
    LPCA_CUDA(cudaMemcpyAsync(ut_out, evecs, sizeof(double) * l * k, cudaMemcpyDeviceToDevice, ctx.stream));
  }
  // pinned staging: the copies are queued, the host does not wait here
  const double* lam = ctx.stage_read(evals, l);
  const int* hsw = ctx.stage_read(st, 2);
  const double* hgapp = ctx.stage_read(gap, 1);
  int hst = 0;
  cudaEvent_t checked = nullptr;
  if (before_sync) {  // work enqueued behind the spectral step, before the host checks wait
    LPCA_CUDA(cudaEventCreateWithFlags(&checked, cudaEventDisableTiming));
    LPCA_CUDA(cudaEventRecord(checked, ctx.stream));
    before_sync();
    LPCA_CUDA(cudaEventSynchronize(checked));
    LPCA_CUDA(cudaEventDestroy(checked));
  } else {
    LPCA_CUDA(cudaStreamSynchronize(ctx.stream));
  }
  if (pre_check) pre_check();  // earlier phases' deferred checks (power steps, SPCA's QR) come first
  hst = hsw[0];
  ctx.last_sweeps = hsw[1];
  const double hgap = hgapp[0];
  if (std::getenv("LPCA_VERBOSE")) std::fprintf(stderr, "lazypca_b200: eigh l=%lld sweeps=%d\n", (long long)l, hsw[1]);
  if (hst == 2)
    throw Error(kInvalidArgument, "eigh: input is not symmetric (max |a_ij - a_ji| = " +
                                      std::to_string(hgap) + ")");
  if (hst == 1)
    throw Error(kConvergence, "eigh: Jacobi off-diagonal " + std::to_string(hgap) +
                                  " still above tolerance after 50 sweeps", -1, hgap);
  // rank floor (truncated_svd.cpp:28-39)
  const double lambda_max = lam[0];
  const double floor = 1e-12 * (lambda_max > 0.0 ? lambda_max : 0.0);
  index_t safe = 0;
  while (safe < l && lam[static_cast<std::size_t>(safe)] > floor && lam[static_cast<std::size_t>(safe)] > 0.0)
    ++safe;
  if (k > safe)
    throw Error(kRankDeficiency, "truncated_svd_via_gram: requested rank " + S(k) +
                                     " exceeds the numerical rank; largest safe k = " + S(safe),
                safe);
  sigma.resize(static_cast<std::size_t>(k));
  for (index_t r = 0; r < k; ++r) sigma[static_cast<std::size_t>(r)] = std::sqrt(lam[static_cast<std::size_t>(r)]);
}

struct FitResult {
  lpca_map* map = nullptr;
};

// The fit pipeline on a device-resident X (this rank's rows).
// after_spectral (optional): enqueued on the stream right behind the spectral
// step, before the host reads the eigenvalues back (the fused fit + transform);
// it gets the map (V ready on the stream) and the device max|X| of the fit.
using AfterSpectral = std::function<void(lpca_map&, const uint32_t*)>;

// The row gather's schedule for this very sparse Omega (cached on the context:
// a fit's Omega is fixed by n, l, density and seed). Builds it from Omega's
// column lists (one small device-to-host copy and a host edge colouring, once
// per Omega); false when some column or bank has more than 192 entries.
bool row_schedule(lpca_ctx& ctx, const lpca_config& c, const double* omega, index_t n, index_t l) {
  char key[160];
  std::snprintf(key, sizeof key, "%lld/%lld/%.17g/%llu", static_cast<long long>(n), static_cast<long long>(l),
                c.density, static_cast<unsigned long long>(c.seed));
  if (ctx.row_sched_key == key) return ctx.row_sched_steps > 0;
  constexpr int cap = 193;  // one past the longest schedule
  int* cnt = ctx.get<int>("so.cnt", l);
  auto* cols = ctx.get<std::uint32_t>("so.cols", l * cap);
  launch_omega_col_lists(ctx.stream, omega, n, l, cap, cnt, cols);
  LPCA_LAUNCHED(ctx);
  std::vector<int> hc(static_cast<size_t>(l));
  std::vector<std::uint32_t> hl(static_cast<size_t>(l) * cap);
  LPCA_CUDA(cudaMemcpyAsync(hc.data(), cnt, sizeof(int) * l, cudaMemcpyDeviceToHost, ctx.stream));
  LPCA_CUDA(cudaMemcpyAsync(hl.data(), cols, sizeof(std::uint32_t) * l * cap, cudaMemcpyDeviceToHost, ctx.stream));
  LPCA_CUDA(cudaStreamSynchronize(ctx.stream));
  std::vector<std::uint32_t> packed;
  int smax = 0, splits = 1;
  const int steps = build_row_schedule(hc.data(), hl.data(), cap, n, l, packed, &smax, &splits);
  if (steps > 0) {
    void* d = ctx.buf("so.rows", packed.size() * sizeof(std::uint32_t));
    LPCA_CUDA(cudaMemcpyAsync(d, packed.data(), packed.size() * sizeof(std::uint32_t), cudaMemcpyHostToDevice,
                              ctx.stream));
    LPCA_CUDA(cudaStreamSynchronize(ctx.stream));  // packed dies here
  }
  ctx.row_sched_key = key;
  ctx.row_sched_steps = steps;
  ctx.row_sched_smax = smax;
  ctx.row_sched_splits = splits;
  return steps > 0;
}

lpca_map* fit_dev(lpca_ctx& ctx, const lpca_config& cfg_in, const DevX& x, lpca_timings* t,
                  const AfterSpectral* after_spectral = nullptr) {
  // Ranks first agree on the shape (one small collective), so a rank-specific
  // input error is raised on every rank instead of leaving the others waiting
  // in a collective; the global row count sets the QR shifts.
  double m_global = static_cast<double>(x.m);
  if (ctx.world > 1) {
    const std::vector<double> all = ctx.gather_host({static_cast<double>(x.n), static_cast<double>(x.m)});
    m_global = 0.0;
    for (int r = 0; r < ctx.world; ++r) {
      if (all[2 * r] != static_cast<double>(x.n))
        throw Error(kDimension, "ranks disagree on the column count: rank " + std::to_string(r) + " has " +
                                    S(static_cast<index_t>(all[2 * r])) + ", rank " + std::to_string(ctx.rank) +
                                    " has " + S(x.n));
      m_global += all[2 * r + 1];
    }
  }
  const lpca_config c = resolve(cfg_in, x.n);
  if (c.streaming)
    throw Error(kInvalidArgument,
                "streaming reducers take a row-block stream; use block_rows = 0 for in-core data");
  PhaseEvents ev(ctx);
  ev.mark(0);
  const index_t n = x.n, l = c.l, k = c.k, m = x.m;
  auto map = new lpca_map();
  map->device = ctx.device;
  map->method = c.method;
  map->k = k;
  map->l = l;
  map->n = n;
  map->seed = c.seed;
  map->density = c.density;
  map->scale = projection_scale(c);
  try {
    map->alloc_v(ctx, sizeof(double) * (n * k > 0 ? n * k : 1));
    double* omega = ctx.get<double>("omega", n * l);
    regenerate_dev(ctx, c, omega);
    if (c.method == LPCA_RP) {
      launch_scale_f64(ctx.stream, omega, map->v, n * k, 1.0 / map->scale);
      LPCA_LAUNCHED(ctx);
      ev.mark(1);
      LPCA_CUDA(cudaStreamSynchronize(ctx.stream));
      if (t) {
        t->sketch += ev.secs(0, 1);
        t->total += ev.secs(0, 1);
      }
      return map;
    }
    const bool exact = ctx.exact != 0 && x.dtype == 8;
    const bool tc = use_tc(ctx, x, l);
    const index_t mm = m > 0 ? m : 1;
    // fp16 encoding for every pass after the sketch (pair kernels, Lazy SPCA)
    const bool f16 = tc && tc_pair_mode() && f16_enabled() && c.method == LPCA_LAZY_SPCA;
    XScale xs;
    if (f16) {
      xs.dev = ctx.get<uint32_t>("xmax", 1);
      launch_zero(ctx.stream, xs.dev, sizeof(uint32_t));
    }
    // U (m x l, row-major, ld padded to 16): the plain matrix for the SIMT and
    // SPCA paths, tf32 hi/lo planes for the tensor-core U^T X kernel.
    Panel u;
    u.ld = round_up(l, 16);
    if (!tc || c.method == LPCA_SPCA) u.plain = ctx.buf("u", dsize(x.dtype) * mm * u.ld);
    if (f16) {
      u.ldt16 = round_up(mm, 8);
      u.h16hi = ctx.get<__half>("u.h16hi", u.ld * u.ldt16);
      u.h16lo = ctx.get<__half>("u.h16lo", u.ld * u.ldt16);
      u.uinv = ctx.get<float>("u.inv", ceil_div(mm, kUScaleRows) * u.ld);
    } else if (tc) {
      u.ldt = planes_ld(m);
      u.hi = ctx.get<float>("u.hi", u.ld * u.ldt);
      u.lo = ctx.get<float>("u.lo", u.ld * u.ldt);
    }
    // sketch U = X Omega (reducer.cpp:163-169): fp16 with per-(row, run) scales
    // scanned in-kernel, recording max|X| for the single scale of later passes
    XScale sketch;
    sketch.use = true;
    sketch.check = xs.dev;
    // very sparse Omega on dense X: the sketch as a gather (csrc/sparse_omega.cu,
    // one read of X, the reference's summation order) where the dense pass
    // would be DMMA or SIMT (sparse_omega_mode)
    const int so_mode = sparse_omega_mode();
    const bool very_sparse = c.projection_kind == LPCA_VERY_SPARSE && !x.sparse() && so_mode != 0;
    // fp32: the row gather (lanes = Omega columns, a bank-conflict-free schedule)
    const bool rows = very_sparse && x.dtype == 4 && (so_mode == 1 || !tc || n > 8192) &&
                      row_gather_feasible(m, n, x.ld, l) && row_schedule(ctx, c, omega, n, l);
    const bool gather = very_sparse && !rows && u.ld <= 512 && (so_mode == 1 || !tc);
    int* xovf = nullptr;
    if (f16 && !ctx.force_scan && !gather && !rows) {  // scales from each run's first stage (rerun with the scan if flagged)
      xovf = ctx.get<int>("xovf", 1);
      launch_zero(ctx.stream, xovf, sizeof(int));
      sketch.ovf = xovf;
    }
    ev.mark(12);
    ev.mark(13);
    if (rows) {
      float* up = u.plain ? static_cast<float*>(u.plain) : ctx.get<float>("u.gather", mm * u.ld);
      // one launch per landed chunk of a host X still crossing PCIe (else one)
      auto chunks = std::move(ctx.arrivals);
      ctx.arrivals.clear();
      if (chunks.empty()) chunks.emplace_back(m, nullptr);
      index_t r0 = 0;
      for (const auto& ch : chunks) {
        if (ch.second) LPCA_CUDA(cudaStreamWaitEvent(ctx.stream, ch.second, 0));
        launch_sparse_sketch_rows(ctx.stream, static_cast<const float*>(x.p) + r0 * x.ld, ch.first - r0, n, x.ld,
                                  static_cast<const std::uint32_t*>(ctx.buf("so.rows", 4)), ctx.row_sched_steps,
                                  ctx.row_sched_smax, ctx.row_sched_splits, l, up + r0 * u.ld, u.ld,
                                  f16 ? xs.dev : nullptr, ctx.num_sms);
        LPCA_LAUNCHED(ctx);
        r0 = ch.first;
      }
      if (f16) {
        launch_u_planes_f16(ctx.stream, up, m, u.ld, u.ld, u.h16hi, u.h16lo, u.ldt16, u.uinv);
        ctx.note_launch();
      } else if (u.hi && m > 0) {
        launch_split_tf32_transpose(ctx.stream, up, m, l, u.ld, u.hi, u.lo, u.ldt);
        ctx.note_launch();
      }
      ev.mark(13);
    } else if (gather) {
      ctx.wait_arrivals();
      const index_t nch = sparse_sketch_chunks(n, x.dtype);
      int* counts = ctx.get<int>("so.counts", nch * l);
      int* ptr = ctx.get<int>("so.ptr", nch * l + 1);
      // per (chunk, column): its nonzeros padded to pairs, at least one pair
      auto* ent = ctx.get<std::uint32_t>("so.ent", (n + 2 * nch) * l);
      launch_omega_chunk_lists(ctx.stream, omega, n, l, x.dtype, counts, ptr, ent);
      ctx.note_launch(3);
      ev.mark(12);
      if (x.dtype == 8) {
        launch_sparse_sketch<double>(ctx.stream, static_cast<const double*>(x.p), m, n, x.ld, ptr, ent, l,
                                     static_cast<double*>(u.plain), u.ld, nullptr, ctx.num_sms);
      } else {
        float* up = u.plain ? static_cast<float*>(u.plain) : ctx.get<float>("u.gather", mm * u.ld);
        launch_sparse_sketch<float>(ctx.stream, static_cast<const float*>(x.p), m, n, x.ld, ptr, ent, l, up, u.ld,
                                    f16 ? xs.dev : nullptr, ctx.num_sms);
        if (f16) {
          launch_u_planes_f16(ctx.stream, up, m, u.ld, u.ld, u.h16hi, u.h16lo, u.ldt16, u.uinv);
          ctx.note_launch();
        } else if (u.hi && m > 0) {
          launch_split_tf32_transpose(ctx.stream, up, m, l, u.ld, u.hi, u.lo, u.ldt);
          ctx.note_launch();
        }
      }
      LPCA_LAUNCHED(ctx);
      ev.mark(13);
    } else if (x.sparse() && c.projection_kind == LPCA_VERY_SPARSE && so_mode != 0 && l <= 512) {
      // sparse X, very sparse Omega: W's rows as sign bit masks (csrc/sparse.cu),
      // bitwise the dense-W gather with 1/25 of its L2 reads at l = 100
      auto* masks = ctx.get<std::uint32_t>("so.masks", n * 2 * pm1_mask_words(l));
      launch_pm1_masks(ctx.stream, omega, n, l, n, masks);
      LPCA_LAUNCHED(ctx);
      ev.mark(12);
      launch_spmm_csr_pm1(ctx.stream, m, x.rp, x.ci, x.rv, masks, l, static_cast<double*>(u.plain), u.ld, 1);
      LPCA_LAUNCHED(ctx);
      ev.mark(13);
    } else {
      ctx.pass_slot = 12;
      xw_pass(ctx, x, omega, l, n, u, exact, f16 ? &sketch : nullptr);
      ctx.pass_slot = -1;
    }
    ctx.wait_arrivals();  // everything after the sketch reads all of X
    double* xovf_all = nullptr;  // the flag summed over ranks: every rank reruns, or none
    if (ctx.world > 1 && !ctx.force_scan) {  // issued by every rank, with or without an fp16 sketch
      xovf_all = ctx.get<double>("xovf.all", 1);
      if (xovf) {
        launch_flag_to_f64(ctx.stream, xovf, xovf_all);
        LPCA_LAUNCHED(ctx);
      } else {
        launch_zero(ctx.stream, xovf_all, sizeof(double));
      }
      ctx.allreduce(xovf_all, 1);
    }
    xs.use = f16;
    ev.mark(1);
    // Whether a later sketch stage outgrew its run's first-stage scale (summed
    // over ranks, so every rank takes the same branch). Read only after the
    // stream has drained past the flag's producer.
    auto sketch_flagged = [&]() -> bool {
      if (!xovf && !xovf_all) return false;
      LPCA_CUDA(cudaStreamSynchronize(ctx.stream));
      if (xovf_all) {
        double all = 0.0;
        LPCA_CUDA(cudaMemcpy(&all, xovf_all, sizeof(double), cudaMemcpyDeviceToHost));
        return all > 0.0;
      }
      int flagged = 0;
      LPCA_CUDA(cudaMemcpy(&flagged, xovf, sizeof(int), cudaMemcpyDeviceToHost));
      return flagged != 0;
    };
    // An overflowed stage leaves inf/NaN in U, so the host checks below (power
    // step pivots, rank floor) may throw before the flag is read: an error
    // raised while the flag is set reruns the fit with the full scan instead.
    auto rerun_scanned = [&]() -> lpca_map* {
      delete map;
      map = nullptr;
      ctx.force_scan = true;
      try {
        lpca_map* again = fit_dev(ctx, cfg_in, x, t, after_spectral);
        ctx.force_scan = false;
        return again;
      } catch (...) {
        ctx.force_scan = false;
        throw;
      }
    };
    try {
    // power iterations (builder extension; SPEC.md:371 lists them as a non-goal)
    double* f = ctx.get<double>("f", l * n);
    // deferred checks: status words stay on the device until the one readback
    // in front of the spectral step's host checks (no host sync per phase)
    int* pst = c.power_iters > 0 ? ctx.get<int>("power.st", 3 * c.power_iters) : nullptr;
    QrDev spca_qr;
    if (c.power_iters > 0) {
      double* z = ctx.get<double>("z.w", l * n);
      for (int it = 0; it < c.power_iters; ++it) {
        const bool timed = it < lpca_ctx::kPowerEvSteps;
        const int pe = 18 + 4 * it;
        if (timed) {  // both passes' kernels bracketed (lpca_timings.power_pass)
          ev.mark(pe);
          ev.mark(pe + 1);
          ctx.pass_slot = pe;
        }
        utx_pass(ctx, x, u, l, f, exact, &xs);               // F = U^T X  (= Z^T)
        ctx.pass_slot = -1;
        orth_rows(ctx, f, l, n, pst + 3 * it);              // Z <- orth(Z), shifted CholeskyQR3
        launch_transpose(ctx.stream, 8, f, l, l, n, z, n);  // W = Z as n x l column-major
        LPCA_LAUNCHED(ctx);
        if (timed) {
          ev.mark(pe + 2);
          ev.mark(pe + 3);
          ctx.pass_slot = pe + 2;
        }
        xw_pass(ctx, x, z, l, n, u, exact, f16 ? &xs : nullptr);  // U = X Z
        ctx.pass_slot = -1;
      }
    }
    ev.mark(2);
    if (c.method == LPCA_SPCA) {
      // Q of U by shifted CholeskyQR3 (the reference: householder_qr,
      // qr.cpp:104-132; the same Q once R's diagonal is positive, the same rank
      // test on R's diagonal, checked with the spectral step's readback)
      spca_qr = cholqr3(ctx, nullptr, u.plain, x.dtype, m, u.ld, l, m_global, true, exact, nullptr, "spca");
      if (u.hi && m > 0) {  // Q's tf32 planes for the tensor-core F = Q^T X
        launch_split_tf32_transpose(ctx.stream, static_cast<const float*>(u.plain), m, l, u.ld, u.hi, u.lo,
                                    u.ldt);
        LPCA_LAUNCHED(ctx);
      }
    }
    ev.mark(3);
    ev.mark(14);
    ev.mark(15);
    ctx.pass_slot = 14;
    utx_pass(ctx, x, u, l, f, exact, &xs);  // F = U^T X (or Q^T X)
    ctx.pass_slot = -1;
    ev.mark(4);
    const float* xmax_h = f16 ? ctx.stage_read(reinterpret_cast<const float*>(xs.dev), 1) : nullptr;
    const int* pst_h = pst ? ctx.stage_read(pst, 3 * c.power_iters) : nullptr;
    QrHost qr_h;
    if (spca_qr.rdiag) qr_h = qr_stage(ctx, spca_qr, l);
    auto pre_check = [&] {  // in the reference's order: power steps, then the QR
      if (xmax_h) map->xmax = xmax_h[0];
      for (int it = 0; pst_h && it < c.power_iters; ++it) check_orth_status(pst_h + 3 * it);
      if (qr_h.rdiag) {
        double norm = 0.0;
        const index_t j = qr_first_dependent(qr_h, &norm);
        if (j >= 0)
          throw Error(kRankDeficiency, "qr: column " + S(j) + " is numerically dependent on earlier columns" +
                                           " (remaining norm " + std::to_string(norm) + ")",
                      j);
      }
    };
    bool marked = false;
    if (after_spectral) {
      finish_spectral(ctx, f, l, n, k, map->v, map->sigma, nullptr, [&] {
        ev.mark(5);
        marked = true;
        (*after_spectral)(*map, f16 ? xs.dev : nullptr);
      }, pre_check);
    } else {
      finish_spectral(ctx, f, l, n, k, map->v, map->sigma, nullptr, std::function<void()>(), pre_check);
    }
    if (!marked) ev.mark(5);
    LPCA_CUDA(cudaEventSynchronize(ctx.ev[5]));
    } catch (const Error&) {
      if (sketch_flagged()) return rerun_scanned();
      throw;
    }
    if (sketch_flagged()) return rerun_scanned();  // finite but imprecise: redo with the scan
    if (t) {
      t->sketch += ev.secs(0, 1);
      t->power += ev.secs(1, 2);
      t->qr += ev.secs(2, 3);
      t->f_form += ev.secs(3, 4);
      t->svd += ev.secs(4, 5);
      t->total += ev.secs(0, 5);
      t->sketch_pass += ev.secs(12, 13);
      t->f_pass += ev.secs(14, 15);
      for (int it = 0; it < c.power_iters && it < lpca_ctx::kPowerEvSteps; ++it)
        t->power_pass += ev.secs(18 + 4 * it, 19 + 4 * it) + ev.secs(20 + 4 * it, 21 + 4 * it);
    }
    return map;
  } catch (...) {
    delete map;
    throw;
  }
}

// Y = X V into a caller buffer (apply_map, reducer.cpp:348-353).
void transform_finish(lpca_ctx& ctx, lpca_timings* t) {
  LPCA_CUDA(cudaEventSynchronize(ctx.ev[8]));
  const int* flag = ctx.tr_flag;
  auto redo = std::move(ctx.tr_redo);
  ctx.tr_flag = nullptr;
  ctx.tr_redo = nullptr;
  if (flag && *flag && redo) {  // a run's first-stage scale did not cover the run
    redo();
    LPCA_CUDA(cudaStreamSynchronize(ctx.stream));
  }
  if (t) {
    float a = 0.f, b = 0.f, c = 0.f;
    LPCA_CUDA(cudaEventElapsedTime(&a, ctx.ev[6], ctx.ev[7]));
    LPCA_CUDA(cudaEventElapsedTime(&b, ctx.ev[16], ctx.ev[17]));
    LPCA_CUDA(cudaEventElapsedTime(&c, ctx.ev[7], ctx.ev[8]));
    t->transform += a * 1e-3;
    t->transform_pass += b * 1e-3;
    t->d2h += c * 1e-3;
  }
}

// xmax_dev: the fit's device max|X| when X is the fitted matrix itself (fused
// fit + transform: the fp16 scale needs no host value and no range check);
// finish = false leaves the final wait (and the timings) to transform_finish.
void transform_dev(lpca_ctx& ctx, const lpca_map& map, const DevX& x, void* y, int y_dtype,
                   int y_layout, int y_location, index_t ldy, lpca_timings* t, double* d2h,
                   const uint32_t* xmax_dev = nullptr, bool finish = true) {
  if (x.n != map.n)
    throw Error(kDimension, "apply_map: data has " + S(x.n) + " columns but the map expects " + S(map.n));
  if (y_dtype != LPCA_F32 && y_dtype != LPCA_F64) throw Error(kInvalidArgument, "transform: bad y dtype");
  if (y_layout != LPCA_ROW_MAJOR && y_layout != LPCA_COL_MAJOR)
    throw Error(kInvalidArgument, "transform: bad y layout");
  const index_t m = x.m, k = map.k;
  const bool row = y_layout == LPCA_ROW_MAJOR;
  if (ldy <= 0) ldy = row ? k : m;
  if (ldy < (row ? k : m))
    throw Error(kInvalidArgument, "transform: ldy = " + S(ldy) + " is smaller than the output's " +
                                      (row ? "row length k = " + S(k) : "column length m = " + S(m)));
  ctx.wait_arrivals();
  PhaseEvents ev(ctx);
  ev.mark(6);
  ev.mark(16);
  ev.mark(17);
  ctx.pass_slot = 16;
  bool y_copied = false;  // Y already on its way to the host chunk by chunk
  if (m > 0 && k > 0) {
    const std::size_t ybytes = dsize(y_dtype) * static_cast<std::size_t>(row ? m * ldy : k * ldy);
    void* ydev = y_location == LPCA_DEVICE ? y : ctx.buf("y", ybytes);
    const index_t ors = row ? ldy : 1, ocs = row ? 1 : ldy;
    if (x.sparse()) {  // spmm over CSR (apply_map = spmm(X, V), reducer.cpp:348-353)
      double* vt = ctx.get<double>("v.rows", map.n * k);
      launch_transpose(ctx.stream, 8, map.v, map.n, map.n, k, vt, k);
      LPCA_LAUNCHED(ctx);
      pass_mark(ctx, 0);
      launch_spmm_csr(ctx.stream, m, x.rp, x.ci, x.rv, vt, k, k, ydev, y_dtype, ors, ocs);
      LPCA_LAUNCHED(ctx);
      pass_mark(ctx, 1);
    } else if (x.dtype == 8) {
      pass_mark(ctx, 0);
      if (y_dtype == 8)
        launch_xw_simt<double, double>(ctx.stream, static_cast<const double*>(x.p), m, x.n, x.ld,
                                       map.v, k, map.n, static_cast<double*>(ydev), ors, ocs, ctx.exact != 0);
      else
        launch_xw_simt<double, float>(ctx.stream, static_cast<const double*>(x.p), m, x.n, x.ld,
                                      map.v, k, map.n, static_cast<float*>(ydev), ors, ocs, ctx.exact != 0);
      LPCA_LAUNCHED(ctx);
      pass_mark(ctx, 1);
    } else if (row && y_dtype == 4 && use_tc(ctx, x, k) && ldy % 4 == 0) {
      Panel yo;
      yo.plain = ydev;
      yo.ld = ldy;
      if (tc_pair_mode() && f16_enabled()) {
        // fp16 encoding with a power-of-two scale per (row, run) taken
        // from the run's first stage (16x headroom): every row of Y keeps its
        // own relative precision whatever the rows' dynamic range. A later
        // stage outside the scale's range sets the flag; transform_finish then
        // redoes the pass with every run scanned first.
        XScale xs;
        xs.use = true;
        xs.ovf = ctx.get<int>("t.ovf", 1);
        launch_zero(ctx.stream, xs.ovf, sizeof(int));
        const index_t ych = y_location == LPCA_HOST ? d2h_chunk_rows(m) : 0;
        if (ych > 0) {
          // Y to a host buffer: each row chunk's copy (copy stream) runs
          // behind the next chunk's launch, so only the last chunk's copy
          // is exposed
          cudaStream_t cs = ctx.copies();
          const std::size_t es = dsize(y_dtype);
          pass_mark(ctx, 0);
          ctx.pass_slot = -1;
          std::size_t i = 0;
          for (index_t r0 = 0; r0 < m; r0 += ych, ++i) {
            const index_t r1 = r0 + ych < m ? r0 + ych : m;
            DevX xc = x;
            xc.p = static_cast<const float*>(x.p) + r0 * x.ld;
            xc.m = r1 - r0;
            Panel yc = yo;
            yc.plain = static_cast<char*>(ydev) + es * r0 * ldy;
            xw_pass(ctx, xc, map.v, k, map.n, yc, false, &xs);
            const cudaEvent_t e = ctx.chunk_event(1, i);
            LPCA_CUDA(cudaEventRecord(e, ctx.stream));
            LPCA_CUDA(cudaStreamWaitEvent(cs, e, 0));
            LPCA_CUDA(cudaMemcpyAsync(static_cast<char*>(y) + es * r0 * ldy, yc.plain, es * (r1 - r0) * ldy,
                                      cudaMemcpyDeviceToHost, cs));
          }
          ctx.pass_slot = 16;
          pass_mark(ctx, 1);
          ev.mark(7);
          const cudaEvent_t done = ctx.chunk_event(1, i);
          LPCA_CUDA(cudaEventRecord(done, cs));
          LPCA_CUDA(cudaStreamWaitEvent(ctx.stream, done, 0));
          y_copied = true;
          if (d2h) *d2h += static_cast<double>(ybytes);
        } else {
          xw_pass(ctx, x, map.v, k, map.n, yo, false, &xs);
        }
        ctx.tr_flag = ctx.stage_read(xs.ovf, 1);
        const double* v = map.v;
        const index_t kk = k, nn = map.n;
        const bool to_host = y_location == LPCA_HOST;
        const std::size_t yb = ybytes;
        ctx.tr_redo = [&ctx, x, v, kk, nn, yo, to_host, y, ydev, yb]() {
          XScale scan;
          scan.use = true;
          xw_pass(ctx, x, v, kk, nn, yo, false, &scan);
          if (to_host) LPCA_CUDA(cudaMemcpyAsync(y, ydev, yb, cudaMemcpyDeviceToHost, ctx.stream));
        };
      } else {
        xw_pass(ctx, x, map.v, k, map.n, yo, false);
      }
    } else {
      float* w32 = ctx.get<float>("v.f32", k * x.n);
      launch_convert_f64_to_f32(ctx.stream, map.v, map.n, w32, x.n, x.n, k, 1.0);
      LPCA_LAUNCHED(ctx);
      pass_mark(ctx, 0);
      if (y_dtype == 4)
        launch_xw_simt<float, float>(ctx.stream, static_cast<const float*>(x.p), m, x.n, x.ld, w32,
                                     k, x.n, static_cast<float*>(ydev), ors, ocs, false);
      else
        launch_xw_simt<float, double>(ctx.stream, static_cast<const float*>(x.p), m, x.n, x.ld, w32,
                                      k, x.n, static_cast<double*>(ydev), ors, ocs, false);
      LPCA_LAUNCHED(ctx);
      pass_mark(ctx, 1);
    }
    if (!y_copied) ev.mark(7);
    ctx.pass_slot = -1;
    if (y_location == LPCA_HOST && !y_copied) {
      LPCA_CUDA(cudaMemcpyAsync(y, ydev, ybytes, cudaMemcpyDeviceToHost, ctx.stream));
      if (d2h) *d2h += static_cast<double>(ybytes);
    }
  } else {
    ev.mark(7);
    ctx.pass_slot = -1;
  }
  ev.mark(8);
  if (finish) transform_finish(ctx, t);
}

// ---- streaming reducers (Algorithms 3 and 4, reducer.cpp:236-335) ------------
// A pull-model source of row blocks (RowBlockStream::next, sparse_matrix.hpp:58-65).
struct BlockSource {
  virtual ~BlockSource() = default;
  virtual bool next(lpca_matrix_view* v, int64_t* slice) = 0;
};

struct CallbackSource final : BlockSource {
  lpca_next_block_fn fn;
  void* user;
  CallbackSource(lpca_next_block_fn f, void* u) : fn(f), user(u) {}
  bool next(lpca_matrix_view* v, int64_t* slice) override {
    const int32_t r = fn(user, v, slice);
    if (r < 0) {
      Error e(kInvalidArgument, "");
      if (take_callback_error(&e)) throw e;  // e.g. a ParseError from lpca_file_stream_next
      throw Error(kInvalidArgument, "streaming: the block callback reported error " + S(r));
    }
    return r > 0;
  }
};

// Row slices of a device-resident X: reduce() with block_rows > 0 runs the
// streaming reducer over SliceRowBlockStream (reducer.cpp:340-346,
// sparse_matrix.cpp:125-139).
struct SliceSource final : BlockSource {
  DevX x;
  index_t block_rows, slices, next_slice = 0;
  SliceSource(const DevX& d, index_t br) : x(d), block_rows(br), slices(ceil_div(d.m, br)) {}
  bool next(lpca_matrix_view* v, int64_t* slice) override {
    if (next_slice >= slices) return false;
    const index_t lo = next_slice * block_rows;
    const index_t hi = lo + block_rows < x.m ? lo + block_rows : x.m;
    *v = lpca_matrix_view{};
    v->dtype = x.dtype;
    v->layout = LPCA_ROW_MAJOR;
    v->location = LPCA_DEVICE;
    v->rows = hi - lo;
    v->cols = x.n;
    v->ld = x.ld;
    v->data = static_cast<const char*>(x.p) + static_cast<std::size_t>(lo) * x.ld * dsize(x.dtype);
    *slice = next_slice++;
    return true;
  }
};

// Stages host row-major blocks through a copy stream into two alternating
// device buffers, so block s+1 crosses PCIe while block s is reduced; other
// layouts are staged on the compute stream.
struct BlockStager {
  lpca_ctx& ctx;
  cudaStream_t cs = nullptr;
  cudaEvent_t copied[2] = {}, used[2] = {};
  int turn = 0, cur = -1;
  explicit BlockStager(lpca_ctx& c) : ctx(c) {
    LPCA_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    for (int b = 0; b < 2; ++b) {
      LPCA_CUDA(cudaEventCreateWithFlags(&copied[b], cudaEventDisableTiming));
      LPCA_CUDA(cudaEventCreateWithFlags(&used[b], cudaEventDisableTiming));
    }
  }
  ~BlockStager() {
    cudaStreamSynchronize(cs);
    for (int b = 0; b < 2; ++b) {
      cudaEventDestroy(copied[b]);
      cudaEventDestroy(used[b]);
    }
    cudaStreamDestroy(cs);
  }
  // The caller's block memory may be reused once the previous copy has landed.
  void before_next() { LPCA_CUDA(cudaStreamSynchronize(cs)); }
  DevX stage(const lpca_matrix_view* v, double* h2d) {
    cur = -1;
    check_view(v);
    if (v->location == LPCA_HOST && v->layout == LPCA_ROW_MAJOR && v->rows > 0 && v->cols > 0) {
      const int b = turn;
      turn ^= 1;
      const std::size_t es = dsize(v->dtype), bytes = es * v->rows * v->cols;
      const std::string slot = b ? "stream.b1" : "stream.b0";
      auto it = ctx.ws.find(slot);
      if (it == ctx.ws.end() || it->second.second < bytes) {  // growing: let both streams drain first
        LPCA_CUDA(cudaStreamSynchronize(cs));
        LPCA_CUDA(cudaStreamSynchronize(ctx.stream));
      }
      void* dst = ctx.buf(slot, bytes);
      LPCA_CUDA(cudaStreamWaitEvent(cs, used[b], 0));  // block s-2's kernels are done with this buffer
      LPCA_CUDA(cudaMemcpy2DAsync(dst, es * v->cols, v->data, es * v->ld, es * v->cols, v->rows,
                                  cudaMemcpyHostToDevice, cs));
      LPCA_CUDA(cudaEventRecord(copied[b], cs));
      LPCA_CUDA(cudaStreamWaitEvent(ctx.stream, copied[b], 0));
      if (h2d) *h2d += static_cast<double>(bytes);
      cur = b;
      return DevX{dst, v->dtype, v->rows, v->cols, v->cols};
    }
    return stage_x(ctx, v, "stream.x", h2d);
  }
  void release() {
    if (cur >= 0) LPCA_CUDA(cudaEventRecord(used[cur], ctx.stream));
  }
};

// Streaming Lazy SPCA (Algorithm 4) and SPCA (Algorithm 3), reducer.cpp:236-335:
// one pass over the blocks accumulating F = sum_s U_s^T X_s (gemm_t_add). SPCA
// also carries the running R of the stacked sketch, R_s = qr_r([R_{s-1}; U_s])
// (qr.cpp:134-142, reducer.cpp:276-292), here by shifted CholeskyQR3 of the
// stacked matrix with the reference's per-slice rank test ("slice s: qr: ...",
// index s); at the end F <- R^{-T} F (solve_rt_in_place, reducer.cpp:55-73,
// with its 1e-12 ||R||_F diagonal test). Ranks reduce their own blocks; a rank's
// errors are held until every rank reaches the first collective and agree on
// them there (so no rank is left waiting), the ranks' R factors are stacked
// (an allgather through the sum collective) and reduced once more, and F is
// summed with one allreduce. A rank with an empty stream contributes nothing.
lpca_map* fit_stream_dev(lpca_ctx& ctx, const lpca_config& cfg_in, BlockSource& src, lpca_timings* t) {
  BlockStager stager(ctx);
  lpca_matrix_view v{};
  int64_t slice = -1;
  const bool dist = ctx.world > 1;
  // Errors before the first collective: raised at once on a single rank, held
  // and agreed on with world > 1.
  std::unique_ptr<Error> held;
  auto hold = [&](const Error& e) {
    if (!dist) throw e;
    if (!held) held = std::make_unique<Error>(e);
  };
  bool have = false;
  try {
    have = src.next(&v, &slice);
    if (have) {
      if (slice != 0) throw Error(kInvalidArgument, "streaming: first slice index must be 0, got " + S(slice));
      check_view(&v);
    } else if (!dist) {
      throw Error(kInvalidArgument, "streaming: the block stream is empty");
    }
  } catch (const Error& e) {
    hold(e);
    have = false;
  }
  index_t n = have ? v.cols : 0;
  if (dist) {  // agree on the width (ranks with an empty stream take it from the others)
    const std::vector<double> all = ctx.gather_host({have ? 1.0 : 0.0, static_cast<double>(n)});
    index_t nn = -1;
    for (int r = 0; r < ctx.world; ++r) {
      if (all[2 * r] == 0.0) continue;
      const index_t nr = static_cast<index_t>(all[2 * r + 1]);
      if (nn >= 0 && nr != nn)
        throw Error(kDimension, "streaming: ranks disagree on the column count (" + S(nn) + " vs " + S(nr) + ")");
      nn = nr;
    }
    if (nn < 0) throw Error(kInvalidArgument, "streaming: the block stream is empty on every rank");
    n = nn;
  }
  lpca_config c = resolve(cfg_in, n);
  if (c.power_iters > 0)
    throw Error(kInvalidArgument,
                "streaming: power iterations read the data more than once; use the in-core reducers");
  const index_t l = c.l, k = c.k;
  PhaseEvents ev(ctx);
  ev.mark(0);
  auto map = std::make_unique<lpca_map>();
  map->device = ctx.device;
  map->method = c.method;
  map->k = k;
  map->l = l;
  map->n = n;
  map->seed = c.seed;
  map->density = c.density;
  map->scale = projection_scale(c);
  map->alloc_v(ctx, sizeof(double) * (n * k > 0 ? n * k : 1));
  double* omega = ctx.get<double>("omega", n * l);
  regenerate_dev(ctx, c, omega);
  if (c.method == LPCA_RP) {  // no data pass (reduce_rp, reducer.cpp:171-190)
    launch_scale_f64(ctx.stream, omega, map->v, n * k, 1.0 / map->scale);
    LPCA_LAUNCHED(ctx);
    ev.mark(1);
    LPCA_CUDA(cudaEventSynchronize(ctx.ev[1]));
    if (t) {
      t->sketch += ev.secs(0, 1);
      t->total += ev.secs(0, 1);
    }
    return map.release();
  }
  const bool spca = c.method == LPCA_SPCA;
  double* f = ctx.get<double>("stream.f", l * n);
  double* fb = ctx.get<double>("stream.fb", l * n);
  double* rrun = spca ? ctx.get<double>("stream.r", l * l) : nullptr;   // running R (upper, column-major)
  double* rtop = spca ? ctx.get<double>("stream.rtop", l * l) : nullptr;  // R_{s-1} as the stacked top block
  launch_zero(ctx.stream, f, sizeof(double) * l * n);
  if (spca) launch_zero(ctx.stream, rrun, sizeof(double) * l * l);
  uint32_t* xmax = ctx.get<uint32_t>("xmax", 1);
  double sk = 0, ff = 0, qr = 0, h2d = 0;
  index_t expected = 0;
  bool first = true;
  try {
    while (have) {
      if (!first) {
        stager.before_next();
        if (!src.next(&v, &slice)) break;
        // pull(): slice order and width (reducer.cpp:101-113)
        if (slice != expected)
          throw Error(kInvalidArgument, "streaming: expected slice " + S(expected) + ", got " + S(slice));
        check_view(&v);
        if (v.cols != n)
          throw Error(kDimension,
                      "streaming: block has " + S(v.cols) + " columns but the projection expects " + S(n));
      }
      if (spca && first && v.rows < l)
        throw Error(kDimension, "streaming spca: first block has " + S(v.rows) +
                                    " rows; the orthonormal route needs at least l = " + S(l));
      ++expected;
      const DevX x = stager.stage(&v, &h2d);
      if (x.m > 0) {
        const bool exact = ctx.exact != 0 && x.dtype == 8;
        const bool tc = use_tc(ctx, x, l);
        const bool f16 = tc && tc_pair_mode() && f16_enabled() && !spca;
        XScale xs;
        xs.dev = xmax;
        Panel u;
        u.ld = round_up(l, 16);
        if (!tc || spca) u.plain = ctx.buf("stream.u", dsize(x.dtype) * x.m * u.ld);
        if (f16) {
          launch_zero(ctx.stream, xmax, sizeof(uint32_t));
          u.ldt16 = round_up(x.m, 8);
          u.h16hi = ctx.get<__half>("u.h16hi", u.ld * u.ldt16);
          u.h16lo = ctx.get<__half>("u.h16lo", u.ld * u.ldt16);
          u.uinv = ctx.get<float>("u.inv", ceil_div(x.m, kUScaleRows) * u.ld);
        } else if (tc) {
          u.ldt = planes_ld(x.m);
          u.hi = ctx.get<float>("u.hi", u.ld * u.ldt);
          u.lo = ctx.get<float>("u.lo", u.ld * u.ldt);
        }
        ev.mark(1);
        XScale sketch;
        sketch.use = true;
        sketch.check = xmax;
        xw_pass(ctx, x, omega, l, n, u, exact, f16 ? &sketch : nullptr);  // U_s = X_s Omega
        xs.use = f16;
        ev.mark(2);
        if (x.sparse()) {  // gemm_t_add continues the running sums: bitwise the reference's streaming
          launch_gemm_t_csc(ctx.stream, n, x.cp, x.ri, x.cv, static_cast<const double*>(u.plain), u.ld, l, f, true);
          LPCA_LAUNCHED(ctx);
        } else {
          utx_pass(ctx, x, u, l, fb, exact, &xs, false);  // F += U_s^T X_s
          launch_add_f64(ctx.stream, fb, f, l * n);
          LPCA_LAUNCHED(ctx);
        }
        ev.mark(3);
        if (spca) {  // R_s = qr_r([R_{s-1}; U_s]) (U_s is consumed)
          LPCA_CUDA(cudaMemcpyAsync(rtop, rrun, sizeof(double) * l * l, cudaMemcpyDeviceToDevice, ctx.stream));
          const QrDev qd = cholqr3(ctx, first ? nullptr : rtop, u.plain, x.dtype, x.m, u.ld, l,
                                   static_cast<double>(x.m + (first ? 0 : l)), false, exact, rrun, "stream.qr");
          const QrHost qh = qr_stage(ctx, qd, l);
          ev.mark(4);
          LPCA_CUDA(cudaEventSynchronize(ctx.ev[4]));
          double norm = 0.0;
          const index_t j = qr_first_dependent(qh, &norm);
          if (j >= 0)
            throw Error(kRankDeficiency, "slice " + S(slice) + ": qr: column " + S(j) +
                                             " is numerically dependent on earlier columns (remaining norm " +
                                             std::to_string(norm) + ")",
                        slice);
          ctx.pin_reset();
        } else {
          ev.mark(4);
          LPCA_CUDA(cudaEventSynchronize(ctx.ev[4]));
        }
        sk += ev.secs(1, 2);
        ff += ev.secs(2, 3);
        qr += ev.secs(3, 4);
      }
      stager.release();
      first = false;
    }
  } catch (const Error& e) {
    hold(e);
  }
  if (dist) {  // every rank arrives here: agree on the held errors (lowest rank's first)
    const std::vector<double> all = ctx.gather_host(
        {held ? static_cast<double>(held->code) : 0.0, held ? static_cast<double>(held->index) : -1.0});
    for (int r = 0; r < ctx.world; ++r) {
      if (all[2 * r] == 0.0) continue;
      if (held && r == ctx.rank) throw *held;
      throw Error(static_cast<int>(all[2 * r]), "streaming: rank " + std::to_string(r) + " failed (see its error)",
                  static_cast<std::int64_t>(all[2 * r + 1]));
    }
  }
  ev.mark(1);
  ctx.allreduce(f, l * n);
  if (spca) {
    double* r = rrun;
    if (dist) {  // stack every rank's R and reduce the stack once more
      const index_t wl = static_cast<index_t>(ctx.world) * l;
      double* stack = ctx.get<double>("stream.rstack", wl * l);  // row-major (world l) x l
      double* rt = ctx.get<double>("stream.rt", l * l);
      launch_zero(ctx.stream, stack, sizeof(double) * wl * l);
      launch_transpose(ctx.stream, 8, rrun, l, l, l, rt, l);  // column-major R -> row-major
      LPCA_LAUNCHED(ctx);
      LPCA_CUDA(cudaMemcpyAsync(stack + static_cast<index_t>(ctx.rank) * l * l, rt, sizeof(double) * l * l,
                                cudaMemcpyDeviceToDevice, ctx.stream));
      ctx.allreduce(stack, wl * l);
      r = ctx.get<double>("stream.rall", l * l);
      cholqr3(ctx, nullptr, stack, 8, wl, l, l, static_cast<double>(wl), false, false, r, "stream.qr2");
    }
    // solve_rt_in_place's test (reducer.cpp:55-73): |R_ii| <= 1e-12 ||R||_F
    const double* rh = ctx.stage_read(r, l * l);
    LPCA_CUDA(cudaStreamSynchronize(ctx.stream));
    double fro = 0.0;
    for (index_t e = 0; e < l * l; ++e) fro += rh[e] * rh[e];
    const double tol = 1e-12 * std::sqrt(fro);
    for (index_t i = 0; i < l; ++i)
      if (!(std::fabs(rh[i * l + i]) > tol))
        throw Error(kRankDeficiency, "triangular solve: R diagonal entry " + S(i) + " is numerically zero", i);
    double* w = ctx.get<double>("spca.w", l * l);
    double* lm = ctx.get<double>("spca.l", l * l);
    int* st = ctx.get<int>("spca.status", 1);
    launch_upper_inverse(ctx.stream, r, l, w, lm, st);
    LPCA_LAUNCHED(ctx);
    launch_apply_rinv_t(ctx.stream, w, l, f, n, ctx.get<double>("orth.tmp", l * n));  // F <- R^{-T} F
    LPCA_LAUNCHED(ctx);
  }
  ev.mark(2);
  finish_spectral(ctx, f, l, n, k, map->v, map->sigma, nullptr);
  ev.mark(3);
  LPCA_CUDA(cudaEventSynchronize(ctx.ev[3]));
  if (t) {
    t->sketch += sk;
    t->f_form += ff;
    t->qr += qr + ev.secs(1, 2);
    t->svd += ev.secs(2, 3);
    t->total += ev.secs(0, 3);
  }
  (void)h2d;
  return map.release();
}

int num_sms_of(int device) {
  int v = 148;
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
  return v;
}

}  // namespace

// ============================== C ABI =========================================
extern "C" {

const char* lpca_last_error(void) { return g_err_msg.c_str(); }
int64_t lpca_last_error_index(void) { return g_err_index; }
double lpca_last_error_gap(void) { return g_err_gap; }
int32_t lpca_abi_version(void) { return LPCA_ABI_VERSION; }

lpca_status lpca_ctx_create(int32_t device, lpca_ctx** out) {
  return lpca_ctx_create_dist(device, 0, 1, nullptr, out);
}

lpca_status lpca_nccl_unique_id(void* out_128_bytes) {
  return guarded([&] {
    ncclUniqueId id;
    nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
    static_assert(sizeof(id) == 128, "NCCL unique id is 128 bytes");
    std::memcpy(out_128_bytes, &id, sizeof(id));
  });
}

namespace {
lpca_ctx* make_ctx(int32_t device, int32_t rank, int32_t world) {
  if (world < 1 || rank < 0 || rank >= world) throw Error(kInvalidArgument, "bad rank/world");
  int count = 0;
  LPCA_CUDA(cudaGetDeviceCount(&count));
  if (device < 0 || device >= count)
    throw Error(kCuda, "device " + std::to_string(device) + " not present (" + std::to_string(count) + " visible)");
  cudaDeviceProp prop;
  LPCA_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    throw Error(kCuda, "lazypca_b200 needs an sm_100 (B200) device; found sm_" + std::to_string(prop.major) +
                           std::to_string(prop.minor));
  LPCA_CUDA(cudaSetDevice(device));
  auto ctx = new lpca_ctx();
  ctx->device = device;
  ctx->rank = rank;
  ctx->world = world;
  ctx->num_sms = num_sms_of(device);
  const char* path = std::getenv("LPCA_GEMM_PATH");
  if (path && std::string(path) == "simt") ctx->gemm_path = 1;
  const cudaError_t e = cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete ctx;
    LPCA_CUDA(e);
  }
  ctx->stream = ctx->own_stream;
  return ctx;
}
}  // namespace

lpca_status lpca_ctx_create_hooked(int32_t device, int32_t rank, int32_t world, lpca_allreduce_fn fn, void* user,
                                   lpca_ctx** out) {
  return guarded([&] {
    if (!out) throw Error(kInvalidArgument, "null output");
    *out = nullptr;
    if (world > 1 && !fn) throw Error(kInvalidArgument, "world > 1 needs an allreduce function");
    lpca_ctx* ctx = make_ctx(device, rank, world);
    ctx->hook = fn;
    ctx->hook_user = user;
    *out = ctx;
  });
}

lpca_status lpca_ctx_create_dist(int32_t device, int32_t rank, int32_t world,
                                 const void* nccl_id_128, lpca_ctx** out) {
  return guarded([&] {
    if (!out) throw Error(kInvalidArgument, "null output");
    *out = nullptr;
    lpca_ctx* ctx = make_ctx(device, rank, world);
    try {
      // world == 1 with an id: a one-rank communicator (every exchange still
      // goes through ncclAllReduce, so the NCCL path runs on a one-GPU box)
      if (world > 1 || nccl_id_128) {
        if (!nccl_id_128) throw Error(kInvalidArgument, "world > 1 needs an NCCL unique id");
        ncclUniqueId id;
        std::memcpy(&id, nccl_id_128, sizeof(id));
        nccl_check(nccl().comm_init_rank(&ctx->comm, world, id, rank), "ncclCommInitRank");
      }
    } catch (...) {
      lpca_ctx_destroy(ctx);
      throw;
    }
    *out = ctx;
  });
}

lpca_status lpca_ctx_destroy(lpca_ctx* ctx) {
  return guarded([&] {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    for (lpca_map* m : ctx->live_maps) {  // maps may outlive their context
      m->owner = nullptr;
      m->stream = nullptr;
    }
    for (auto& kv : ctx->ws) cudaFree(kv.second.first);
    for (auto& e : ctx->ev)
      if (e) cudaEventDestroy(e);
    if (ctx->comm) nccl().comm_destroy(ctx->comm);
    if (ctx->pin) cudaFreeHost(ctx->pin);
    if (ctx->copy_stream) {
      cudaStreamSynchronize(ctx->copy_stream);
      cudaStreamDestroy(ctx->copy_stream);
    }
    for (auto& pool : ctx->chunk_ev)
      for (cudaEvent_t e : pool) cudaEventDestroy(e);
    if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    delete ctx;
  });
}

lpca_status lpca_ctx_set_stream(lpca_ctx* ctx, void* cuda_stream) {
  return guarded([&] {
    check_ctx(ctx);
    ctx->stream = cuda_stream ? static_cast<cudaStream_t>(cuda_stream) : ctx->own_stream;
  });
}

int32_t lpca_debug_row_schedule(const int32_t* cnt, const uint32_t* cols, int32_t cap, int64_t n, int64_t l,
                                uint32_t* out, int64_t out_capacity, int32_t* smax, int32_t* splits) {
  if (smax) *smax = 0;
  if (splits) *splits = 0;
  if (!cnt || !cols || !out || !smax || !splits || cap < 1 || n < 1 || l < 1) return -1;
  try {
    std::vector<std::uint32_t> packed;
    int sm = 0, sp = 0;
    const int steps = build_row_schedule(cnt, cols, cap, n, l, packed, &sm, &sp);
    if (steps < 0 || static_cast<int64_t>(packed.size()) > out_capacity) return -1;
    std::copy(packed.begin(), packed.end(), out);
    *smax = sm;
    *splits = sp;
    return steps;
  } catch (...) {
    return -1;
  }
}

int64_t lpca_debug_check_guards(lpca_ctx* ctx, char* names, int64_t capacity) {
  if (!ctx || !lpca_ctx::guards()) return -1;
  cudaSetDevice(ctx->device);
  if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return -2;
  std::vector<unsigned char> band(lpca_ctx::kGuardBytes);
  std::string bad;
  int64_t count = 0;
  for (const auto& kv : ctx->ws) {
    if (cudaMemcpy(band.data(), static_cast<const char*>(kv.second.first) + kv.second.second, band.size(),
                   cudaMemcpyDeviceToHost) != cudaSuccess)
      return -2;
    for (unsigned char b : band)
      if (b != lpca_ctx::kGuardByte) {
        ++count;
        bad += kv.first + " ";
        break;
      }
  }
  if (names && capacity > 0) {
    const std::size_t n = std::min<std::size_t>(bad.size(), static_cast<std::size_t>(capacity - 1));
    std::memcpy(names, bad.data(), n);
    names[n] = '\0';
  }
  return count;
}

lpca_status lpca_ctx_synchronize(lpca_ctx* ctx) {
  return guarded([&] {
    check_ctx(ctx);
    LPCA_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

lpca_status lpca_ctx_set_gemm_path(lpca_ctx* ctx, int32_t path) {
  return guarded([&] {
    check_ctx(ctx);
    if (path != 0 && path != 1) throw Error(kInvalidArgument, "gemm path must be 0 (tcgen05) or 1 (simt)");
    ctx->gemm_path = path;
  });
}

lpca_status lpca_ctx_set_exact_order(lpca_ctx* ctx, int32_t exact) {
  return guarded([&] {
    check_ctx(ctx);
    ctx->exact = exact != 0;
  });
}

int64_t lpca_ctx_launch_count(const lpca_ctx* ctx) { return ctx ? ctx->launches : 0; }

lpca_status lpca_config_resolve(const lpca_config* in, int64_t data_cols, lpca_config* out) {
  return guarded([&] {
    if (!in || !out) throw Error(kInvalidArgument, "null config");
    *out = resolve(*in, data_cols);
  });
}

lpca_status lpca_density_for(int32_t mode, int64_t k, double value, double* out) {
  return guarded([&] {
    if (k < 2) throw Error(kInvalidArgument, "density policy: k must be at least 2, got " + S(k));
    double d;
    switch (mode) {
      case LPCA_DENSITY_AGGRESSIVE: d = std::log(static_cast<double>(k)) / static_cast<double>(k); break;
      case LPCA_DENSITY_CONSERVATIVE: d = 1.0 / std::sqrt(static_cast<double>(k)); break;
      case LPCA_DENSITY_EXPLICIT: d = value; break;
      default: d = 1.0;
    }
    if (d > 1.0) d = 1.0;
    if (!(d > 0.0)) throw Error(kInvalidArgument, "density policy: derived density is not positive");
    *out = d;
  });
}

lpca_status lpca_regenerate(lpca_ctx* ctx, int32_t kind, int64_t n, int64_t l, double density,
                            uint64_t seed, void* out, int32_t out_location, double* scale) {
  return guarded([&] {
    check_ctx(ctx);
    if (l < 2) throw Error(kInvalidArgument, "projection: sketch width l must be at least 2, got " + S(l));
    if (l > n)
      throw Error(kInvalidArgument, "projection: sketch width l = " + S(l) +
                                        " exceeds data dimensionality n = " + S(n));
    if (!(density > 0.0) || density > 1.0)
      throw Error(kInvalidArgument, "projection: density must lie in (0, 1], got " + std::to_string(density));
    lpca_config c{};
    c.projection_kind = kind;
    c.proj_n = n;
    c.proj_l = l;
    c.density = density;
    c.seed = seed;
    double* dst = out_location == LPCA_DEVICE ? static_cast<double*>(out) : ctx->get<double>("regen", n * l);
    regenerate_dev(*ctx, c, dst);
    if (out_location != LPCA_DEVICE)
      LPCA_CUDA(cudaMemcpyAsync(out, dst, sizeof(double) * n * l, cudaMemcpyDeviceToHost, ctx->stream));
    LPCA_CUDA(cudaStreamSynchronize(ctx->stream));
    if (scale) *scale = projection_scale(c);
  });
}

lpca_status lpca_fit(lpca_ctx* ctx, const lpca_config* cfg, const lpca_matrix_view* x,
                     lpca_map** out_map, lpca_timings* timings) {
  return guarded([&] {
    check_ctx(ctx);
    if (!cfg || !out_map) throw Error(kInvalidArgument, "null argument");
    *out_map = nullptr;
    PhaseEvents ev(*ctx);
    CopyScope copies(*ctx);
    ev.mark(9);
    double h2d = 0.0;
    const bool streamed = (cfg->block_rows > 0 || cfg->streaming) && cfg->method != LPCA_RP;
    // in-core fits take a host X chunk by chunk (the sketch overlaps the copy)
    const DevX dx = streamed ? stage_x(*ctx, x, "x", &h2d) : stage_x_arriving(*ctx, x, "x", &h2d, ctx->ev[9], ctx->ev[10]);
    if (streamed) ev.mark(10);
    if (streamed) {
      // reduce() with block_rows: the streaming reducer over row slices (reducer.cpp:340-346)
      if (cfg->block_rows < 1) throw Error(kInvalidArgument, "reducer: streaming mode needs block_rows >= 1");
      SliceSource src(dx, cfg->block_rows);
      *out_map = fit_stream_dev(*ctx, *cfg, src, timings);
    } else {
      lpca_config c = *cfg;
      c.block_rows = 0;
      c.streaming = 0;
      *out_map = fit_dev(*ctx, c, dx, timings);
      ctx->wait_arrivals();  // RP reads no X
    }
    if (timings) {
      LPCA_CUDA(cudaEventSynchronize(ctx->ev[10]));  // (recorded on the copy stream for a chunked X)
      timings->h2d += ev.secs(9, 10);
    }
  });
}

lpca_status lpca_fit_stream(lpca_ctx* ctx, const lpca_config* cfg, lpca_next_block_fn next, void* user,
                            lpca_map** out_map, lpca_timings* timings) {
  return guarded([&] {
    check_ctx(ctx);
    if (!cfg || !out_map || !next) throw Error(kInvalidArgument, "null argument");
    *out_map = nullptr;
    CallbackSource src(next, user);
    *out_map = fit_stream_dev(*ctx, *cfg, src, timings);
  });
}

lpca_status lpca_transform(lpca_ctx* ctx, const lpca_map* map, const lpca_matrix_view* x, void* y,
                           int32_t y_dtype, int32_t y_layout, int32_t y_location, int64_t ldy,
                           lpca_timings* timings) {
  return guarded([&] {
    check_ctx(ctx);
    if (!map) throw Error(kInvalidArgument, "null map");
    if (!y && x && x->rows > 0 && map->k > 0) throw Error(kInvalidArgument, "null output");
    PhaseEvents ev(*ctx);
    ev.mark(9);
    const DevX dx = stage_x(*ctx, x, "x", nullptr);
    ev.mark(10);
    transform_dev(*ctx, *map, dx, y, y_dtype, y_layout, y_location, ldy, timings, nullptr);
    if (timings) {
      LPCA_CUDA(cudaEventSynchronize(ctx->ev[10]));  // (recorded on the copy stream for a chunked X)
      timings->h2d += ev.secs(9, 10);
    }
  });
}

lpca_status lpca_fit_transform(lpca_ctx* ctx, const lpca_config* cfg, const lpca_matrix_view* x,
                               lpca_map** out_map, void* y, int32_t y_dtype, int32_t y_layout,
                               int32_t y_location, int64_t ldy, lpca_timings* timings) {
  return guarded([&] {
    check_ctx(ctx);
    if (!cfg || !out_map) throw Error(kInvalidArgument, "null argument");
    *out_map = nullptr;
    PhaseEvents ev(*ctx);
    CopyScope copies(*ctx);
    ev.mark(9);
    const bool streamed = (cfg->block_rows > 0 || cfg->streaming) && cfg->method != LPCA_RP;
    const DevX dx = streamed ? stage_x(*ctx, x, "x", nullptr)
                             : stage_x_arriving(*ctx, x, "x", nullptr, ctx->ev[9], ctx->ev[10]);
    if (streamed) ev.mark(10);
    lpca_map* map = nullptr;
    bool fused = false;
    if (streamed) {
      if (cfg->block_rows < 1) throw Error(kInvalidArgument, "reducer: streaming mode needs block_rows >= 1");
      SliceSource src(dx, cfg->block_rows);
      map = fit_stream_dev(*ctx, *cfg, src, timings);
    } else {
      lpca_config c = *cfg;
      c.block_rows = 0;
      c.streaming = 0;
      // the transform is enqueued behind the spectral step, before the fit's
      // host checks: no idle gap between the two on the device
      const AfterSpectral tr = [&](lpca_map& mp, const uint32_t* xmax_dev) {
        transform_dev(*ctx, mp, dx, y, y_dtype, y_layout, y_location, ldy, nullptr, nullptr, xmax_dev, false);
        fused = true;
      };
      map = fit_dev(*ctx, c, dx, timings, &tr);
      ctx->wait_arrivals();  // RP reads no X before its transform
    }
    try {
      if (fused)
        transform_finish(*ctx, timings);
      else  // RP and the streaming reducers: transform after the fit
        transform_dev(*ctx, *map, dx, y, y_dtype, y_layout, y_location, ldy, timings, nullptr);
    } catch (...) {
      delete map;
      throw;
    }
    if (timings) {
      LPCA_CUDA(cudaEventSynchronize(ctx->ev[10]));  // (recorded on the copy stream for a chunked X)
      timings->h2d += ev.secs(9, 10);
    }
    *out_map = map;
  });
}

lpca_status lpca_map_info_get(const lpca_map* map, lpca_map_info* out) {
  return guarded([&] {
    if (!map || !out) throw Error(kInvalidArgument, "null argument");
    std::memset(out, 0, sizeof(*out));
    out->method = map->method;
    out->k = map->k;
    out->l = map->l;
    out->n = map->n;
    out->seed = map->seed;
    out->density = map->density;
    out->scale = map->scale;
    out->has_singular_values = map->sigma.empty() ? 0 : 1;
  });
}

lpca_status lpca_map_copy_v(const lpca_map* map, double* v_out, int32_t out_location) {
  return guarded([&] {
    if (!map || !v_out) throw Error(kInvalidArgument, "null argument");
    LPCA_CUDA(cudaSetDevice(map->device));
    LPCA_CUDA(cudaMemcpyAsync(v_out, map->v, sizeof(double) * map->n * map->k,
                              out_location == LPCA_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                              map->stream));
    LPCA_CUDA(cudaStreamSynchronize(map->stream));
  });
}

lpca_status lpca_map_copy_sigma(const lpca_map* map, double* sigma_out) {
  return guarded([&] {
    if (!map || !sigma_out) throw Error(kInvalidArgument, "null argument");
    std::copy(map->sigma.begin(), map->sigma.end(), sigma_out);
  });
}

lpca_status lpca_map_create(lpca_ctx* ctx, const lpca_map_info* info, const double* v_host,
                            const double* sigma_host, lpca_map** out) {
  return guarded([&] {
    check_ctx(ctx);
    if (!info || !out || (!v_host && info->n * info->k > 0)) throw Error(kInvalidArgument, "null argument");
    if (info->k < 0 || info->n < 0) throw Error(kInvalidArgument, "map: negative shape");
    auto map = new lpca_map();
    map->device = ctx->device;
    map->method = info->method;
    map->k = info->k;
    map->l = info->l;
    map->n = info->n;
    map->seed = info->seed;
    map->density = info->density;
    map->scale = info->scale;
    try {
      map->alloc_v(*ctx, sizeof(double) * (info->n * info->k > 0 ? info->n * info->k : 1));
      if (info->n * info->k > 0)
        LPCA_CUDA(cudaMemcpyAsync(map->v, v_host, sizeof(double) * info->n * info->k, cudaMemcpyHostToDevice, ctx->stream));
      LPCA_CUDA(cudaStreamSynchronize(ctx->stream));
      if (info->has_singular_values && sigma_host) map->sigma.assign(sigma_host, sigma_host + info->k);
    } catch (...) {
      delete map;
      throw;
    }
    *out = map;
  });
}

lpca_status lpca_map_destroy(lpca_map* map) {
  return guarded([&] {
    if (!map) return;
    cudaSetDevice(map->device);
    delete map;
  });
}

// ---- kernel-level exports (fp64, reference summation order) -------------------
namespace {

// fp64 row-major device copy of a view (f32 data widened exactly).
DevX stage_x_f64(lpca_ctx& ctx, const lpca_matrix_view* x) {
  DevX d = stage_x(ctx, x, "kx", nullptr);
  if (d.sparse() || d.dtype == 8 || d.m * d.n == 0) {
    d.dtype = 8;
    return d;
  }
  double* wide = ctx.get<double>("kx.f64", d.m * d.n);
  launch_widen_f32(ctx.stream, static_cast<const float*>(d.p), d.ld, d.m, d.n, wide);
  LPCA_LAUNCHED(ctx);
  return DevX{wide, 8, d.m, d.n, d.n};
}

const double* stage_f64(lpca_ctx& ctx, const double* p, index_t count, int location, const char* slot) {
  if (location == LPCA_DEVICE) return p;
  double* d = ctx.get<double>(slot, count > 0 ? count : 1);
  if (count > 0) LPCA_CUDA(cudaMemcpyAsync(d, p, sizeof(double) * count, cudaMemcpyHostToDevice, ctx.stream));
  return d;
}

void finish_out(lpca_ctx& ctx, double* out, const double* dev, index_t count, int location) {
  if (location != LPCA_DEVICE && count > 0)
    LPCA_CUDA(cudaMemcpyAsync(out, dev, sizeof(double) * count, cudaMemcpyDeviceToHost, ctx.stream));
  LPCA_CUDA(cudaStreamSynchronize(ctx.stream));
}

}  // namespace

lpca_status lpca_spmm(lpca_ctx* ctx, const lpca_matrix_view* x, const double* w, int64_t w_cols,
                      int32_t w_location, double* out, int32_t out_location) {
  return guarded([&] {
    check_ctx(ctx);
    const DevX d = stage_x_f64(*ctx, x);
    const index_t m = d.m, n = d.n;
    const double* wd = stage_f64(*ctx, w, n * w_cols, w_location, "k.w");
    double* od = out_location == LPCA_DEVICE ? out : ctx->get<double>("k.out", m * w_cols);
    if (m > 0 && w_cols > 0 && d.sparse()) {
      double* wt = ctx->get<double>("k.wrows", n * w_cols);
      launch_transpose(ctx->stream, 8, wd, n, n, w_cols, wt, w_cols);
      LPCA_LAUNCHED(*ctx);
      launch_spmm_csr(ctx->stream, m, d.rp, d.ci, d.rv, wt, w_cols, w_cols, od, 8, 1, m);
      LPCA_LAUNCHED(*ctx);
    } else if (m > 0 && w_cols > 0) {
      launch_xw_simt<double, double>(ctx->stream, static_cast<const double*>(d.p), m, n, d.ld, wd,
                                     w_cols, n, od, 1, m, true);
      LPCA_LAUNCHED(*ctx);
    }
    finish_out(*ctx, out, od, m * w_cols, out_location);
  });
}

lpca_status lpca_gemm_t(lpca_ctx* ctx, const double* u, int64_t m, int64_t l, int32_t u_location,
                        const lpca_matrix_view* x, double* out, int32_t out_location) {
  return guarded([&] {
    check_ctx(ctx);
    const DevX d = stage_x_f64(*ctx, x);
    if (d.m != m)
      throw Error(kDimension, "gemm_t: inner dimensions differ (" + S(m) + " vs " + S(d.m) + ")");
    const index_t n = d.n;
    const double* ud = stage_f64(*ctx, u, m * l, u_location, "k.u");
    double* urow = ctx->get<double>("k.urow", m * l);
    if (m * l > 0) {
      launch_transpose(ctx->stream, 8, ud, m, m, l, urow, l);
      LPCA_LAUNCHED(*ctx);
    }
    double* od = out_location == LPCA_DEVICE ? out : ctx->get<double>("k.out", l * n);
    if (l * n > 0) {
      if (m > 0 && d.sparse()) {
        launch_gemm_t_csc(ctx->stream, n, d.cp, d.ri, d.cv, urow, l, l, od, false);
        LPCA_LAUNCHED(*ctx);
      } else if (m > 0) {
        launch_utx_simt<double>(ctx->stream, urow, l, static_cast<const double*>(d.p), d.ld, m, l, n,
                                round_up(m, 16), od, true);
        LPCA_LAUNCHED(*ctx);
      } else {
        launch_zero(ctx->stream, od, sizeof(double) * l * n);
      }
    }
    finish_out(*ctx, out, od, l * n, out_location);
  });
}

lpca_status lpca_chordal_distance(lpca_ctx* ctx, const double* v1, int64_t n1, int64_t k1, const double* v2,
                                  int64_t n2, int64_t k2, int32_t location, double* out) {
  return guarded([&] {
    check_ctx(ctx);
    if (!out || (!v1 && n1 * k1 > 0) || (!v2 && n2 * k2 > 0)) throw Error(kInvalidArgument, "null argument");
    if (n1 != n2)
      throw Error(kDimension, "chordal_distance: bases live in different dimensions (" + S(n1) + " vs " + S(n2) + ")");
    const index_t n = n1;
    const double* a = stage_f64(*ctx, v1, n * k1, location, "ch.v1");
    const double* b = stage_f64(*ctx, v2, n * k2, location, "ch.v2");
    double* g1 = ctx->get<double>("ch.g1", k1 * k1 > 0 ? k1 * k1 : 1);
    double* g2 = ctx->get<double>("ch.g2", k2 * k2 > 0 ? k2 * k2 : 1);
    double* c12 = ctx->get<double>("ch.c12", k1 * k2 > 0 ? k1 * k2 : 1);
    double* c21 = ctx->get<double>("ch.c21", k1 * k2 > 0 ? k1 * k2 : 1);
    launch_atb(ctx->stream, a, n, k1, a, k1, g1);
    launch_atb(ctx->stream, b, n, k2, b, k2, g2);
    launch_atb(ctx->stream, a, n, k1, b, k2, c12);
    launch_atb(ctx->stream, b, n, k2, a, k1, c21);
    LPCA_LAUNCHED(*ctx);
    const index_t p1 = residual_sq_blocks(n, k1), p2 = residual_sq_blocks(n, k2);
    double* part = ctx->get<double>("ch.part", p1 + p2 > 0 ? p1 + p2 : 1);
    launch_residual_sq(ctx->stream, a, n, k1, b, k2, c21, part);       // ||V1 - V2 (V2^T V1)||^2
    launch_residual_sq(ctx->stream, b, n, k2, a, k1, c12, part + p1);  // ||V2 - V1 (V1^T V2)||^2
    LPCA_LAUNCHED(*ctx);
    std::vector<double> h1(static_cast<std::size_t>(k1 * k1)), h2(static_cast<std::size_t>(k2 * k2)),
        hp(static_cast<std::size_t>(p1 + p2));
    if (!h1.empty()) LPCA_CUDA(cudaMemcpyAsync(h1.data(), g1, sizeof(double) * h1.size(), cudaMemcpyDeviceToHost, ctx->stream));
    if (!h2.empty()) LPCA_CUDA(cudaMemcpyAsync(h2.data(), g2, sizeof(double) * h2.size(), cudaMemcpyDeviceToHost, ctx->stream));
    if (!hp.empty()) LPCA_CUDA(cudaMemcpyAsync(hp.data(), part, sizeof(double) * hp.size(), cudaMemcpyDeviceToHost, ctx->stream));
    LPCA_CUDA(cudaStreamSynchronize(ctx->stream));
    // check_orthonormal (metrics.cpp:21-31)
    auto check = [](const std::vector<double>& g, index_t k, const char* which) {
      double worst = 0.0;
      for (index_t j = 0; j < k; ++j)
        for (index_t i = 0; i < k; ++i)
          worst = std::max(worst, std::abs(g[static_cast<std::size_t>(j * k + i)] - (i == j ? 1.0 : 0.0)));
      if (worst > 1e-8 * static_cast<double>(std::max<index_t>(1, k)))
        throw Error(kInvalidArgument, std::string("chordal_distance: ") + which +
                                          " does not have orthonormal columns (max deviation " +
                                          std::to_string(worst) + ")");
    };
    check(h1, k1, "first basis");
    check(h2, k2, "second basis");
    double r = 0.0;
    for (double v : hp) r += v;
    *out = std::sqrt(r);
  });
}

lpca_status lpca_distance_preservation(lpca_ctx* ctx, const lpca_matrix_view* x, const lpca_map* map_a,
                                       const lpca_map* map_b, int64_t max_pairs, uint64_t seed, int64_t* n_pairs,
                                       int64_t* pair_i, int64_t* pair_j, double* original, double* reduced_a,
                                       double* reduced_b, double* max_violation, double* max_discrepancy) {
  return guarded([&] {
    check_ctx(ctx);
    if (!map_a || !n_pairs) throw Error(kInvalidArgument, "null argument");
    const DevX dx = stage_x(*ctx, x, "dp.x", nullptr);
    const index_t m = dx.m;
    if (m < 2) throw Error(kInvalidArgument, "distance_preservation: need at least two rows");
    // pairs exactly as the reference draws them (metrics.cpp:320-335)
    std::vector<std::int64_t> pi, pj;
    const double total = 0.5 * static_cast<double>(m) * static_cast<double>(m - 1);
    if (total <= static_cast<double>(max_pairs)) {
      for (index_t i = 0; i < m; ++i)
        for (index_t j = i + 1; j < m; ++j) {
          pi.push_back(i);
          pj.push_back(j);
        }
    } else {
      Xoshiro rng(mix64(seed ^ 0x9a17b0a155a3f2c1ULL));
      while (static_cast<index_t>(pi.size()) < max_pairs) {
        const index_t i = static_cast<index_t>(rng.next() % static_cast<std::uint64_t>(m));
        const index_t j = static_cast<index_t>(rng.next() % static_cast<std::uint64_t>(m));
        if (i == j) continue;
        pi.push_back(std::min(i, j));
        pj.push_back(std::max(i, j));
      }
    }
    const index_t np = static_cast<index_t>(pi.size());
    const index_t k = map_a->k;
    if (map_b && map_b->k != k) throw Error(kDimension, "distance_preservation: maps reduce to different k");
    double* ya = ctx->get<double>("dp.ya", m * k > 0 ? m * k : 1);
    double* yb = map_b ? ctx->get<double>("dp.yb", m * k > 0 ? m * k : 1) : nullptr;
    transform_dev(*ctx, *map_a, dx, ya, LPCA_F64, LPCA_ROW_MAJOR, LPCA_DEVICE, k, nullptr, nullptr);
    if (map_b) transform_dev(*ctx, *map_b, dx, yb, LPCA_F64, LPCA_ROW_MAJOR, LPCA_DEVICE, k, nullptr, nullptr);
    auto* dpi = ctx->get<std::int64_t>("dp.pi", np);
    auto* dpj = ctx->get<std::int64_t>("dp.pj", np);
    double* dist = ctx->get<double>("dp.d", 3 * np);
    LPCA_CUDA(cudaMemcpyAsync(dpi, pi.data(), sizeof(std::int64_t) * np, cudaMemcpyHostToDevice, ctx->stream));
    LPCA_CUDA(cudaMemcpyAsync(dpj, pj.data(), sizeof(std::int64_t) * np, cudaMemcpyHostToDevice, ctx->stream));
    launch_pair_distances(ctx->stream, dx.dtype, dx.p, dx.ld, dx.n, dx.rp, dx.ci, dx.rv, ya, yb, k, dpi, dpj, np,
                          dist, dist + np, dist + 2 * np);
    LPCA_LAUNCHED(*ctx);
    std::vector<double> hd(static_cast<std::size_t>(3 * np));
    LPCA_CUDA(cudaMemcpyAsync(hd.data(), dist, sizeof(double) * 3 * np, cudaMemcpyDeviceToHost, ctx->stream));
    LPCA_CUDA(cudaStreamSynchronize(ctx->stream));
    double worst_violation = -1e300, worst_gap = 0.0;
    for (index_t p = 0; p < np; ++p) {
      const double o = hd[p], a = hd[np + p], b = hd[2 * np + p];
      worst_violation = std::max(worst_violation, a - o);
      if (map_b) {
        worst_violation = std::max(worst_violation, b - o);
        worst_gap = std::max(worst_gap, std::abs(a - b));
      }
      if (pair_i) pair_i[p] = pi[static_cast<std::size_t>(p)];
      if (pair_j) pair_j[p] = pj[static_cast<std::size_t>(p)];
      if (original) original[p] = o;
      if (reduced_a) reduced_a[p] = a;
      if (reduced_b) reduced_b[p] = map_b ? b : 0.0;
    }
    *n_pairs = np;
    if (max_violation) *max_violation = worst_violation;
    if (max_discrepancy) *max_discrepancy = worst_gap;
  });
}

namespace {

// ---- residual norms (metrics.cpp:148-308, spectral_norm.cpp:23-57) ----------
// Linear operator on the device, seen through products (SpectralOperator,
// spectral_norm.hpp:12-17): apply maps cols -> rows, apply_t rows -> cols.
struct DevOperator {
  index_t rows = 0, cols = 0;
  std::function<void(const double*, double*)> apply, apply_t;
};

// sqrt(sum of squares) of a device vector, partials summed on the host in order.
double dev_norm2(lpca_ctx& ctx, const double* v, index_t count) {
  const index_t g = sumsq_blocks(count);
  double* part = ctx.get<double>("sn.part", g);
  launch_sumsq(ctx.stream, 8, v, count, 1, count, part);
  LPCA_LAUNCHED(ctx);
  std::vector<double> h(static_cast<std::size_t>(g));
  LPCA_CUDA(cudaMemcpyAsync(h.data(), part, sizeof(double) * g, cudaMemcpyDeviceToHost, ctx.stream));
  LPCA_CUDA(cudaStreamSynchronize(ctx.stream));
  double s = 0.0;
  for (double x : h) s += x;
  return std::sqrt(s);
}

double dev_sumsq_x(lpca_ctx& ctx, const DevX& x) {
  const index_t count = x.sparse() ? x.nnz : x.m * x.n;
  const index_t g = sumsq_blocks(count);
  double* part = ctx.get<double>("sn.xpart", g);
  if (x.sparse())
    launch_sumsq(ctx.stream, 8, x.rv, count, 1, count, part);
  else
    launch_sumsq(ctx.stream, x.dtype, x.p, x.ld, x.m, x.n, part);
  LPCA_LAUNCHED(ctx);
  std::vector<double> h(static_cast<std::size_t>(g));
  LPCA_CUDA(cudaMemcpyAsync(h.data(), part, sizeof(double) * g, cudaMemcpyDeviceToHost, ctx.stream));
  LPCA_CUDA(cudaStreamSynchronize(ctx.stream));
  double s = 0.0;
  for (double v : h) s += v;
  return s;
}

// spectral_norm (spectral_norm.cpp:23-57): power iteration on A^T A from the
// reference's seeded start vector; the iterates stay on the device, the two
// norms per step come back to the host for the same tests in the same order.
double dev_spectral_norm(lpca_ctx& ctx, const DevOperator& op, double abs_tol) {
  if (op.rows < 1 || op.cols < 1) throw Error(kInvalidArgument, "spectral_norm: operator must be non-empty");
  Xoshiro rng(0x5eed0f0e57a7ULL);
  std::vector<double> hv(static_cast<std::size_t>(op.cols));
  for (double& x : hv) x = u64_to_uniform(rng.next()) - 0.5;
  double vn = 0.0;
  for (double x : hv) vn += x * x;
  vn = std::sqrt(vn);
  if (vn == 0.0) return 0.0;
  for (double& x : hv) x /= vn;
  double* v = ctx.get<double>("sn.v", op.cols);
  double* av = ctx.get<double>("sn.av", op.rows);
  LPCA_CUDA(cudaMemcpyAsync(v, hv.data(), sizeof(double) * op.cols, cudaMemcpyHostToDevice, ctx.stream));
  constexpr int kMaxIters = 10000;
  constexpr double kRelTol = 1e-8;
  double estimate = 0.0, gap = 0.0;
  for (int it = 0; it < kMaxIters; ++it) {
    op.apply(v, av);
    const double sigma = dev_norm2(ctx, av, op.rows);
    if (sigma == 0.0) return 0.0;
    if (sigma <= abs_tol) return sigma;
    gap = std::abs(sigma - estimate);
    if (it > 0 && gap <= kRelTol * sigma + abs_tol) return sigma;
    estimate = sigma;
    op.apply_t(av, v);
    const double wn = dev_norm2(ctx, v, op.cols);
    if (wn == 0.0) return sigma;
    launch_scale_f64(ctx.stream, v, v, op.cols, 1.0 / wn);
    LPCA_LAUNCHED(ctx);
  }
  throw Error(kConvergence, "spectral_norm: estimate gap " + std::to_string(gap) + " still above relative " +
                                std::to_string(kRelTol) + " after " + std::to_string(kMaxIters) + " iterations",
              -1, gap);
}

// X v and X^T t on a staged X (dense dtype or CSR/CSC)
void x_apply(lpca_ctx& ctx, const DevX& x, const double* v, double* y) {
  launch_matvec(ctx.stream, x.dtype, x.p, x.ld, x.m, x.n, x.rp, x.ci, x.rv, v, y);
  LPCA_LAUNCHED(ctx);
}
void x_apply_t(lpca_ctx& ctx, const DevX& x, const double* t, double* y) {
  double* part = x.sparse() ? nullptr : ctx.get<double>("sn.mtpart", matvec_t_chunks(x.m, x.n) * x.n);
  launch_matvec_t(ctx.stream, x.dtype, x.p, x.ld, x.m, x.n, x.cp, x.ri, x.cv, t, part, y);
  LPCA_LAUNCHED(ctx);
}

// F (l x n, column-major) = B^T X for a row-major m x l basis (gemm_t paths of
// lpca_gemm_t); x is fp64 (widened) or sparse.
void basis_gemm_t(lpca_ctx& ctx, const DevX& x, const double* brow, index_t l, double* f) {
  if (l * x.n == 0) return;
  if (x.m > 0 && x.sparse()) {
    launch_gemm_t_csc(ctx.stream, x.n, x.cp, x.ri, x.cv, brow, l, l, f, false);
  } else if (x.m > 0) {
    launch_utx_simt<double>(ctx.stream, brow, l, static_cast<const double*>(x.p), x.ld, x.m, l, x.n,
                            round_up(x.m, 16), f, true);
  } else {
    launch_zero(ctx.stream, f, sizeof(double) * l * x.n);
  }
  LPCA_LAUNCHED(ctx);
}

double dev_sumsq(lpca_ctx& ctx, const double* a, index_t count) {
  const double r = dev_norm2(ctx, a, count);
  return r * r;
}

// sigma_{k+1} of X from the eigenvalues of its smaller Gram (the reference runs
// a one-sided Jacobi SVD on the densified X, metrics.cpp:250-256).
std::vector<double> dev_singular_values(lpca_ctx& ctx, const DevX& x) {
  const index_t m = x.m, n = x.n;
  double* dense = ctx.get<double>("rb.dense", m * n);  // row-major m x n
  if (x.sparse()) {
    launch_csr_to_dense(ctx.stream, m, n, x.rp, x.ci, x.rv, dense);
  } else {
    LPCA_CUDA(cudaMemcpy2DAsync(dense, sizeof(double) * n, x.p, sizeof(double) * x.ld, sizeof(double) * n, m,
                                cudaMemcpyDeviceToDevice, ctx.stream));
  }
  LPCA_LAUNCHED(ctx);
  const index_t w = m < n ? m : n;
  double* g = ctx.get<double>("rb.g", w * w);
  if (n <= m) {  // X^T X: the row-major X is an n x m column-major F
    launch_gram_fast(ctx.stream, dense, n, m, g, ctx.get<double>("rb.gpart", gram_fast_chunks(n, m) * n * n));
  } else {  // X X^T: transpose to an m x n column-major F first
    double* xt = ctx.get<double>("rb.xt", m * n);
    launch_transpose(ctx.stream, 8, dense, n, n, m, xt, m);
    launch_gram_fast(ctx.stream, xt, m, n, g, ctx.get<double>("rb.gpart", gram_fast_chunks(m, n) * m * m));
  }
  LPCA_LAUNCHED(ctx);
  double* evals = ctx.get<double>("rb.evals", w);
  double* evecs = ctx.get<double>("rb.evecs", w * w);
  int* st = ctx.get<int>("rb.st", 2);
  double* gap = ctx.get<double>("rb.gap", 1);
  eigh_dev(ctx, g, w, evals, evecs, st, gap, 0);
  std::vector<double> lam(static_cast<std::size_t>(w));
  LPCA_CUDA(cudaMemcpyAsync(lam.data(), evals, sizeof(double) * w, cudaMemcpyDeviceToHost, ctx.stream));
  LPCA_CUDA(cudaStreamSynchronize(ctx.stream));
  for (double& v : lam) v = std::sqrt(v > 0.0 ? v : 0.0);
  return lam;
}

double bound_value_host(index_t m, index_t n, index_t k, index_t l, double sigma) {
  if (k < 1 || l < k + 2)
    throw Error(kInvalidArgument, "bound_value: needs l >= k + 2 (got k = " + S(k) + ", l = " + S(l) + ")");
  const double minmn = static_cast<double>(m < n ? m : n);
  const double factor = 1.0 + 4.0 * std::sqrt(static_cast<double>(l)) / static_cast<double>(l - k - 1) * std::sqrt(minmn);
  return factor * sigma;
}

void fill_report(lpca_recon_report* out, double spectral, double frob) {
  *out = lpca_recon_report{};
  out->spectral_error = spectral;
  out->frobenius_error = frob;
}

}  // namespace

lpca_status lpca_reconstruction_error(lpca_ctx* ctx, const lpca_matrix_view* x, const double* u, int64_t u_rows,
                                      int64_t u_cols, int32_t u_location, int32_t route, int64_t k, int64_t l,
                                      int32_t with_bound, int64_t densify_limit, lpca_recon_report* out) {
  return guarded([&] {
    check_ctx(ctx);
    if (!out || (!u && u_rows * u_cols > 0)) throw Error(kInvalidArgument, "null argument");
    if (route != LPCA_ROUTE_QR && route != LPCA_ROUTE_LAZY)
      throw Error(kInvalidArgument, "reconstruction_error: route must be LPCA_ROUTE_QR or LPCA_ROUTE_LAZY");
    const DevX dx = stage_x_f64(*ctx, x);
    const index_t m = dx.m, n = dx.n;
    if (u_rows != m)
      throw Error(kDimension, "reconstruction_error: U has " + S(u_rows) + " rows but X has " + S(m));
    if (u_cols != l) throw Error(kDimension, "reconstruction_error: U has " + S(u_cols) + " columns but l = " + S(l));
    lpca_ctx& c = *ctx;
    const double* ud = stage_f64(c, u, m * l, u_location, "re.u");
    const double xf2 = dev_sumsq_x(c, dx);
    double* urow = c.get<double>("re.urow", m * l);  // row-major m x l (an l x m column-major F)
    if (m * l > 0) {
      launch_transpose(c.stream, 8, ud, m, m, l, urow, l);
      LPCA_LAUNCHED(c);
    }
    double* f = c.get<double>("re.f", l * n);
    double* rinv = nullptr;
    const double* basis = ud;  // column-major m x l: U (lazy) or Q (qr)
    if (route == LPCA_ROUTE_QR) {
      orth_rows(c, urow, l, m);  // Q (row-major) = shifted CholeskyQR3 of U
      double* qcol = c.get<double>("re.q", m * l);
      if (m * l > 0) {
        launch_transpose(c.stream, 8, urow, l, l, m, qcol, m);
        LPCA_LAUNCHED(c);
      }
      basis = qcol;
      basis_gemm_t(c, dx, urow, l, f);  // Q^T X
    } else {
      double* g = c.get<double>("re.g", l * l);
      launch_gram_fast(c.stream, urow, l, m, g, c.get<double>("gram.part", gram_fast_chunks(l, m) * l * l));
      LPCA_LAUNCHED(c);
      rinv = c.get<double>("re.rinv", l * l);
      int* st = c.get<int>("re.st", 1);
      launch_chol_inverse(c.stream, g, l, rinv, c.get<double>("re.lm", l * l), st);
      LPCA_LAUNCHED(c);
      int h = 0;
      LPCA_CUDA(cudaMemcpyAsync(&h, st, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
      LPCA_CUDA(cudaStreamSynchronize(c.stream));
      if (h != 0)
        throw Error(kRankDeficiency, "cholesky: pivot " + S(h - 1) + " is not positive definite", h - 1);
      basis_gemm_t(c, dx, urow, l, f);                                       // U^T X
      launch_apply_rinv_t(c.stream, rinv, l, f, n, c.get<double>("re.tmp", l * n));  // L^{-1} U^T X
      LPCA_LAUNCHED(c);
    }
    const double pf2 = dev_sumsq(c, f, l * n);
    const double frob = std::sqrt(std::max(0.0, xf2 - pf2));
    // residual operator (I - P) X and its transpose
    double* t = c.get<double>("re.t", m);
    double* sv = c.get<double>("re.s", l > 0 ? l : 1);
    double* s2 = c.get<double>("re.s2", l > 0 ? l : 1);
    double* stmp = c.get<double>("re.stmp", l > 0 ? l : 1);
    double* bpart = c.get<double>("re.bpart", basis_t_chunks(m) * (l > 0 ? l : 1));
    auto project_out = [&](const double* in, double* y) {  // y = in - P in (m-vectors)
      launch_basis_t(c.stream, basis, m, m, l, in, bpart, sv);
      LPCA_LAUNCHED(c);
      const double* coef = sv;
      if (rinv) {
        launch_chol_solve(c.stream, rinv, l, sv, stmp, s2);
        LPCA_LAUNCHED(c);
        coef = s2;
      }
      launch_basis_sub(c.stream, basis, m, m, l, coef, in, y);
      LPCA_LAUNCHED(c);
    };
    DevOperator op;
    op.rows = m;
    op.cols = n;
    op.apply = [&](const double* in, double* y) {
      x_apply(c, dx, in, t);
      project_out(t, y);
    };
    op.apply_t = [&](const double* in, double* y) {
      project_out(in, t);
      x_apply_t(c, dx, t, y);
    };
    const double spectral = dev_spectral_norm(c, op, 1e-14 * std::sqrt(xf2));
    fill_report(out, spectral, frob);
    if (with_bound && l >= k + 2 && std::max(m, n) <= densify_limit && m > 0 && n > 0) {
      const std::vector<double> sv_x = dev_singular_values(c, dx);
      if (static_cast<index_t>(sv_x.size()) > k && k >= 0) {
        out->has_sigma_k_plus_1 = 1;
        out->sigma_k_plus_1 = sv_x[static_cast<std::size_t>(k)];
        out->has_bound = 1;
        out->bound = bound_value_host(m, n, k, l, out->sigma_k_plus_1);
      }
    }
  });
}

lpca_status lpca_row_space_reconstruction_error(lpca_ctx* ctx, const lpca_matrix_view* x, const double* v,
                                                int64_t v_rows, int64_t v_cols, int32_t v_location,
                                                lpca_recon_report* out) {
  return guarded([&] {
    check_ctx(ctx);
    if (!out || (!v && v_rows * v_cols > 0)) throw Error(kInvalidArgument, "null argument");
    const DevX dx = stage_x_f64(*ctx, x);
    const index_t m = dx.m, n = dx.n, kd = v_cols;
    if (n != v_rows)
      throw Error(kDimension, "row_space_reconstruction_error: X has " + S(n) + " columns but V has " + S(v_rows) +
                                  " rows");
    lpca_ctx& c = *ctx;
    const double* vd = stage_f64(c, v, n * kd, v_location, "rs.v");
    // check_orthonormal (metrics.cpp:21-31) on V^T V
    double* g = c.get<double>("rs.g", kd * kd > 0 ? kd * kd : 1);
    launch_atb(c.stream, vd, n, kd, vd, kd, g);
    LPCA_LAUNCHED(c);
    std::vector<double> hg(static_cast<std::size_t>(kd * kd));
    if (!hg.empty()) LPCA_CUDA(cudaMemcpyAsync(hg.data(), g, sizeof(double) * hg.size(), cudaMemcpyDeviceToHost, c.stream));
    LPCA_CUDA(cudaStreamSynchronize(c.stream));
    double worst = 0.0;
    for (index_t j = 0; j < kd; ++j)
      for (index_t i = 0; i < kd; ++i)
        worst = std::max(worst, std::abs(hg[static_cast<std::size_t>(j * kd + i)] - (i == j ? 1.0 : 0.0)));
    if (worst > 1e-8 * static_cast<double>(std::max<index_t>(1, kd)))
      throw Error(kInvalidArgument,
                  "chordal_distance: basis does not have orthonormal columns (max deviation " + std::to_string(worst) + ")");
    const double xf2 = dev_sumsq_x(c, dx);
    // ||X V||_F^2
    double* xv = c.get<double>("rs.xv", m * kd > 0 ? m * kd : 1);
    if (m > 0 && kd > 0) {
      if (dx.sparse()) {
        double* wt = c.get<double>("rs.vrows", n * kd);
        launch_transpose(c.stream, 8, vd, n, n, kd, wt, kd);
        launch_spmm_csr(c.stream, m, dx.rp, dx.ci, dx.rv, wt, kd, kd, xv, 8, 1, m);
      } else {
        launch_xw_simt<double, double>(c.stream, static_cast<const double*>(dx.p), m, n, dx.ld, vd, kd, n, xv, 1, m, true);
      }
      LPCA_LAUNCHED(c);
    }
    const double frob = std::sqrt(std::max(0.0, xf2 - dev_sumsq(c, xv, m * kd)));
    double* w = c.get<double>("rs.w", n);
    double* sv = c.get<double>("rs.s", kd > 0 ? kd : 1);
    double* bpart = c.get<double>("rs.bpart", basis_t_chunks(n) * (kd > 0 ? kd : 1));
    auto project_out = [&](const double* in, double* y) {  // y = in - V V^T in (n-vectors)
      launch_basis_t(c.stream, vd, n, n, kd, in, bpart, sv);
      LPCA_LAUNCHED(c);
      launch_basis_sub(c.stream, vd, n, n, kd, sv, in, y);
      LPCA_LAUNCHED(c);
    };
    DevOperator op;
    op.rows = m;
    op.cols = n;
    op.apply = [&](const double* in, double* y) {
      project_out(in, w);
      x_apply(c, dx, w, y);
    };
    op.apply_t = [&](const double* in, double* y) {
      x_apply_t(c, dx, in, w);
      project_out(w, y);
    };
    fill_report(out, dev_spectral_norm(c, op, 1e-14 * std::sqrt(xf2)), frob);
  });
}

lpca_status lpca_spectral_norm(lpca_ctx* ctx, const lpca_matrix_view* x, double* out) {
  return guarded([&] {
    check_ctx(ctx);
    if (!out) throw Error(kInvalidArgument, "null argument");
    const DevX dx = stage_x_f64(*ctx, x);
    DevOperator op;
    op.rows = dx.m;
    op.cols = dx.n;
    op.apply = [&](const double* in, double* y) { x_apply(*ctx, dx, in, y); };
    op.apply_t = [&](const double* in, double* y) { x_apply_t(*ctx, dx, in, y); };
    *out = dev_spectral_norm(*ctx, op, 0.0);
  });
}

lpca_status lpca_bound_value(int64_t m, int64_t n, int64_t k, int64_t l, double sigma_k_plus_1, double* out) {
  return guarded([&] {
    if (!out) throw Error(kInvalidArgument, "null argument");
    *out = bound_value_host(m, n, k, l, sigma_k_plus_1);
  });
}

lpca_status lpca_dense_aat(lpca_ctx* ctx, const double* f, int64_t l, int64_t n, int32_t location,
                           double* out) {
  return guarded([&] {
    check_ctx(ctx);
    const double* fd = stage_f64(*ctx, f, l * n, location, "k.f");
    double* od = location == LPCA_DEVICE ? out : ctx->get<double>("k.out", l * l);
    if (l > 0) {
      launch_gram(ctx->stream, fd, l, n, od);
      LPCA_LAUNCHED(*ctx);
    }
    finish_out(*ctx, out, od, l * l, location);
  });
}

static lpca_status eigh_impl(lpca_ctx* ctx, const double* a, int64_t l, int32_t location, double* evals,
                             double* evecs, int method);

lpca_status lpca_eigh(lpca_ctx* ctx, const double* a, int64_t l, int32_t location, double* evals,
                      double* evecs) {
  return eigh_impl(ctx, a, l, location, evals, evecs, 0);
}

lpca_status lpca_eigh_jacobi(lpca_ctx* ctx, const double* a, int64_t l, int32_t location, double* evals,
                             double* evecs) {
  return eigh_impl(ctx, a, l, location, evals, evecs, 1);
}

lpca_status lpca_ctx_set_eigensolver(lpca_ctx* ctx, int32_t method) {
  return guarded([&] {
    check_ctx(ctx);
    if (method != 0 && method != 1) throw Error(kInvalidArgument, "eigensolver must be 0 (tridiagonal) or 1 (jacobi)");
    ctx->eigensolver = method;
  });
}

static lpca_status eigh_impl(lpca_ctx* ctx, const double* a, int64_t l, int32_t location, double* evals,
                             double* evecs, int method) {
  return guarded([&] {
    check_ctx(ctx);
    if (l < 0) throw Error(kDimension, "eigh: negative size");
    if (l == 0) return;
    const double* ad = stage_f64(*ctx, a, l * l, location, "k.a");
    double* acopy = ctx->get<double>("k.acopy", l * l);
    LPCA_CUDA(cudaMemcpyAsync(acopy, ad, sizeof(double) * l * l, cudaMemcpyDeviceToDevice, ctx->stream));
    double* ev = ctx->get<double>("k.evals", l);
    double* vec = location == LPCA_DEVICE ? evecs : ctx->get<double>("k.evecs", l * l);
    int* st = ctx->get<int>("k.status", 2);
    double* gap = ctx->get<double>("k.gap", 1);
    eigh_dev(*ctx, acopy, l, ev, vec, st, gap, method);
    int hst = 0;
    double hgap = 0;
    LPCA_CUDA(cudaMemcpyAsync(&hst, st, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    LPCA_CUDA(cudaMemcpyAsync(&hgap, gap, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    LPCA_CUDA(cudaMemcpyAsync(evals, ev, sizeof(double) * l,
                              location == LPCA_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                              ctx->stream));
    finish_out(*ctx, evecs, vec, l * l, location);
    if (hst == 2)
      throw Error(kInvalidArgument, "eigh: input is not symmetric (max |a_ij - a_ji| = " + std::to_string(hgap) + ")");
    if (hst == 1)
      throw Error(kConvergence, "eigh: Jacobi did not converge in 50 sweeps", -1, hgap);
  });
}

lpca_status lpca_truncated_svd_via_gram(lpca_ctx* ctx, const double* f, int64_t l, int64_t n,
                                        int64_t k, int32_t location, double* sigma, double* v,
                                        double* u_tilde) {
  return guarded([&] {
    check_ctx(ctx);
    const double* fd = stage_f64(*ctx, f, l * n, location, "k.f");
    double* vd = location == LPCA_DEVICE ? v : ctx->get<double>("k.v", n * (k > 0 ? k : 1));
    double* ud = nullptr;
    if (u_tilde) ud = location == LPCA_DEVICE ? u_tilde : ctx->get<double>("k.ut", l * (k > 0 ? k : 1));
    std::vector<double> sg;
    finish_spectral(*ctx, fd, l, n, k, vd, sg, ud);
    std::copy(sg.begin(), sg.end(), sigma);
    finish_out(*ctx, v, vd, n * k, location);
    if (u_tilde) finish_out(*ctx, u_tilde, ud, l * k, location);
  });
}

lpca_status lpca_sketch_f32(lpca_ctx* ctx, const lpca_matrix_view* x, const double* w_dev,
                            int64_t w_cols, float* out_dev, int64_t ldo) {
  return guarded([&] {
    check_ctx(ctx);
    const DevX d = stage_x(*ctx, x, "kx", nullptr);
    if (d.dtype != 4) throw Error(kInvalidArgument, "sketch_f32: X must be fp32");
    if (ldo < w_cols) throw Error(kInvalidArgument, "sketch_f32: ldo < w_cols");
    Panel out;
    out.plain = out_dev;
    out.ld = ldo;
    if (use_tc(*ctx, d, w_cols) && ldo % 4 == 0) {
      // the fit's layout: hi/lo planes at ld round_up(w, 16) plus the plain output
      const index_t ld = round_up(w_cols, 16);
      const index_t wpad = ld;
      float* hi = ctx->get<float>("w.hi", wpad * d.n);
      float* lo = ctx->get<float>("w.lo", wpad * d.n);
      launch_split_tf32_w(ctx->stream, w_dev, d.n, d.n, w_cols, wpad, hi, lo, d.n);
      LPCA_LAUNCHED(*ctx);
      const index_t ldt = planes_ld(d.m);
      float* uh = ctx->get<float>("k.uh", ld * ldt);
      float* ul = ctx->get<float>("k.ul", ld * ldt);
      launch_xw_tc_planes(ctx->stream, static_cast<const float*>(d.p), d.m, d.n, d.ld, hi, lo, wpad, d.n,
                          out_dev, ldo, w_cols, uh, ul, ldt, ctx->num_sms);
      LPCA_LAUNCHED(*ctx);
    } else {
      xw_pass(*ctx, d, w_dev, w_cols, d.n, out, false);
    }
    LPCA_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

lpca_status lpca_gemm_t_f32(lpca_ctx* ctx, const float* u_dev, int64_t ldu, int64_t l,
                            const lpca_matrix_view* x, double* f_dev) {
  return guarded([&] {
    check_ctx(ctx);
    const DevX d = stage_x(*ctx, x, "kx", nullptr);
    if (d.dtype != 4) throw Error(kInvalidArgument, "gemm_t_f32: X must be fp32");
    Panel u;
    u.plain = const_cast<float*>(u_dev);
    u.ld = ldu;
    if (ctx->gemm_path == 0 && tc_utx_supported(l, d.n) && ldu % 4 == 0 && d.ld % 4 == 0) {
      u.ldt = planes_ld(d.m);
      u.hi = ctx->get<float>("k.uh", round_up(l, 16) * u.ldt);
      u.lo = ctx->get<float>("k.ul", round_up(l, 16) * u.ldt);
      launch_zero(ctx->stream, u.hi, sizeof(float) * round_up(l, 16) * u.ldt);
      launch_zero(ctx->stream, u.lo, sizeof(float) * round_up(l, 16) * u.ldt);
      if (d.m > 0) {
        launch_split_tf32_transpose(ctx->stream, u_dev, d.m, l, ldu, u.hi, u.lo, u.ldt);
        LPCA_LAUNCHED(*ctx);
      }
    }
    const int world = ctx->world;
    ctx->world = 1;  // kernel-level: this rank's rows only
    try {
      utx_pass(*ctx, d, u, l, f_dev, false);
    } catch (...) {
      ctx->world = world;
      throw;
    }
    ctx->world = world;
    LPCA_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

lpca_status lpca_synth_lowrank(lpca_ctx* ctx, int64_t row0, int64_t m, int64_t n, int64_t r,
                               double rho, double noise, uint64_t seed, int32_t dtype, void* x_dev,
                               int64_t ldx) {
  return guarded([&] {
    check_ctx(ctx);
    if (dtype != 4 && dtype != 8) throw Error(kInvalidArgument, "synth: dtype must be 4 or 8");
    if (m < 0 || n < 1 || r < 1) throw Error(kInvalidArgument, "synth: bad shape");
    if (ldx <= 0) ldx = n;
    std::vector<double> sig(static_cast<std::size_t>(r));
    double s = 1.0;
    for (index_t t = 0; t < r; ++t) {  // sigma_t = rho^t, t = 0..r-1 (sigma_0 = 1)
      sig[static_cast<std::size_t>(t)] = s;
      s *= rho;
    }
    double* sd = ctx->get<double>("synth.sigma", r);
    LPCA_CUDA(cudaMemcpyAsync(sd, sig.data(), sizeof(double) * r, cudaMemcpyHostToDevice, ctx->stream));
    const index_t batch = std::min<index_t>(m > 0 ? m : 1, 262144);
    const index_t scratch = r * n + batch * r;
    double* sc = ctx->get<double>("synth.scratch", scratch);
    if (m > 0) {
      launch_synth_lowrank(ctx->stream, row0, m, n, r, sd, noise, seed, dtype, x_dev, ldx, sc, scratch);
      LPCA_LAUNCHED(*ctx);
    }
    LPCA_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

}  // extern "C"
