// Shared device/host helpers for the lazypca_b200 kernels (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <stdexcept>
#include <string>

namespace lpca {

using index_t = std::int64_t;

// Host-side exception mirroring the reference hierarchy
// (proj/core/include/lazypca/error.hpp:10-58) plus device/collective failures.
struct Error : std::runtime_error {
  int code;
  std::int64_t index;
  double gap;
  Error(int c, const std::string& what, std::int64_t idx = -1, double g = 0.0)
      : std::runtime_error(what), code(c), index(idx), gap(g) {}
};

enum Code : int {
  kOk = 0,
  kDimension = 1,
  kInvalidArgument = 2,
  kRankDeficiency = 3,
  kConvergence = 4,
  kParse = 5,
  kCuda = 6,
  kNccl = 7,
  kInternal = 9,
};

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess)
    throw Error(kCuda, std::string(what) + ": " + cudaGetErrorString(e) + " (" + file + ":" +
                           std::to_string(line) + ")");
}
#define LPCA_CUDA(x) ::lpca::cuda_check((x), #x, __FILE__, __LINE__)
#define LPCA_LAUNCHED(ctx) \
  do {                      \
    (ctx).note_launch();    \
    LPCA_CUDA(cudaGetLastError()); \
  } while (0)

// Sets the thread's lpca_last_error* state (defined in lpca.cu).
void set_last_error(const std::string& msg, std::int64_t index, double gap);
// An error raised inside a block callback (lpca_file_stream_next), rethrown by
// the streaming reducer that called it (per thread).
void set_callback_error(const Error& e);
bool take_callback_error(Error* out);

inline index_t ceil_div(index_t a, index_t b) { return (a + b - 1) / b; }
inline index_t round_up(index_t a, index_t b) { return ceil_div(a, b) * b; }

}  // namespace lpca
