// Phase timing of the register tridiagonalisation (clock64 per warp):
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DLPCA_TRI_PROF -Ipaper_1709_07175_b200/csrc
//      tools/tri_prof.cu -o tools/tri_prof && tools/tri_prof [l]
#include "../paper_1709_07175_b200/csrc/eigh.cu"

#include <cstdio>
#include <cstdlib>
#include <vector>

namespace lpca {
void set_last_error(const std::string&, std::int64_t, double) {}
}

int main(int argc, char** argv) {
  const int l = argc > 1 ? std::atoi(argv[1]) : 110;
  std::vector<double> a(static_cast<size_t>(l) * l);
  unsigned s = 1;
  for (int j = 0; j < l; ++j)
    for (int i = 0; i <= j; ++i) {
      s = s * 1664525u + 1013904223u;
      const double v = (s >> 8) * (1.0 / 16777216.0) - 0.5;
      a[static_cast<size_t>(j) * l + i] = a[static_cast<size_t>(i) * l + j] = v;
    }
  double *da, *ev, *vec, *gap;
  int* st;
  void* work;
  cudaMalloc(&da, sizeof(double) * l * l);
  cudaMalloc(&ev, sizeof(double) * l);
  cudaMalloc(&vec, sizeof(double) * l * l);
  cudaMalloc(&gap, sizeof(double));
  cudaMalloc(&st, 2 * sizeof(int));
  cudaMalloc(&work, lpca::eigh_tridiag_workspace(l));
  cudaMemcpy(da, a.data(), sizeof(double) * l * l, cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 3; ++rep) lpca::launch_eigh_tridiag(0, da, l, ev, vec, work, st, gap);
  cudaDeviceSynchronize();
  long long prof[17][8];
  cudaMemcpyFromSymbol(prof, lpca::g_tri_prof, sizeof(prof));
  const char* names[] = {"wait1", "matvec", "wait2", "update/build"};
  std::printf("l=%d, cycles per step (avg over %d steps)\n", l, l - 1);
  for (int w = 0; w < 17; ++w) {
    std::printf("warp %d:", w);
    long long tot = 0;
    for (int k = 0; k < 4; ++k) {
      std::printf(" %s %6.0f", names[k], double(prof[w][k]) / (l - 1));
      tot += prof[w][k];
    }
    std::printf("  | total %6.0f\n", double(tot) / (l - 1));
  }
  return 0;
}
