// Instantiation of the greedy search kernel for P = 1 lanes per destination row
// (one translation unit per P so the variants compile in parallel).
#include "greedy_kernel.cuh"

namespace tacos {
int launch_greedy_p1(const Layout &lay, uint32_t V, const Job *d_jobs, uint32_t n_jobs, JobOut *d_outs,
                      cudaStream_t st) {
  return launch_greedy_p<1>(lay, V, d_jobs, n_jobs, d_outs, st);
}
}  // namespace tacos
