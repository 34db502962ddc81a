// Microbenchmark: ceiling of the AAMP / ACAMP inner loop instruction mix on one B200 (no stages,
// barriers, filter or merges): D=8 accumulators per thread, a register ring of D column operands
// refilled from shared memory (one 16-byte operand per sub-step), the row operand broadcast from
// shared memory, and the per-cell 32-bit key min. Experiments only.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/inner_loop_bench.cu -o /tmp/ilb
#include <cstdio>
#include <climits>
#include <cuda_runtime.h>

constexpr int D = 8, T = 128, NS = 512;

template <int MODE, bool KEYS, bool LOADS>
__global__ void __launch_bounds__(T, 4) k(int* out, const double2* in, int reps) {
  __shared__ double2 col[(NS + T * D + 2 * D) * 9 / 8 + 8];  // padded x -> x + x/D (conflict-free)
  __shared__ double2 row[NS];
  for (int i = threadIdx.x; i < (NS + T * D + 2 * D) * 9 / 8 + 8; i += T) col[i] = in[i % 4096];
  for (int i = threadIdx.x; i < NS; i += T) row[i] = in[(i * 7) % 4096];
  __syncthreads();
  double acc[D];
  double2 c[D];
  const int xb = threadIdx.x * D;
#pragma unroll
  for (int d = 0; d < D; ++d) { acc[d] = 0.0; c[d] = col[(xb + d) + (xb + d) / D]; }
  int hmin = INT_MAX;
  for (int r = 0; r < reps; ++r) {
    for (int s = 0; s < NS; s += D) {
      int hb = INT_MAX;
#pragma unroll
      for (int u = 0; u < D; ++u) {
        const double2 rr = LOADS ? row[s + u] : make_double2(1.0 + u, 2.0 + u);
#pragma unroll
        for (int d = 0; d < D; ++d) {
          const double2 cc = c[(d + u) % D];
          if (MODE == 0) acc[d] = fma(rr.x - cc.x, rr.y - cc.y, acc[d]);              // AAMP
          else acc[d] = fma(rr.y, cc.x, fma(rr.x, cc.y, acc[d]));                      // ACAMP
          if (KEYS) hb = min(hb, __double2hiint(acc[d]));
        }
        if (LOADS) { const int x = s + xb + D + u; c[u] = col[x + x / D]; }
        else { c[u].x += 1e-300; }
      }
      hmin = min(hmin, hb);
    }
  }
  int s = hmin;
#pragma unroll
  for (int d = 0; d < D; ++d) s ^= __double2hiint(acc[d]);
  if (s == 12345) out[0] = s;
}

template <int MODE, bool KEYS, bool LOADS>
void run(const char* name, int* out, const double2* in) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 4 * 8, reps = 256;
  k<MODE, KEYS, LOADS><<<blocks, T>>>(out, in, 1);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<MODE, KEYS, LOADS><<<blocks, T>>>(out, in, reps);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double cells = (double)blocks * T * D * NS * reps;
  const double ops = MODE == 0 ? 3.0 : 2.0;
  printf("%-28s %8.3f ms  %6.3f Tcells/s  FP64 pipe %5.1f%%\n", name, ms, cells / (ms * 1e-3) / 1e12,
         100.0 * cells * ops / (ms * 1e-3) / (sms * 64 * 1.965e9));
}

int main() {
  int* out; double2* in;
  cudaMalloc(&out, 8); cudaMalloc(&in, 4096 * 16); cudaMemset(in, 0, 4096 * 16);
  run<0, true, true>("AAMP keys+loads", out, in);
  run<0, false, true>("AAMP loads", out, in);
  run<0, true, false>("AAMP keys", out, in);
  run<0, false, false>("AAMP bare", out, in);
  run<1, true, true>("ACAMP keys+loads", out, in);
  run<1, false, true>("ACAMP loads", out, in);
  run<1, false, false>("ACAMP bare", out, in);
  return 0;
}
