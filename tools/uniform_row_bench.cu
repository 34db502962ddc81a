#include <cstdio>
#include <climits>
#include <cuda_runtime.h>
constexpr int D = 8, T = 128, NS = 512;
__constant__ double2 crow[NS];
template <int SRC, int KEYSV, int G = 1, bool LAG = false>
__global__ void __launch_bounds__(T, 4) k(int* out, const double2* in, int reps) {
  constexpr int KEYS = KEYSV % 100; constexpr bool VOTE = KEYSV >= 100;
  __shared__ double2 col[(NS + T * D + 2 * D) * 9 / 8 + 8];
  __shared__ double2 row[NS];
  for (int i = threadIdx.x; i < (NS + T * D + 2 * D) * 9 / 8 + 8; i += T) col[i] = in[i % 4096];
  for (int i = threadIdx.x; i < NS; i += T) row[i] = in[(i * 7) % 4096];
  __syncthreads();
  double acc[D]; double2 c[D];
  const int xb = threadIdx.x * D;
#pragma unroll
  for (int d = 0; d < D; ++d) { acc[d] = 0.0; c[d] = col[(xb + d) + (xb + d) / D]; }
  int hm = INT_MIN;
  for (int r = 0; r < reps; ++r) {
    int hg = INT_MIN; bool prevhit = false;
#pragma unroll G
    for (int s = 0; s < NS; s += D) {
      int hb = INT_MIN; float hf = -1e30f; unsigned long long hp = 0x8000000080000000ull;
#pragma unroll
      for (int u = 0; u < D; ++u) {
        const double2 rr = SRC == 0 ? row[s + u] : crow[s + u];
#pragma unroll
        for (int d = 0; d < D; ++d) {
          const double2 cc = c[(d + u) % D];
          acc[d] = fma(rr.y, cc.x, fma(rr.x, cc.y, acc[d]));
          if (KEYS == 1 || KEYS == 5 || ((KEYS == 2 || KEYS == 6) && (u == 3 || u == 7)) || ((KEYS == 8 || KEYS == 9) && u == 7)) hb = max(hb, __double2hiint(acc[d]));
          if (KEYS == 3) hf = fmaxf(hf, __int_as_float(__double2hiint(acc[d])));
          if (KEYS == 4) { unsigned long long w = hp; int lo = (int)(unsigned)w; lo = max(lo, __double2hiint(acc[d])); hp = (w & 0xffffffff00000000ull) | (unsigned)lo; }
        }
        const int x = s + xb + D + u; c[u] = col[x + x / D];
      }
      hm = max(hm, hb);
      if (KEYS == 3) hb = __float_as_int(hf);
      if (KEYS == 4) hb = (int)(unsigned)hp;
      if (KEYS == 7) hb = __double2hiint(acc[0]);
      hg = max(hg, hb - 0x100 * (s & 7));   // stand-in for a per-block threshold
      if (KEYS && KEYS != 5 && KEYS != 6 && KEYS != 9 && ((s / D) % G) == G - 1) { if (LAG) { if (prevhit) out[1] = s; prevhit = hg >= 0x7ff00000; } else if (VOTE ? __any_sync(0xffffffffu, hg >= 0x7ff00000) : (hg >= 0x7ff00000)) out[1] = s; hg = INT_MIN; }   // block hit test + branch, never taken
    }
  }
  int s = hm;
#pragma unroll
  for (int d = 0; d < D; ++d) s ^= __double2hiint(acc[d]);
  if (s == 12345) out[0] = s;
}
template <int SRC, int KEYS, int G = 1, bool LAG = false>
void run(const char* name, int* out, const double2* in) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 4 * 8, reps = 256;
  k<SRC, KEYS, G, LAG><<<blocks, T>>>(out, in, 1);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<SRC, KEYS, G, LAG><<<blocks, T>>>(out, in, reps);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double cells = (double)blocks * T * D * NS * reps;
  printf("%-28s %8.3f ms  %6.3f Tcells/s  FP64 pipe %5.1f%%  err=%s\n", name, ms, cells / (ms * 1e-3) / 1e12,
         100.0 * cells * 2.0 / (ms * 1e-3) / (sms * 64 * 1.965e9), cudaGetErrorString(cudaGetLastError()));
}
int main() {
  int* out; double2* in;
  cudaMalloc(&out, 8); cudaMalloc(&in, 4096 * 16); cudaMemset(in, 0, 4096 * 16);
  double2 h[NS]; for (int i = 0; i < NS; ++i) h[i] = make_double2(1e-3 * i, 2e-3 * i);
  cudaMemcpyToSymbol(crow, h, sizeof(h));
  for (int rep = 0; rep < 1; ++rep) {
  run<0, 1, 1>("smem keys G1", out, in);
  run<0, 5, 1>("smem keys nobranch", out, in);
  run<0, 1, 1, true>("smem keys G1 lag", out, in);
  run<0, 1, 2, true>("smem keys G2 lag", out, in);
  run<1, 5, 1>("const keys nobranch", out, in);
  run<1, 1, 1, true>("const keys G1 lag", out, in);
  run<1, 1, 2, true>("const keys G2 lag", out, in);
  run<1, 2, 1, true>("const keys@3,7 G1 lag", out, in);
  run<0, 101, 8>("smem keys G8 vote", out, in);
  run<1, 101, 8>("const keys G8 vote", out, in);
  run<1, 101, 2>("const keys G2 vote", out, in);
  run<1, 101, 1>("const keys G1 vote", out, in);
  run<0, 102, 8>("smem keys@3,7 G8 vote", out, in);
  run<1, 102, 8>("const keys@3,7 G8 vote", out, in);
  run<1, 108, 8>("const keys@7 G8 vote", out, in);
  run<0, 0, 1>("smem nokeys", out, in);
  run<1, 0, 1>("const nokeys", out, in);
  run<0, 1, 8>("smem keys G8", out, in);
  run<1, 1, 8>("const keys G8", out, in);
  run<0, 2, 8>("smem keys@3,7 G8", out, in);
  run<1, 2, 8>("const keys@3,7 G8", out, in);
  run<0, 6, 1>("smem keys@3,7 nobranch", out, in);
  run<1, 6, 1>("const keys@3,7 nobranch", out, in);
  run<0, 8, 8>("smem keys@7 G8", out, in);
  run<1, 8, 8>("const keys@7 G8", out, in);
  run<0, 9, 1>("smem keys@7 nobranch", out, in);
  run<1, 9, 1>("const keys@7 nobranch", out, in);
  }
  return 0;
}
