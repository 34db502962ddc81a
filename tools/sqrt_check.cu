#include <cstdio>
#include <cmath>
__global__ void k(const double* in, double* out, int n, int mode) {
  int i = blockIdx.x * blockDim.x + threadIdx.x; if (i >= n) return;
  double a = in[i], y;
  const bool sub = a < 0x1p-1022;
  const double as = sub ? a * 0x1p108 : a;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(as));
  double h = 0.5 * as;
  y = y * fma(-h * y, y, 1.5);
  if (mode == 2) y = y * fma(-h * y, y, 1.5);
  const double r = as * y;
  out[i] = sub ? (a > 0.0 ? r * 0x1p-54 : 0.0) : r;
}
int main() {
  const int n = 1 << 20; double *h = new double[n], *o = new double[n];
  for (int i = 0; i < n; ++i) h[i] = exp(-300.0 + 600.0 * (i + 0.5) / n) * (1.0 + 0.37 * sin(i));
  h[0] = 0; h[1] = 1e-310; h[2] = 4.9e-324;
  double *di, *dout; cudaMalloc(&di, n * 8); cudaMalloc(&dout, n * 8);
  cudaMemcpy(di, h, n * 8, cudaMemcpyHostToDevice);
  for (int mode = 2; mode <= 3; ++mode) {
    k<<<n / 256, 256>>>(di, dout, n, mode); cudaMemcpy(o, dout, n * 8, cudaMemcpyDeviceToHost);
    printf("denormals: %g (want %g) %g (want %g)\n", o[1], sqrt(1e-310), o[2], sqrt(4.9e-324));
    double worst = 0; for (int i = 3; i < n; ++i) { double r = sqrt(h[i]); worst = fmax(worst, fabs(o[i] - r) / r); }
    printf("mode %d worst rel err %.3e  o[0]=%g o[1]=%g\n", mode, worst, o[0], o[1]);
  }
}
