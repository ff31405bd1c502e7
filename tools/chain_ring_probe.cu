// Probe (not part of the library): cycles per step of one dependent fp64 FMA chain per thread
// with operands streamed from shared memory through a register ring (router_ws_kernel's loop).
// 32-thread CTAs (2 tokens x 16 experts), one CTA per SM, chunk of L steps repeated `reps` times.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 chain_ring_probe.cu -o chain_ring_probe
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N4 = 16, TPC = 2, L = 128, LP = L + 2;  // padded expert-major row

template <int V>
__global__ void __launch_bounds__(32, 1) chain(const double* gx, const double* gw, double* out, long long* cyc,
                                               int reps, int n4_rt) {
  __shared__ __align__(16) double sx[TPC * (L + 16)];
  __shared__ __align__(16) double sw[(L + 16) * N4];  // [l][e]
  __shared__ __align__(16) double swT[N4 * LP + 64];  // [e][l] padded (+ ring overrun)
  for (int i = threadIdx.x; i < TPC * (L + 16); i += 32) sx[i] = gx[i % (TPC * L)];
  for (int i = threadIdx.x; i < (L + 16) * N4; i += 32) sw[i] = gw[i % (L * N4)];
  for (int i = threadIdx.x; i < N4 * LP + 64; i += 32) swT[i] = gw[(i % LP) % L * N4 + i / LP];
  __syncthreads();
  const int tl = threadIdx.x / N4, e = threadIdx.x % N4;
  const double* xr = sx + tl * (L + 16);
  const double* we = swT + e * LP;
  const int n4 = V == 1 ? n4_rt : N4;  // runtime vs compile-time W stride
  const double* wc = sw + e;
  double acc = 0.0;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (V == 0) {  // registers only (upper bound)
      double xv[16], wv[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) { xv[i] = xr[i]; wv[i] = wc[i * N4]; }
#pragma unroll 1
      for (int b = 0; b < L; b += 16)
#pragma unroll
        for (int i = 0; i < 16; ++i) acc = fma(xv[i], wv[i], acc);
    } else if (V == 1 || V == 2) {  // [l][e] W, ring distance 16, 32-step body (runtime / compile-time stride)
      constexpr int kD = 16, kB = 32;
      double xa[kD], wa[kD];
#pragma unroll
      for (int i = 0; i < kD; i += 2) {
        const double2 t = *reinterpret_cast<const double2*>(xr + i);
        xa[i] = t.x;
        xa[i + 1] = t.y;
      }
#pragma unroll
      for (int i = 0; i < kD; ++i) wa[i] = wc[i * n4];
#pragma unroll 1
      for (int b = 0; b < L; b += kB) {
        const double* xq = xr + b + kD;
        const double* wq = wc + (b + kD) * n4;
#pragma unroll
        for (int i = 0; i < kB; ++i) {
          const double xx = xa[i % kD], ww = wa[i % kD];
          if (i & 1) {
            const double2 t = *reinterpret_cast<const double2*>(xq + i - 1);
            xa[(i - 1) % kD] = t.x;
            xa[i % kD] = t.y;
          }
          wa[i % kD] = wq[i * n4];
          acc = fma(xx, ww, acc);
        }
      }
    } else if (V == 3 || V == 4) {  // [e][l] W, LDS.128 for both operands, ring distance kD
      constexpr int kD = V == 3 ? 16 : 32, kB = 32;
      double xa[kD], wa[kD];
#pragma unroll
      for (int i = 0; i < kD; i += 2) {
        const double2 t = *reinterpret_cast<const double2*>(xr + i);
        const double2 u = *reinterpret_cast<const double2*>(we + i);
        xa[i] = t.x; xa[i + 1] = t.y; wa[i] = u.x; wa[i + 1] = u.y;
      }
#pragma unroll 1
      for (int b = 0; b < L; b += kB) {
        const double* xq = xr + b + kD;
        const double* wq = we + b + kD;
#pragma unroll
        for (int i = 0; i < kB; ++i) {
          const double xx = xa[i % kD], ww = wa[i % kD];
          if (i & 1) {
            const double2 t = *reinterpret_cast<const double2*>(xq + i - 1);
            const double2 u = *reinterpret_cast<const double2*>(wq + i - 1);
            xa[(i - 1) % kD] = t.x; xa[i % kD] = t.y;
            wa[(i - 1) % kD] = u.x; wa[i % kD] = u.y;
          }
          acc = fma(xx, ww, acc);
        }
      }
    } else {  // V == 5: as 3, every step one asm block (fma + the ring loads) so the order is fixed in PTX
      constexpr int kD = 16, kB = 32;
      double xa[kD], wa[kD];
#pragma unroll
      for (int i = 0; i < kD; i += 2) {
        const double2 t = *reinterpret_cast<const double2*>(xr + i);
        const double2 u = *reinterpret_cast<const double2*>(we + i);
        xa[i] = t.x; xa[i + 1] = t.y; wa[i] = u.x; wa[i + 1] = u.y;
      }
      const unsigned xs = static_cast<unsigned>(__cvta_generic_to_shared(xr));
      const unsigned ws = static_cast<unsigned>(__cvta_generic_to_shared(we));
#pragma unroll 1
      for (int b = 0; b < L; b += kB) {
        const unsigned xq = xs + (b + kD) * 8, wq = ws + (b + kD) * 8;
#pragma unroll
        for (int i = 0; i < kB; ++i) {
          const double xx = xa[i % kD], ww = wa[i % kD];
          if (i & 1) {
            asm volatile(
                "fma.rn.f64 %0, %5, %6, %0;\n\t"
                "ld.shared.v2.f64 {%1, %2}, [%7];\n\t"
                "ld.shared.v2.f64 {%3, %4}, [%8];"
                : "+d"(acc), "=d"(xa[(i - 1) % kD]), "=d"(xa[i % kD]), "=d"(wa[(i - 1) % kD]), "=d"(wa[i % kD])
                : "d"(xx), "d"(ww), "r"(xq + (i - 1) * 8), "r"(wq + (i - 1) * 8));
          } else {
            asm volatile("fma.rn.f64 %0, %1, %2, %0;" : "+d"(acc) : "d"(xx), "d"(ww));
          }
        }
      }
    }
  }
  long long t1 = clock64();
  out[blockIdx.x * 32 + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int V>
void run(const char* name, const double* gx, const double* gw, double* out, long long* cyc) {
  const int reps = 64;
  long long h[8];
  chain<V><<<8, 32>>>(gx, gw, out, cyc, reps, N4);
  chain<V><<<8, 32>>>(gx, gw, out, cyc, reps, N4);
  cudaError_t err = cudaMemcpy(h, cyc, 8 * 8, cudaMemcpyDeviceToHost);
  printf("%-58s %.2f cyc/step  (%s)\n", name, (double)h[0] / (reps * L), cudaGetErrorString(err));
}

int main() {
  double *gx, *gw, *out;
  long long* cyc;
  cudaMalloc(&gx, TPC * L * 8);
  cudaMalloc(&gw, L * N4 * 8);
  cudaMalloc(&out, 8 * 32 * 8);
  cudaMalloc(&cyc, 8 * 8);
  cudaMemset(gx, 0, TPC * L * 8);
  cudaMemset(gw, 0, L * N4 * 8);
  run<0>("registers only", gx, gw, out, cyc);
  run<1>("[l][e] W, ring 16, runtime stride (router_ws_kernel)", gx, gw, out, cyc);
  run<2>("[l][e] W, ring 16, compile-time stride", gx, gw, out, cyc);
  run<3>("[e][l] W, LDS.128 both, ring 16", gx, gw, out, cyc);
  run<4>("[e][l] W, LDS.128 both, ring 32", gx, gw, out, cyc);
  run<5>("[e][l] W, LDS.128 both, ring 16, asm-ordered", gx, gw, out, cyc);
  return 0;
}
