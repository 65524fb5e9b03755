// pipe_bench.cu -- issue rate of the integer instructions the AOT probe can be
// built from, per SM sub-partition (SMSP), on the device it runs on.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_bench tools/pipe_bench.cu && ./pipe_bench
//
// Each kernel runs ILP independent dependency chains of one instruction kind
// per thread (operands come from kernel parameters, so ptxas cannot fold
// them), 8 warps per SMSP.  Printed: cycles per warp instruction per SMSP
// (1.0 = the issue limit, 2.0 = a half-rate pipe).  The question it answers
// for DESIGN §4: can the bitmap probe's shifts / masks / adds (ALU pipe, 64%
// busy in the C4 count kernel) move to the FMA pipe as IMAD / IMAD.HI?
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ILP = 8, ITER = 4096;

enum Kind { kShf, kLop, kImad, kImadHi, kImadHiAcc, kMixShfImadHi, kMixLopImad, kViaddmnmx, kMix3 };

template <int K>
__global__ void __launch_bounds__(1024) bench(unsigned* out, unsigned a, unsigned b, unsigned c, long long* cyc) {
  unsigned v[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) v[i] = threadIdx.x * 7 + i + a;
  const long long t0 = clock64();
  for (int it = 0; it < ITER; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      if constexpr (K == kShf) asm volatile("shf.r.wrap.b32 %0, %0, %1, %2;" : "+r"(v[i]) : "r"(b), "r"(c));
      if constexpr (K == kLop) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(v[i]) : "r"(b), "r"(c));
      if constexpr (K == kImad) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(v[i]) : "r"(b), "r"(c));
      if constexpr (K == kImadHi) asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(v[i]) : "r"(b));
      if constexpr (K == kImadHiAcc) asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(v[i]) : "r"(b), "r"(c));
      if constexpr (K == kViaddmnmx) v[i] = min(v[i] - b, c);
      if constexpr (K == kMixShfImadHi) {
        if (i & 1) asm volatile("shf.r.wrap.b32 %0, %0, %1, %2;" : "+r"(v[i]) : "r"(b), "r"(c));
        else asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(v[i]) : "r"(b), "r"(c));
      }
      if constexpr (K == kMixLopImad) {
        if (i & 1) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(v[i]) : "r"(b), "r"(c));
        else asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(v[i]) : "r"(b), "r"(c));
      }
      if constexpr (K == kMix3) {  // the proposed probe's mix: 2 ALU : 3 FMA-pipe (of which 2 are .HI)
        if (i % 5 == 0) asm volatile("shf.l.wrap.b32 %0, %0, %1, %2;" : "+r"(v[i]) : "r"(b), "r"(c));
        else if (i % 5 == 1) v[i] = min(v[i] - b, c);
        else if (i % 5 == 2) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(v[i]) : "r"(b), "r"(c));
        else asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(v[i]) : "r"(b), "r"(c));
      }
    }
  }
  const long long t1 = clock64();
  unsigned s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s ^= v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int K>
void run(const char* name, unsigned* out, long long* cyc, int sms) {
  bench<K><<<sms, 1024>>>(out, 3, 0x08000001u, 5, cyc);  // warm-up
  bench<K><<<sms, 1024>>>(out, 3, 0x08000001u, 5, cyc);
  cudaDeviceSynchronize();
  long long h[1024];
  cudaMemcpy(h, cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < sms; ++i) mean += double(h[i]);
  mean /= sms;
  // 32 warps per SM = 8 per SMSP, each issuing ILP * ITER instructions of the kind
  std::printf("%-28s %.3f cycles per warp instruction per SMSP\n", name, mean / (8.0 * ILP * ITER));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* out;
  long long* cyc;
  cudaMalloc(&out, sizeof(unsigned) * sms * 1024);
  cudaMalloc(&cyc, sizeof(long long) * sms);
  run<kShf>("SHF (alu)", out, cyc, sms);
  run<kLop>("LOP3 (alu)", out, cyc, sms);
  run<kViaddmnmx>("VIADDMNMX (alu)", out, cyc, sms);
  run<kImad>("IMAD (fma)", out, cyc, sms);
  run<kImadHi>("IMAD.HI mul (fma?)", out, cyc, sms);
  run<kImadHiAcc>("IMAD.HI mad (fma?)", out, cyc, sms);
  run<kMixShfImadHi>("SHF + IMAD.HI 1:1", out, cyc, sms);
  run<kMixLopImad>("LOP3 + IMAD 1:1", out, cyc, sms);
  run<kMix3>("probe mix 2 alu : 3 fma", out, cyc, sms);
  if (cudaDeviceSynchronize() != cudaSuccess) return 1;
  return 0;
}
