// Micro-benchmark of the CUDA-core pipes this path is bound by (B200, sm_100a):
// FFMA, FFMA2 (fma.rn.f32x2), FFMA.SAT, FMNMX, MUFU.RCP and a mix, all with
// 8 independent dependency chains per thread.  Prints warp-instr/clk/SM.
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 4096
__device__ __forceinline__ unsigned long long pk(float a, float b){ unsigned long long r; asm volatile("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r; }

template <int MODE>
__global__ void kern(float* out, float s)
{
    float a[8];
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i;
    unsigned long long p[8];
    for (int i = 0; i < 8; ++i) p[i] = pk(a[i], a[i] + 1.f);
    const unsigned long long S = pk(s, s), T = pk(0.5f, 0.25f);
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE == 0) a[i] = fmaf(a[i], s, 0.5f);                       // FFMA (imm)
            if (MODE == 1) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(s), "f"(a[(i+1)&7]));  // FFMA 3-reg
            if (MODE == 2) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[i]) : "l"(S), "l"(T));       // FFMA2
            if (MODE == 3) asm volatile("fma.rn.sat.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(s), "f"(a[(i+1)&7])); // FFMA.SAT
            if (MODE == 4) asm volatile("max.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(a[(i+3)&7]));             // FMNMX
            if (MODE == 5) { float r; asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a[i])); a[i] = r + 1.0f; }  // MUFU.RCP (+FADD)
            if (MODE == 6) { // mix: 2 FFMA2 + 1 FFMA.SAT + 1 FMNMX
                asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[i]) : "l"(S), "l"(T));
                asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[(i+4)&7]) : "l"(S), "l"(T));
                asm volatile("fma.rn.sat.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(s), "f"(a[(i+1)&7]));
                asm volatile("max.f32 %0, %0, %1;" : "+f"(a[(i+2)&7]) : "f"(a[(i+3)&7]));
            }
            if (MODE == 7) { // mix: 3 FFMA (3-reg) + 1 FMNMX
                asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(s), "f"(a[(i+1)&7]));
                asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[(i+4)&7]) : "f"(s), "f"(a[(i+5)&7]));
                asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[(i+2)&7]) : "f"(s), "f"(a[(i+6)&7]));
                asm volatile("max.f32 %0, %0, %1;" : "+f"(a[(i+3)&7]) : "f"(a[(i+7)&7]));
            }
        }
    }
    float acc = 0;
    for (int i = 0; i < 8; ++i) { float x, y; asm("mov.b64 {%0,%1}, %2;" : "=f"(x), "=f"(y) : "l"(p[i])); acc += a[i] + x + y; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int MODE>
void run(const char* name, int ipi, float* d, int sms, int clk_khz)
{
    const int blocks = sms * 8, threads = 256;
    kern<MODE><<<blocks, threads>>>(d, 0.999f);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) kern<MODE><<<blocks, threads>>>(d, 0.999f);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (cudaGetLastError() != cudaSuccess) printf("launch error\n");
    double warp_instr = 5.0 * blocks * (threads / 32) * (double)ITERS * 8 * ipi;
    double per_s = warp_instr / (ms * 1e-3);
    printf("%-28s %8.2f ms  %7.3f warp-instr/clk/SM (at %d MHz)  %.1f Tinstr-lane/s\n", name, ms,
           per_s / sms / (clk_khz * 1e3), clk_khz / 1000, per_s * 32 / 1e12);
}

int main()
{
    int sms, clk; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    float* d; cudaMalloc(&d, sizeof(float) * sms * 8 * 256);
    printf("SMs %d, clock attr %d kHz\n", sms, clk);
    run<0>("FFMA imm", 1, d, sms, clk);
    run<1>("FFMA 3-reg", 1, d, sms, clk);
    run<2>("FFMA2 (f32x2)", 1, d, sms, clk);
    run<3>("FFMA.SAT 3-reg", 1, d, sms, clk);
    run<4>("FMNMX", 1, d, sms, clk);
    run<5>("MUFU.RCP", 1, d, sms, clk);
    run<6>("mix 2xFFMA2+SAT+FMNMX", 4, d, sms, clk);
    run<7>("mix 3xFFMA+FMNMX", 4, d, sms, clk);
    return 0;
}
