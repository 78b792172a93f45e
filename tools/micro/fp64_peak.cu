// fp64 roof of this B200 ("measure the fp64 peak before quoting compute
// fractions"): DFMA throughput with 8 independent chains per thread, a full-chip grid, CUDA events.
// Also the rate of the conversions the lattice generator uses (I2F.F64.U32) and of DADD.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu && ./fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CH = 8;

__global__ void k_dfma(double* out, int iters, double a, double b) {
    double x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-9 + c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) x[c] = fma(x[c], a, b);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c];
    if (s == 1.2345) out[0] = s;
}

__global__ void k_i2f(double* out, int iters) {
    double s[CH];
    unsigned u = threadIdx.x * 2654435761u;
#pragma unroll
    for (int c = 0; c < CH; ++c) s[c] = 0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) s[c] += double(u + c * 7u + i);  // I2F.F64.U32 + DADD
    }
    double t = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) t += s[c];
    if (t == 1.2345) out[0] = t;
}

__global__ void k_dadd(double* out, int iters, double a) {
    double x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-9 + c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) x[c] = x[c] + a;
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c];
    if (s == 1.2345) out[0] = s;
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    double* d;
    cudaMalloc(&d, 8);
    const int nsm = p.multiProcessorCount, nt = 512, blocks = nsm * 4, iters = 20000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](auto launch, double ops_per_iter_thread, const char* name, const char* unit) {
        for (int w = 0; w < 3; ++w) launch();
        cudaDeviceSynchronize();
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        const double ops = double(blocks) * nt * iters * ops_per_iter_thread;
        printf("{\"kernel\": \"%s\", \"ms\": %.4f, \"rate\": %.4f, \"unit\": \"%s\", \"sms\": %d}\n", name, best,
               ops / (best * 1e-3) / 1e12, unit, nsm);
    };
    run([&] { k_dfma<<<blocks, nt>>>(d, iters, 0.999999, 1e-7); }, 2.0 * CH, "dfma", "TFLOP/s (2 per FMA)");
    run([&] { k_dadd<<<blocks, nt>>>(d, iters, 1e-7); }, 1.0 * CH, "dadd", "Tops/s");
    run([&] { k_i2f<<<blocks, nt>>>(d, iters); }, 1.0 * CH, "i2f_f64_u32+dadd", "Tconv/s");
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(err));
        return 1;
    }
    return 0;
}
