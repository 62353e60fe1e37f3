// micro-latencies on B200: dependent DFMA / DDIV / DSQRT chains, shared loads (LDS vs generic), shuffles
#include <cstdio>
__device__ double sink;
__global__ void k(double* out, long long* t, int n, double* gptr) {
    __shared__ double sm[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = 1.0 + i * 1e-3;
    __syncthreads();
    double x = out[0], y = 1.0000001;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = fma(x, y, 1e-9);
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) x = 1.0 / (x + 1.5);
    long long t2 = clock64();
    for (int i = 0; i < n; ++i) x = sqrt(x + 2.0);
    long long t3 = clock64();
    int idx = threadIdx.x;
    for (int i = 0; i < n; ++i) { x += sm[idx]; idx = (idx + (int)(x > 1e30)) & 1023; }
    long long t4 = clock64();
    double* g = gptr ? gptr : sm;  // generic pointer to shared
    for (int i = 0; i < n; ++i) { x += g[idx]; idx = (idx + (int)(x > 1e30)) & 1023; }
    long long t5 = clock64();
    for (int i = 0; i < n; ++i) x += __shfl_xor_sync(0xffffffff, x, 1);
    long long t6 = clock64();
    float xf = (float)x;
    for (int i = 0; i < n; ++i) xf = fmaf(xf, 1.0000001f, 1e-9f);
    long long t7 = clock64();
    if (threadIdx.x == 0) { t[0]=t1-t0; t[1]=t2-t1; t[2]=t3-t2; t[3]=t4-t3; t[4]=t5-t4; t[5]=t6-t5; t[6]=t7-t6; }
    if (x == 12345.0 || xf == 1.f) sink = x + xf;
}
int main() {
    double* o; long long* t; cudaMalloc(&o, 8); cudaMalloc(&t, 64);
    double one = 1.0; cudaMemcpy(o, &one, 8, cudaMemcpyHostToDevice);
    for (int threads : {32, 512}) {
        k<<<1, threads>>>(o, t, 1000, nullptr); cudaDeviceSynchronize();
        long long h[8]; cudaMemcpy(h, t, 64, cudaMemcpyDeviceToHost);
        printf("threads %d cycles/op: dfma %.1f ddiv %.1f dsqrt %.1f lds %.1f generic-lds %.1f shfl %.1f ffma %.1f\n", threads,
               h[0]/1000.0, h[1]/1000.0, h[2]/1000.0, h[3]/1000.0, h[4]/1000.0, h[5]/1000.0, h[6]/1000.0);
    }
    cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
    printf("%s sm %d.%d clock %d kHz SMs %d\n", p.name, p.major, p.minor, p.clockRate, p.multiProcessorCount);
    return 0;
}
