// debug harness: hk_fft_matvec on a tiny problem from C++ (device buffers via cudaMalloc)
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "hk.h"
int main(int argc, char **argv) {
    const int kind = 0, n = argc > 1 ? atoi(argv[1]) : 8, P = argc > 2 ? atoi(argv[2]) : 300;
    hk_fft_plan_info info;
    int rc = hk_fft_plan(kind, n, P, &info);
    printf("plan rc=%d w=%d Ls=%d n1=%d n2=%d ws=%llu\n", rc, info.w, info.Ls, info.log_n1, info.log_n2,
           (unsigned long long)info.ws_bytes);
    fflush(stdout);
    const int L = (P + 63) / 64, Ly = 2 * L + 1, na = 2 * n - 1;
    std::vector<uint64_t> am((size_t)na * L, 1), xm((size_t)n * L, 1);
    std::vector<int8_t> as(na, 1), xs(n, 1);
    uint64_t *dam, *dxm, *dym; int8_t *das, *dxs, *dys; void *ws;
    cudaMalloc(&dam, am.size() * 8); cudaMalloc(&dxm, xm.size() * 8); cudaMalloc(&dym, (size_t)n * Ly * 8);
    cudaMalloc(&das, na); cudaMalloc(&dxs, n); cudaMalloc(&dys, n); cudaMalloc(&ws, info.ws_bytes + 256);
    cudaMemcpy(dam, am.data(), am.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dxm, xm.data(), xm.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(das, as.data(), na, cudaMemcpyHostToDevice);
    cudaMemcpy(dxs, xs.data(), n, cudaMemcpyHostToDevice);
    rc = hk_fft_workspace_init(kind, n, P, ws, info.ws_bytes, nullptr);
    printf("init rc=%d sync=%s\n", rc, cudaGetErrorString(cudaDeviceSynchronize()));
    fflush(stdout);
    rc = hk_fft_matvec(kind, n, P, dam, das, dxm, dxs, dym, dys, ws, info.ws_bytes, nullptr);
    printf("matvec rc=%d sync=%s\n", rc, cudaGetErrorString(cudaDeviceSynchronize()));
    fflush(stdout);
    std::vector<uint64_t> y((size_t)n * Ly);
    cudaMemcpy(y.data(), dym, y.size() * 8, cudaMemcpyDeviceToHost);
    printf("y[0][0..3] = %llu %llu %llu (expect %d)\n", (unsigned long long)y[0], (unsigned long long)y[1],
           (unsigned long long)y[2], n);
    return 0;
}
