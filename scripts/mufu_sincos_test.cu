// Dev aid: accuracy of SFU sin/cos with a first-order correction of the SFU's input
// rounding (t' = RZ(x / 2pi) is what MUFU sees; delta = x - 2 pi t' is computed exactly
// with two FMAs and sin x = s0 + delta c0, cos x = c0 - delta s0).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/mufu_sincos_test scripts/mufu_sincos_test.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>

__device__ __forceinline__ void poly_sincos(float a, float& s, float& c) {
    const float k = rintf(a * 0.636619772367581343f);
    float r = fmaf(-k, 1.5703125f, a);
    r = fmaf(-k, 4.837512969970703125e-4f, r);
    r = fmaf(-k, 7.54978995489188216e-8f, r);
    const float r2 = r * r;
    float ps = fmaf(r2, -1.9515295891e-4f, 8.3321608736e-3f);
    ps = fmaf(r2, ps, -1.6666654611e-1f);
    ps = fmaf(r2 * r, ps, r);
    float pc = fmaf(r2, 2.443315711809948e-5f, -1.388731625493765e-3f);
    pc = fmaf(r2, pc, 4.166664568298827e-2f);
    pc = fmaf(r2 * r2, pc, fmaf(-0.5f, r2, 1.0f));
    const int q = static_cast<int>(k) & 3;
    const float sv = (q & 1) ? pc : ps, cv = (q & 1) ? ps : pc;
    s = (q & 2) ? -sv : sv;
    c = ((q + 1) & 2) ? -cv : cv;
}
__device__ __forceinline__ void fast_sincos(float a, float& s, float& c) {
    const float k = rintf(a * 0.15915494309189535f);
    float x = fmaf(-k, 6.28318548202514648f, a);
    x = fmaf(-k, -1.7484556e-07f, x);
    s = __sinf(x);
    c = __cosf(x);
}
// corrected: reduce to [-pi, pi] (2-term), then correct the SFU input rounding
__device__ __forceinline__ void corr_sincos(float a, float& s, float& c) {
    const float k = rintf(a * 0.15915494309189535f);
    float x = fmaf(-k, 6.28318548202514648f, a);
    x = fmaf(-k, -1.7484556e-07f, x);
    const float t = __fmul_rz(x, 0.15915493667125701904f);  // what MUFU consumes (revolutions)
    float d = fmaf(-t, 6.28318548202514648f, x);
    d = fmaf(-t, -1.7484556e-07f, d);
    const float s0 = __sinf(x), c0 = __cosf(x);
    s = fmaf(d, c0, s0);
    c = fmaf(-d, s0, c0);
}
__global__ void k(const float* a, int n, double* err) {
    double e[6] = {0, 0, 0, 0, 0, 0};
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const float x = a[i];
        const double sd = sin((double)x), cd = cos((double)x);
        float s, c;
        poly_sincos(x, s, c);
        e[0] = fmax(e[0], fabs(s - sd)); e[1] = fmax(e[1], fabs(c - cd));
        fast_sincos(x, s, c);
        e[2] = fmax(e[2], fabs(s - sd)); e[3] = fmax(e[3], fabs(c - cd));
        corr_sincos(x, s, c);
        e[4] = fmax(e[4], fabs(s - sd)); e[5] = fmax(e[5], fabs(c - cd));
    }
    for (int j = 0; j < 6; ++j) {
        // max via atomicMax on the bit pattern (non-negative doubles order like integers)
        atomicMax(reinterpret_cast<unsigned long long*>(err + j), (unsigned long long)__double_as_longlong(e[j]));
    }
}
int main() {
    const int n = 1 << 24;
    float* h = (float*)malloc(n * sizeof(float));
    for (double range : {3.14159, 10.0, 100.0, 1000.0}) {
        srand(1);
        for (int i = 0; i < n; ++i) h[i] = (float)((2.0 * rand() / RAND_MAX - 1.0) * range);
        float* d; double* e;
        cudaMalloc(&d, n * sizeof(float)); cudaMalloc(&e, 6 * sizeof(double));
        cudaMemcpy(d, h, n * sizeof(float), cudaMemcpyHostToDevice);
        cudaMemset(e, 0, 6 * sizeof(double));
        k<<<296, 256>>>(d, n, e);
        double he[6];
        cudaMemcpy(he, e, sizeof(he), cudaMemcpyDeviceToHost);
        printf("|a| <= %-8g poly sin %.2e cos %.2e | sfu sin %.2e cos %.2e | corrected sin %.2e cos %.2e\n", range, he[0], he[1],
               he[2], he[3], he[4], he[5]);
        cudaFree(d); cudaFree(e);
    }
    return 0;
}
