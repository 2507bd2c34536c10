// Checks the tiled lower-block fixed-point -> double conversion of B-check (k_fx_to_double,
// with its mirror) against the plain row-wise conversion of a full symmetric matrix: bit-equal.
// (This caught 3 x 3 diagonal blocks straddling a 64-tile edge.)
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
__device__ __forceinline__ double fx_scale(const double *dmax, int n_pairs) {
    const double m = fmax(*dmax, 1e-300);
    const int e = ilogb(m) + 1 + ilogb((double)max(1, 64 * n_pairs)) + 1;
    return ldexp(1.0, 61 - e);
}
constexpr double kFxLo = 1099511627776.0;
__device__ __forceinline__ double fx_get(long long hi, long long lo, double inv_sc) {
    return ((double)hi + (double)lo / kFxLo) * inv_sc;
}
__global__ void k_old(long long *M, const long long *Ml, int ld, const int *nS_ptr, int capS, const double *dmax, const int *acnt) {
    const int n = 3 * min(*nS_ptr, capS);
    const double inv = 1.0 / fx_scale(dmax, acnt[1]);
    const int lane = threadIdx.x & 31, nw = (gridDim.x * blockDim.x) >> 5;
    for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n; r += nw)
        for (int c = lane; c < n; c += 32) {
            const size_t off = (size_t)r * ld + c;
            reinterpret_cast<double *>(M)[off] = fx_get(M[off], Ml[off], inv);
        }
}
__global__ void __launch_bounds__(256) k_new(long long *M, const long long *Ml, int ld, const int *nS_ptr,
                                                      int capS, const double *dmax, const int *acnt) {
    __shared__ double S[64][65];
    const int n = 3 * min(*nS_ptr, capS);
    const double inv = 1.0 / fx_scale(dmax, acnt[1]);
    const int nt = (n + 63) / 64, ntile = nt * (nt + 1) / 2;
    double *D = reinterpret_cast<double *>(M);
    for (int t = blockIdx.x; t < ntile; t += gridDim.x) {
        int R = 0, C = t;
        while (C > R) { C -= R + 1; ++R; }
        const int r0 = 64 * R, c0 = 64 * C;
        for (int e = threadIdx.x; e < 64 * 64; e += blockDim.x) {
            const int rr = e >> 6, cc = e & 63, r = r0 + rr, c = c0 + cc;
            double v = 0.0;
            if (r < n && c < n && c < 3 * (r / 3) + 3) {
                const size_t off = (size_t)r * ld + c;
                v = fx_get(M[off], Ml[off], inv);
                D[off] = v;
            }
            S[rr][cc] = v;
        }
        if (R == C && threadIdx.x < 64) {
            const int r = r0 + threadIdx.x;
            for (int c = c0 + 64; r < n && c < min(n, 3 * (r / 3) + 3); ++c) {
                const size_t off = (size_t)r * ld + c;
                D[off] = fx_get(M[off], Ml[off], inv);
            }
        }
        __syncthreads();
        for (int e = threadIdx.x; e < 64 * 64; e += blockDim.x) {
            const int cc = e >> 6, rr = e & 63, r = r0 + rr, c = c0 + cc;
            if (r < n && c < 3 * (r / 3)) D[(size_t)c * ld + r] = S[rr][cc];
        }
        __syncthreads();
    }
}
int main() {
    const int capS = 120, nS = 100, ld = 3 * capS, n = 3 * nS;
    std::vector<long long> hi((size_t)ld * ld), lo((size_t)ld * ld);
    srand(1);
    for (int r = 0; r < n; ++r) for (int c = 0; c <= r; ++c) {
        long long h = (long long)(rand() % 2000001) - 1000000, l = (long long)(rand() % 2001) - 1000;
        hi[(size_t)r * ld + c] = hi[(size_t)c * ld + r] = h; lo[(size_t)r * ld + c] = lo[(size_t)c * ld + r] = l;
    }
    long long *dA, *dB, *dl; int *dn, *dac; double *dm;
    cudaMalloc(&dA, hi.size() * 8); cudaMalloc(&dB, hi.size() * 8); cudaMalloc(&dl, lo.size() * 8);
    cudaMalloc(&dn, 4); cudaMalloc(&dac, 8); cudaMalloc(&dm, 16);
    int ac[2] = {5, 5}; double dmx[2] = {1.0, 0};
    cudaMemcpy(dn, &nS, 4, cudaMemcpyHostToDevice); cudaMemcpy(dac, ac, 8, cudaMemcpyHostToDevice); cudaMemcpy(dm, dmx, 16, cudaMemcpyHostToDevice);
    cudaMemcpy(dA, hi.data(), hi.size() * 8, cudaMemcpyHostToDevice); cudaMemcpy(dB, hi.data(), hi.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dl, lo.data(), lo.size() * 8, cudaMemcpyHostToDevice);
    k_old<<<296, 256>>>(dA, dl, ld, dn, capS, dm, dac);
    k_new<<<592, 256>>>(dB, dl, ld, dn, capS, dm, dac);
    printf("launch: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    std::vector<double> a(hi.size()), b(hi.size());
    cudaMemcpy(a.data(), dA, a.size() * 8, cudaMemcpyDeviceToHost); cudaMemcpy(b.data(), dB, b.size() * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int r = 0; r < n; ++r) for (int c = 0; c < n; ++c) {
        const size_t o = (size_t)r * ld + c;
        if (a[o] != b[o]) { if (bad < 10) printf("diff at %d %d: %g %g\n", r, c, a[o], b[o]); ++bad; }
    }
    printf("mismatches %d of %d\n", bad, n * n);
}
