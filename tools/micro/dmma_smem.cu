// DMMA throughput with shared-memory operands in the trailing-update pattern of k_chol_large /
// k_schur_coop: per 4-wide k step a warp loads 2 A and 8 B fragments (LDS.64) and issues 16
// DMMA.8x8x4 into 16 accumulators.  Grid = #SMs x 1 CTA; reports flop/clk/SM for 256 and 512
// threads, and the register-operand ceiling (no LDS) for comparison.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <bool SMEM, int NTB>
__global__ void __launch_bounds__(NTB, 1) k(double *out, long long *cyc, int reps) {
    __shared__ double X[128 * 36];
    for (int e = threadIdx.x; e < 128 * 36; e += blockDim.x) X[e] = 1e-3 * (e % 7);
    // (row stride 36: offsets up to 8 + 4 * 7 + 3 stay inside a row)
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, gr = lane >> 2, gc = lane & 3;
    const int wr = w & 7;
    const double *xa0 = X + (16 * wr + gr) * 36 + gc, *yb0 = X + gr * 36 + gc;
    double acc[2][8][2] = {};
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        // the operand slab moves every rep (no hoisting: the loads stay in the loop, like the
        // pipelined trailing update's stage rotation)
        const int off = r % 3;
        const double *xa = xa0 + off, *yb = yb0 + off;
#pragma unroll
        for (int k4 = 0; k4 < 8; ++k4) {
            double a0, a1;
            if (SMEM) { a0 = xa[4 * k4]; a1 = xa[8 * 36 + 4 * k4]; } else { a0 = 1.0 + k4; a1 = 2.0 + k4; }
#pragma unroll
            for (int nb = 0; nb < 8; ++nb) {
                const double b = SMEM ? yb[8 * nb * 36 + 4 * k4] : 0.5 + nb;
                dmma(acc[0][nb][0], acc[0][nb][1], a0, b);
                dmma(acc[1][nb][0], acc[1][nb][1], a1, b);
            }
        }
    }
    long long t1 = clock64();
    double s = 0;
    for (int h = 0; h < 2; ++h) for (int nb = 0; nb < 8; ++nb) s += acc[h][nb][0] + acc[h][nb][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    double *o; long long *c, h;
    cudaMalloc(&o, sizeof(double) * nsm * 1024);
    cudaMalloc(&c, sizeof(long long) * nsm);
    const int reps = 4096;
    for (int nt : {256, 512}) {
        for (int sm = 0; sm < 2; ++sm) {
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            float ms = 0.f;
            for (int it = 0; it < 2; ++it) {
                cudaEventRecord(e0);
                if (nt == 256) {
                    if (sm) k<true, 256><<<nsm, nt>>>(o, c, reps); else k<false, 256><<<nsm, nt>>>(o, c, reps);
                } else {
                    if (sm) k<true, 512><<<nsm, nt>>>(o, c, reps); else k<false, 512><<<nsm, nt>>>(o, c, reps);
                }
                cudaError_t err = cudaGetLastError();
                if (err != cudaSuccess) printf("launch error: %s\n", cudaGetErrorString(err));
                cudaEventRecord(e1);
                cudaDeviceSynchronize();
                cudaEventElapsedTime(&ms, e0, e1);
            }
            cudaMemcpy(&h, c, sizeof(long long), cudaMemcpyDeviceToHost);
            const double dmmas = (double)(nt / 32) * reps * 8 * 16;
            const double total_flop = dmmas * 512 * nsm;
            printf("%s operands, %d threads: %.1f flop/clk/SM (%.3f DMMA/clk, CTA 0 clock64); whole grid %.2f TFLOP/s "
                   "(CUDA events, %.3f ms)\n", sm ? "smem" : "register", nt, dmmas * 512 / h, dmmas / h,
                   total_flop / (ms * 1e-3) / 1e12, ms);
        }
    }
    return 0;
}
