// Isolates the trailing-update block of k_schur_coop's large-system Cholesky (update_pair:
// A_ij -= sum_k L_ik L_jk^T on a 128 x 64 block, k streamed in 32-wide chunks through a 3-stage
// cp.async pipeline) on a 9 024 x 9 024 FP64 matrix (C3 scale).  Each of the 148 CTAs updates
// P blocks with a 256-deep k range (one panel), like the update group of one look-ahead
// iteration.  Variants switch parts off to find what keeps the block below the DMMA rate:
//   bit 0: no accumulator load / store (registers start at 0, one sum written at the end)
//   bit 1: no cp.async (operands stay whatever the stage holds)
//   bit 2: no __syncthreads in the chunk loop
// Prints us per block and the fraction of the per-SM DMMA rate (128 flop/clk at the clock read).
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdint>

constexpr int TB = 64, NT = 256, KC = 32, XS = 36;
constexpr int SMEM = 3 * (128 + 64) * XS * 8;
__device__ long long g_cyc[2];
#define CYC0 long long cyc_t0 = clock64();
#define CYC1 if (blockIdx.x == 0 && threadIdx.x == 0) { g_cyc[0] = cyc_t0; g_cyc[1] = clock64(); }

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int V>
__global__ void __launch_bounds__(NT, 1) k_pairs(double *Sh, int ldh, int ma, int P, int nrow_pairs, double *out) {
    CYC0
    extern __shared__ double sm[];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, gr = lane >> 2, gc = lane & 3;
    double *Xs = sm, *Ys = sm + 3 * 128 * XS;
    double tot = 0.0;
    for (int p = 0; p < P; ++p) {
        const int b = blockIdx.x * P + p;
        const int ti = 4 + 2 * (b % nrow_pairs), tj = 4 + (b / nrow_pairs) % ((ma / TB) - 4);
        const int r0 = ti * TB, c0 = tj * TB;
        const int rows = min(2 * TB, ma - r0), cols = min(TB, ma - c0);
        const int kbeg = 0, nch = 4 * TB / KC;
        auto issue = [&](int ch) {
            if (!(V & 2) && ch < nch) {
                const int sg = ch % 3, kc = kbeg + ch * KC;
                double *X = Xs + sg * 128 * XS, *Y = Ys + sg * 64 * XS;
                for (int e = tid; e < 3 * 1024; e += NT) {
                    const bool isx = e < 2048;
                    const int ee = isx ? e : e - 2048, r = ee >> 4, c2 = (ee & 15) * 2;
                    double *dst = (isx ? X : Y) + r * XS + c2;
                    if (r < (isx ? rows : cols)) {
                        const double *src = Sh + (size_t)((isx ? r0 : c0) + r) * ldh + kc + c2;
                        const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(src));
                    } else {
                        dst[0] = 0.0;
                        dst[1] = 0.0;
                    }
                }
            }
            asm volatile("cp.async.commit_group;\n" ::);
        };
        issue(0);
        issue(1);
        if ((V & 8) && p + 1 < P) {
            const int bn = b + 1;
            const int tin = 4 + 2 * (bn % nrow_pairs), tjn = 4 + (bn / nrow_pairs) % ((ma / TB) - 4);
            for (int i = tid; i < 512; i += NT) {
                const double *ln = Sh + (size_t)(tin * TB + (i >> 2)) * ldh + tjn * TB + (i & 3) * 16;
                if (tin * TB + (i >> 2) < ma) asm volatile("prefetch.global.L2 [%0];\n" ::"l"(ln));
            }
        }
        double acc[2][8][2];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int nb = 0; nb < 8; ++nb) {
                const int r = 16 * wid + 8 * h + gr, c = 8 * nb + 2 * gc;
                if (V & 1) { acc[h][nb][0] = 0.0; acc[h][nb][1] = 0.0; continue; }
                if ((V & 16) && r < rows && c + 1 < cols) {
                    const double2 v = *reinterpret_cast<const double2 *>(Sh + (size_t)(r0 + r) * ldh + c0 + c);
                    acc[h][nb][0] = -v.x; acc[h][nb][1] = -v.y; continue;
                }
                acc[h][nb][0] = (r < rows && c < cols) ? -Sh[(size_t)(r0 + r) * ldh + c0 + c] : 0.0;
                acc[h][nb][1] = (r < rows && c + 1 < cols) ? -Sh[(size_t)(r0 + r) * ldh + c0 + c + 1] : 0.0;
            }
        for (int ch = 0; ch < nch; ++ch) {
            issue(ch + 2);
            asm volatile("cp.async.wait_group 2;\n" ::);
            if (!(V & 4)) __syncthreads();
            const double *X = Xs + (ch % 3) * 128 * XS + (16 * wid + gr) * XS + gc;
            const double *Y = Ys + (ch % 3) * 64 * XS + gr * XS + gc;
#pragma unroll
            for (int k4 = 0; k4 < KC / 4; ++k4) {
                const double a0 = X[4 * k4], a1 = X[8 * XS + 4 * k4];
#pragma unroll
                for (int nb = 0; nb < 8; ++nb) {
                    const double bv = Y[8 * nb * XS + 4 * k4];
                    dmma(acc[0][nb][0], acc[0][nb][1], a0, bv);
                    dmma(acc[1][nb][0], acc[1][nb][1], a1, bv);
                }
            }
            if (!(V & 4)) __syncthreads();
        }
        asm volatile("cp.async.wait_group 0;\n" ::);
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int nb = 0; nb < 8; ++nb) {
                const int r = 16 * wid + 8 * h + gr, c = 8 * nb + 2 * gc;
                if (V & 1) { tot += acc[h][nb][0] + acc[h][nb][1]; continue; }
                if ((V & 16) && r < rows && c + 1 < cols) {
                    *reinterpret_cast<double2 *>(Sh + (size_t)(r0 + r) * ldh + c0 + c) = make_double2(-acc[h][nb][0], -acc[h][nb][1]);
                    continue;
                }
                if (r < rows && c < cols) Sh[(size_t)(r0 + r) * ldh + c0 + c] = -acc[h][nb][0];
                if (r < rows && c + 1 < cols) Sh[(size_t)(r0 + r) * ldh + c0 + c + 1] = -acc[h][nb][1];
            }
    }
    if (V & 1) out[blockIdx.x * NT + tid] = tot;
    CYC1
}


// Optimised block: accumulators start at 0 (the block of A is prefetched into L2 at the block
// start and read once in the epilogue: A - acc), ONE __syncthreads per chunk (the refill of the
// stage consumed in the previous chunk is issued after it), and per-thread copy addresses
// computed once per block.  OPT bit 0: chunk stream continues across blocks (next block's first
// two chunks issued before the epilogue).
template <int OPT>
__global__ void __launch_bounds__(NT, 1) k_pairs_opt(double *Sh, int ldh, int ma, int P, int nrow_pairs) {
    CYC0
    extern __shared__ double sm[];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, gr = lane >> 2, gc = lane & 3;
    double *Xs = sm, *Ys = sm + 3 * 128 * XS;
    constexpr int nch = 4 * TB / KC;
    auto block_of = [&](int p, int &r0, int &c0) {
        const int b = blockIdx.x * P + p;
        r0 = (4 + 2 * (b % nrow_pairs)) * TB;
        c0 = (4 + (b / nrow_pairs) % ((ma / TB) - 4)) * TB;
    };
    // per-thread copy pieces: 12 per chunk (8 of X, 4 of Y); source offsets without kc
    long long srco[12];
    unsigned dsto[12];
    unsigned valid = 0;
    auto setup = [&](int r0, int c0) {
        const int rows = min(2 * TB, ma - r0), cols = min(TB, ma - c0);
        valid = 0;
#pragma unroll
        for (int i = 0; i < 12; ++i) {
            const int e = tid + i * NT;
            const bool isx = e < 2048;
            const int ee = isx ? e : e - 2048, r = ee >> 4, c2 = (ee & 15) * 2;
            dsto[i] = (unsigned)__cvta_generic_to_shared((isx ? Xs : Ys) + r * XS + c2);
            srco[i] = (long long)((isx ? r0 : c0) + r) * ldh + c2;
            if (r < (isx ? rows : cols)) valid |= 1u << i;
        }
    };
    auto issue = [&](int ch, int g) {         // chunk ch of the current block into stage g % 3
        if (ch < nch) {
            const int sg = g % 3, kc = ch * KC;
#pragma unroll
            for (int i = 0; i < 12; ++i) {
                const unsigned d = dsto[i] + (unsigned)(sg * (i < 8 ? 128 : 64) * XS * 8);
                if (valid >> i & 1) {
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(Sh + srco[i] + kc));
                } else {
                    asm volatile("st.shared.v2.f64 [%0], {%1, %1};\n" ::"r"(d), "d"(0.0));
                }
            }
        }
        asm volatile("cp.async.commit_group;\n" ::);
    };
    int r0, c0, g = 0;                            // g: chunks consumed so far (stage ring index)
    block_of(0, r0, c0);
    setup(r0, c0);
    issue(0, 0);
    issue(1, 1);
    for (int p = 0; p < P; ++p) {
        const int rows = min(2 * TB, ma - r0), cols = min(TB, ma - c0);
        for (int i = tid; i < 512; i += NT) {          // the A block into L2: 128 rows x 4 lines
            const double *ln = Sh + (size_t)(r0 + (i >> 2)) * ldh + c0 + (i & 3) * 16;
            if ((i >> 2) < rows) asm volatile("prefetch.global.L2 [%0];\n" ::"l"(ln));
        }
        double acc[2][8][2] = {};
        for (int ch = 0; ch < nch; ++ch, ++g) {
            asm volatile("cp.async.wait_group 1;\n" ::);
            __syncthreads();                      // chunk ch visible; stage (g + 2) % 3 free
            issue(ch + 2, g + 2);
            const double *X = Xs + (g % 3) * 128 * XS + (16 * wid + gr) * XS + gc;
            const double *Y = Ys + (g % 3) * 64 * XS + gr * XS + gc;
#pragma unroll
            for (int k4 = 0; k4 < KC / 4; ++k4) {
                const double a0 = X[4 * k4], a1 = X[8 * XS + 4 * k4];
#pragma unroll
                for (int nb = 0; nb < 8; ++nb) {
                    const double bv = Y[8 * nb * XS + 4 * k4];
                    dmma(acc[0][nb][0], acc[0][nb][1], a0, bv);
                    dmma(acc[1][nb][0], acc[1][nb][1], a1, bv);
                }
            }
        }
        // the loop committed empty groups for chunks nch, nch + 1: drop them from the count
        const int pr0 = r0, pc0 = c0;
        if ((OPT & 1) && p + 1 < P) {
            // next block's first two chunks into stages g % 3, (g + 1) % 3, consumed by chunks
            // g - 3, g - 2: every warp is past the barrier of chunk g - 1
            block_of(p + 1, r0, c0);
            setup(r0, c0);
            issue(0, g);
            issue(1, g + 1);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int nb = 0; nb < 8; ++nb) {
                const int r = 16 * wid + 8 * h + gr, c = 8 * nb + 2 * gc;
                double *dst = Sh + (size_t)(pr0 + r) * ldh + pc0 + c;
                if (r < rows && c + 1 < cols) {
                    const double2 v = *reinterpret_cast<const double2 *>(dst);
                    *reinterpret_cast<double2 *>(dst) = make_double2(v.x - acc[h][nb][0], v.y - acc[h][nb][1]);
                } else if (r < rows && c < cols) {
                    dst[0] -= acc[h][nb][0];
                }
            }
        if (!(OPT & 1) && p + 1 < P) {
            block_of(p + 1, r0, c0);
            setup(r0, c0);
            issue(0, g);
            issue(1, g + 1);
        }
    }
    asm volatile("cp.async.wait_group 0;\n" ::);
    CYC1
}

template <int V>
void run(double *Sh, int ldh, int ma, int nsm, double *out, double clk_ghz) {
    cudaFuncSetAttribute(k_pairs<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    const int P = 24, nrow_pairs = (ma / TB - 4) / 2;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int it = 0; it < 4; ++it) {
        cudaEventRecord(e0);
        k_pairs<V><<<nsm, NT, SMEM>>>(Sh, ldh, ma, P, nrow_pairs, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaError_t err = cudaGetLastError();
    long long cy[2];
    cudaMemcpyFromSymbol(cy, g_cyc, sizeof(cy));
    printf("  [CTA 0: %.3f GHz effective over the last launch]\n", (cy[1] - cy[0]) / (best * 1e6));
    const double us_pair = best * 1e3 / P;
    const double flop = 2.0 * 128 * 64 * 256;
    const double ideal_us = flop / (128.0 * clk_ghz * 1e3);
    printf("variant %d (%s%s%s%s%s): %.2f us per block, %.1f %% of the DMMA rate%s\n", V, (V & 1) ? "no-acc " : "",
           (V & 2) ? "no-cp.async " : "", (V & 4) ? "no-sync " : "", (V & 8) ? "L2-prefetch-next " : "", (V & 16) ? "double2-acc " : "", us_pair, 100.0 * ideal_us / us_pair,
           err == cudaSuccess ? "" : cudaGetErrorString(err));
}

template <int OPT>
void run_opt(double *Sh, int ldh, int ma, int nsm, double clk_ghz) {
    cudaFuncSetAttribute(k_pairs_opt<OPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    const int P = 24, nrow_pairs = (ma / TB - 4) / 2;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int it = 0; it < 4; ++it) {
        cudaEventRecord(e0);
        k_pairs_opt<OPT><<<nsm, NT, SMEM>>>(Sh, ldh, ma, P, nrow_pairs);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaError_t err = cudaGetLastError();
    long long cy[2];
    cudaMemcpyFromSymbol(cy, g_cyc, sizeof(cy));
    printf("  [CTA 0: %.3f GHz effective over the last launch]\n", (cy[1] - cy[0]) / (best * 1e6));
    const double us_pair = best * 1e3 / P;
    const double ideal_us = 2.0 * 128 * 64 * 256 / (128.0 * clk_ghz * 1e3);
    printf("optimised %d: %.2f us per block, %.1f %% of the DMMA rate %s\n", OPT, us_pair, 100.0 * ideal_us / us_pair,
           err == cudaSuccess ? "" : cudaGetErrorString(err));
}


// 128 x 128 block (row tiles ti, ti + 1 x column tiles tj, tj + 1): warp w owns rows
// 32 (w & 3) .. + 31 x columns 64 (w >> 2) .. + 63, i.e. per 4-wide k step 4 A + 8 B fragment
// loads feed 32 independent DMMAs; 3-stage ring of 32-wide k chunks (3 x 256 rows x 36).
constexpr int SMEMQ = 3 * 256 * XS * 8;
__global__ void __launch_bounds__(NT, 1) k_quad(double *Sh, int ldh, int ma, int P, int nrow_pairs) {
    CYC0
    extern __shared__ double sm[];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, gr = lane >> 2, gc = lane & 3;
    const int wr = wid & 3, wc = wid >> 2;
    for (int p = 0; p < P; ++p) {
        const int b = blockIdx.x * P + p;
        const int ti = 4 + 2 * (b % nrow_pairs), tj = 4 + 2 * ((b / nrow_pairs) % ((ma / TB - 4) / 2));
        const int r0 = ti * TB, c0 = tj * TB;
        const int rows = min(2 * TB, ma - r0), cols = min(2 * TB, ma - c0);
        constexpr int nch = 4 * TB / KC;
        auto issue = [&](int ch) {
            if (ch < nch) {
                const int sg = ch % 3, kc = ch * KC;
                double *Z = sm + sg * 256 * XS;
#pragma unroll 4
                for (int e = tid; e < 4096; e += NT) {      // 256 rows x 16 pieces: X rows, then Y rows
                    const int r = e >> 4, c2 = (e & 15) * 2;
                    const bool isx = r < 128;
                    const int rr = isx ? r : r - 128;
                    double *dst = Z + r * XS + c2;
                    if (rr < (isx ? rows : cols)) {
                        const double *src = Sh + (size_t)((isx ? r0 : c0) + rr) * ldh + kc + c2;
                        const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(src));
                    } else {
                        dst[0] = 0.0;
                        dst[1] = 0.0;
                    }
                }
            }
            asm volatile("cp.async.commit_group;\n" ::);
        };
        issue(0);
        issue(1);
        double acc[4][8][2];
#pragma unroll
        for (int h = 0; h < 4; ++h)
#pragma unroll
            for (int nb = 0; nb < 8; ++nb) {
                const int r = 32 * wr + 8 * h + gr, c = 64 * wc + 8 * nb + 2 * gc;
                acc[h][nb][0] = (r < rows && c < cols) ? -Sh[(size_t)(r0 + r) * ldh + c0 + c] : 0.0;
                acc[h][nb][1] = (r < rows && c + 1 < cols) ? -Sh[(size_t)(r0 + r) * ldh + c0 + c + 1] : 0.0;
            }
        for (int ch = 0; ch < nch; ++ch) {
            issue(ch + 2);
            asm volatile("cp.async.wait_group 2;\n" ::);
            __syncthreads();
            const double *X = sm + (ch % 3) * 256 * XS + (32 * wr + gr) * XS + gc;
            const double *Y = sm + (ch % 3) * 256 * XS + (128 + 64 * wc + gr) * XS + gc;
#pragma unroll
            for (int k4 = 0; k4 < KC / 4; ++k4) {
                double av[4];
#pragma unroll
                for (int h = 0; h < 4; ++h) av[h] = X[8 * h * XS + 4 * k4];
#pragma unroll
                for (int nb = 0; nb < 8; ++nb) {
                    const double bv = Y[8 * nb * XS + 4 * k4];
#pragma unroll
                    for (int h = 0; h < 4; ++h) dmma(acc[h][nb][0], acc[h][nb][1], av[h], bv);
                }
            }
            __syncthreads();
        }
        asm volatile("cp.async.wait_group 0;\n" ::);
#pragma unroll
        for (int h = 0; h < 4; ++h)
#pragma unroll
            for (int nb = 0; nb < 8; ++nb) {
                const int r = 32 * wr + 8 * h + gr, c = 64 * wc + 8 * nb + 2 * gc;
                if (r < rows && c < cols) Sh[(size_t)(r0 + r) * ldh + c0 + c] = -acc[h][nb][0];
                if (r < rows && c + 1 < cols) Sh[(size_t)(r0 + r) * ldh + c0 + c + 1] = -acc[h][nb][1];
            }
    }
    CYC1
}

// the same block on 16 warps (4 per SM sub-partition), warp tile 16 x 64
__global__ void __launch_bounds__(2 * NT, 1) k_quad16(double *Sh, int ldh, int ma, int P, int nrow_pairs) {
    CYC0
    extern __shared__ double sm[];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, gr = lane >> 2, gc = lane & 3;
    const int wr = wid & 7, wc = wid >> 3;   // 16 warps: rows 16 wr.., columns 64 wc..
    for (int p = 0; p < P; ++p) {
        const int b = blockIdx.x * P + p;
        const int ti = 4 + 2 * (b % nrow_pairs), tj = 4 + 2 * ((b / nrow_pairs) % ((ma / TB - 4) / 2));
        const int r0 = ti * TB, c0 = tj * TB;
        const int rows = min(2 * TB, ma - r0), cols = min(2 * TB, ma - c0);
        constexpr int nch = 4 * TB / KC;
        auto issue = [&](int ch) {
            if (ch < nch) {
                const int sg = ch % 3, kc = ch * KC;
                double *Z = sm + sg * 256 * XS;
#pragma unroll 4
                for (int e = tid; e < 4096; e += 2 * NT) {      // 256 rows x 16 pieces: X rows, then Y rows
                    const int r = e >> 4, c2 = (e & 15) * 2;
                    const bool isx = r < 128;
                    const int rr = isx ? r : r - 128;
                    double *dst = Z + r * XS + c2;
                    if (rr < (isx ? rows : cols)) {
                        const double *src = Sh + (size_t)((isx ? r0 : c0) + rr) * ldh + kc + c2;
                        const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(src));
                    } else {
                        dst[0] = 0.0;
                        dst[1] = 0.0;
                    }
                }
            }
            asm volatile("cp.async.commit_group;\n" ::);
        };
        issue(0);
        issue(1);
        double acc[2][8][2];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int nb = 0; nb < 8; ++nb) {
                const int r = 16 * wr + 8 * h + gr, c = 64 * wc + 8 * nb + 2 * gc;
                acc[h][nb][0] = (r < rows && c < cols) ? -Sh[(size_t)(r0 + r) * ldh + c0 + c] : 0.0;
                acc[h][nb][1] = (r < rows && c + 1 < cols) ? -Sh[(size_t)(r0 + r) * ldh + c0 + c + 1] : 0.0;
            }
        for (int ch = 0; ch < nch; ++ch) {
            issue(ch + 2);
            asm volatile("cp.async.wait_group 2;\n" ::);
            __syncthreads();
            const double *X = sm + (ch % 3) * 256 * XS + (16 * wr + gr) * XS + gc;
            const double *Y = sm + (ch % 3) * 256 * XS + (128 + 64 * wc + gr) * XS + gc;
#pragma unroll
            for (int k4 = 0; k4 < KC / 4; ++k4) {
                double av[2];
#pragma unroll
                for (int h = 0; h < 2; ++h) av[h] = X[8 * h * XS + 4 * k4];
#pragma unroll
                for (int nb = 0; nb < 8; ++nb) {
                    const double bv = Y[8 * nb * XS + 4 * k4];
#pragma unroll
                    for (int h = 0; h < 2; ++h) dmma(acc[h][nb][0], acc[h][nb][1], av[h], bv);
                }
            }
            __syncthreads();
        }
        asm volatile("cp.async.wait_group 0;\n" ::);
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int nb = 0; nb < 8; ++nb) {
                const int r = 16 * wr + 8 * h + gr, c = 64 * wc + 8 * nb + 2 * gc;
                if (r < rows && c < cols) Sh[(size_t)(r0 + r) * ldh + c0 + c] = -acc[h][nb][0];
                if (r < rows && c + 1 < cols) Sh[(size_t)(r0 + r) * ldh + c0 + c + 1] = -acc[h][nb][1];
            }
    }
    CYC1
}

void run_quad(double *Sh, int ldh, int ma, int nsm, double clk_ghz) {
    cudaFuncSetAttribute(k_quad, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEMQ);
    const int P = 12, nrow_pairs = (ma / TB - 4) / 2;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int it = 0; it < 4; ++it) {
        cudaEventRecord(e0);
        k_quad<<<nsm, NT, SMEMQ>>>(Sh, ldh, ma, P, nrow_pairs);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaError_t err = cudaGetLastError();
    long long cy[2];
    cudaMemcpyFromSymbol(cy, g_cyc, sizeof(cy));
    printf("  [CTA 0: %.3f GHz effective over the last launch]\n", (cy[1] - cy[0]) / (best * 1e6));
    const double us = best * 1e3 / P;
    const double ideal_us = 2.0 * 128 * 128 * 256 / (128.0 * clk_ghz * 1e3);
    printf("128x128 block: %.2f us per block, %.1f %% of the DMMA rate %s\n", us, 100.0 * ideal_us / us,
           err == cudaSuccess ? "" : cudaGetErrorString(err));
}
void run_quad16(double *Sh, int ldh, int ma, int nsm, double clk_ghz) {
    cudaFuncSetAttribute(k_quad16, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEMQ);
    const int P = 12, nrow_pairs = (ma / TB - 4) / 2;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int it = 0; it < 4; ++it) {
        cudaEventRecord(e0);
        k_quad16<<<nsm, 2 * NT, SMEMQ>>>(Sh, ldh, ma, P, nrow_pairs);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaError_t err = cudaGetLastError();
    long long cy[2];
    cudaMemcpyFromSymbol(cy, g_cyc, sizeof(cy));
    printf("  [CTA 0: %.3f GHz effective over the last launch]\n", (cy[1] - cy[0]) / (best * 1e6));
    const double us = best * 1e3 / P;
    const double ideal_us = 2.0 * 128 * 128 * 256 / (128.0 * clk_ghz * 1e3);
    printf("128x128 block, 16 warps: %.2f us per block, %.1f %% of the DMMA rate %s\n", us, 100.0 * ideal_us / us,
           err == cudaSuccess ? "" : cudaGetErrorString(err));
}

// TMA version of the 128 x 64 block: thread 0 streams 32-wide k chunks with 2-D tensor copies
// (boxes of 16 doubles x 64 rows, 128-byte swizzle: dense 48 KB stages, conflict-free fragment
// loads) into a 4-stage ring guarded by mbarriers (full: TMA bytes landed; empty: 8 warps done),
// two chunks ahead, across block boundaries.  No __syncthreads and no copy code in the loop.
constexpr int TS_STAGES = 4, TS_STAGE_B = 48 * 1024;
constexpr int SMEMT = TS_STAGES * TS_STAGE_B + 1024 + 64;
__device__ __forceinline__ unsigned su32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_wait(unsigned bar, unsigned parity) {
    asm volatile("{\n.reg .pred P1;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra WAIT_%=;\n}\n"
                 :: "r"(bar), "r"(parity) : "memory");
}
template <int PREF>
__global__ void __launch_bounds__(NT, 1) k_tma(const __grid_constant__ CUtensorMap tmap, double *Sh, int ldh, int ma,
                                               int P, int nrow_pairs) {
    CYC0
    extern __shared__ unsigned char smraw[];
    const unsigned base = (su32(smraw) + 1023u) & ~1023u;
    const unsigned bars = base + TS_STAGES * TS_STAGE_B;          // full[S], empty[S]
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, gr = lane >> 2, gc = lane & 3;
    constexpr int nch = 4 * TB / KC;
    const int G = P * nch;
    if (tid == 0) {
        for (int i = 0; i < TS_STAGES; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" :: "r"(bars + 8 * i));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;\n" :: "r"(bars + 8 * (TS_STAGES + i)));
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    auto block_rc = [&](int p, int &r0, int &c0) {
        const int b = blockIdx.x * P + p;
        r0 = (4 + 2 * (b % nrow_pairs)) * TB;
        c0 = (4 + (b / nrow_pairs) % ((ma / TB) - 4)) * TB;
    };
    int gi = 0;                                   // next chunk to issue (thread 0)
    auto produce = [&](int upto) {
        for (; gi < upto && gi < G; ++gi) {
            const int st = gi % TS_STAGES;
            if (gi >= TS_STAGES) mb_wait(bars + 8 * (TS_STAGES + st), ((gi / TS_STAGES) - 1) & 1);
            int r0, c0;
            block_rc(gi / nch, r0, c0);
            const int kc = (gi % nch) * KC;
            const unsigned fb = bars + 8 * st, sb = base + st * TS_STAGE_B;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" :: "r"(fb), "r"(TS_STAGE_B) : "memory");
            const unsigned long long tm = reinterpret_cast<unsigned long long>(&tmap);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
#pragma unroll
                for (int j = 0; j < 2; ++j)
                    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
                                 :: "r"(sb + h * 16384 + j * 8192), "l"(tm), "r"(kc + 16 * h), "r"(r0 + 64 * j), "r"(fb) : "memory");
                asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
                             :: "r"(sb + 32768 + h * 8192), "l"(tm), "r"(kc + 16 * h), "r"(c0), "r"(fb) : "memory");
            }
        }
    };
    if (tid == 0) produce(PREF);
    unsigned sw[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) sw[q] = ((((2 * q) + (gc >> 1)) ^ gr) << 4) + ((gc & 1) << 3);
    int g = 0;
    for (int p = 0; p < P; ++p) {
        int r0, c0;
        block_rc(p, r0, c0);
        const int rows = min(2 * TB, ma - r0), cols = min(TB, ma - c0);
        double acc[2][8][2];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int nb = 0; nb < 8; ++nb) {
                const int r = 16 * wid + 8 * h + gr, c = 8 * nb + 2 * gc;
                acc[h][nb][0] = (r < rows && c < cols) ? -Sh[(size_t)(r0 + r) * ldh + c0 + c] : 0.0;
                acc[h][nb][1] = (r < rows && c + 1 < cols) ? -Sh[(size_t)(r0 + r) * ldh + c0 + c + 1] : 0.0;
            }
        for (int ch = 0; ch < nch; ++ch, ++g) {
            if (tid == 0) produce(g + PREF);
            const int st = g % TS_STAGES;
            mb_wait(bars + 8 * st, (g / TS_STAGES) & 1);
            const unsigned sb = base + st * TS_STAGE_B;
            const unsigned xa = sb + (16 * wid + gr) * 128, yb = sb + 32768 + gr * 128;
#pragma unroll
            for (int k4 = 0; k4 < KC / 4; ++k4) {
                const unsigned hx = (k4 >> 2) * 16384 + sw[k4 & 3], hy = (k4 >> 2) * 8192 + sw[k4 & 3];
                double a0, a1;
                asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(a0) : "r"(xa + hx));
                asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(a1) : "r"(xa + 1024 + hx));
#pragma unroll
                for (int nb = 0; nb < 8; ++nb) {
                    double bv;
                    asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(bv) : "r"(yb + nb * 1024 + hy));
                    dmma(acc[0][nb][0], acc[0][nb][1], a0, bv);
                    dmma(acc[1][nb][0], acc[1][nb][1], a1, bv);
                }
            }
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" :: "r"(bars + 8 * (TS_STAGES + st)) : "memory");
        }
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int nb = 0; nb < 8; ++nb) {
                const int r = 16 * wid + 8 * h + gr, c = 8 * nb + 2 * gc;
                if (r < rows && c < cols) Sh[(size_t)(r0 + r) * ldh + c0 + c] = -acc[h][nb][0];
                if (r < rows && c + 1 < cols) Sh[(size_t)(r0 + r) * ldh + c0 + c + 1] = -acc[h][nb][1];
            }
    }
    CYC1
}

template <int NSTG, int PREF>
__global__ void __launch_bounds__(NT, 1) k_tma_c(const __grid_constant__ CUtensorMap tmap, double *Sh, int ldh, int ma,
                                               int P, int nrow_pairs) {
    CYC0
    extern __shared__ unsigned char smraw[];
    const unsigned base = (su32(smraw) + 1023u) & ~1023u;
    const unsigned bars = base + NSTG * TS_STAGE_B + 65536;  // full[S], empty[S], cfull, cempty
    const unsigned cbase = base + NSTG * TS_STAGE_B;                  // C staging, 128 x 64 swizzled
    const unsigned cfull = bars + 16 * NSTG, cempty = cfull + 8;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, gr = lane >> 2, gc = lane & 3;
    constexpr int nch = 4 * TB / KC;
    const int G = P * nch;
    if (tid == 0) {
        for (int i = 0; i < NSTG; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" :: "r"(bars + 8 * i));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;\n" :: "r"(bars + 8 * (NSTG + i)));
        }
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" :: "r"(cfull));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;\n" :: "r"(cempty));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    auto block_rc = [&](int p, int &r0, int &c0) {
        const int b = blockIdx.x * P + p;
        r0 = (4 + 2 * (b % nrow_pairs)) * TB;
        c0 = (4 + (b / nrow_pairs) % ((ma / TB) - 4)) * TB;
    };
    int gi = 0;                                   // next chunk to issue (thread 0)
    auto produce = [&](int upto) {
        for (; gi < upto && gi < G; ++gi) {
            const int st = gi % NSTG;
            if (gi >= NSTG) mb_wait(bars + 8 * (NSTG + st), ((gi / NSTG) - 1) & 1);
            int r0, c0;
            block_rc(gi / nch, r0, c0);
            const int kc = (gi % nch) * KC;
            const unsigned fb = bars + 8 * st, sb = base + st * TS_STAGE_B;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" :: "r"(fb), "r"(TS_STAGE_B) : "memory");
            const unsigned long long tm = reinterpret_cast<unsigned long long>(&tmap);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
#pragma unroll
                for (int j = 0; j < 2; ++j)
                    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
                                 :: "r"(sb + h * 16384 + j * 8192), "l"(tm), "r"(kc + 16 * h), "r"(r0 + 64 * j), "r"(fb) : "memory");
                asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
                             :: "r"(sb + 32768 + h * 8192), "l"(tm), "r"(kc + 16 * h), "r"(c0), "r"(fb) : "memory");
            }
        }
    };
    auto produce_c = [&](int p) {                 // thread 0: C of block p into the staging buffer
        int r0, c0;
        block_rc(p, r0, c0);
        const unsigned long long tm = reinterpret_cast<unsigned long long>(&tmap);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" :: "r"(cfull), "r"(65536) : "memory");
        for (int g4 = 0; g4 < 4; ++g4)
            for (int j = 0; j < 2; ++j)
                asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
                             :: "r"(cbase + g4 * 16384 + j * 8192), "l"(tm), "r"(c0 + 16 * g4), "r"(r0 + 64 * j), "r"(cfull) : "memory");
    };
    if (tid == 0) { produce_c(0); produce(PREF); }
    unsigned sw[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) sw[q] = ((((2 * q) + (gc >> 1)) ^ gr) << 4) + ((gc & 1) << 3);
    int g = 0;
    for (int p = 0; p < P; ++p) {
        int r0, c0;
        block_rc(p, r0, c0);
        const int rows = min(2 * TB, ma - r0), cols = min(TB, ma - c0);
        double acc[2][8][2];
        mb_wait(cfull, p & 1);
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int nb = 0; nb < 8; ++nb) {
                const int r = 16 * wid + 8 * h + gr;
                const unsigned ad = cbase + (nb >> 1) * 16384 + r * 128 + ((((nb & 1) * 4 + gc) ^ gr) << 4);
                double v0, v1;
                asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v0), "=d"(v1) : "r"(ad));
                acc[h][nb][0] = -v0;
                acc[h][nb][1] = -v1;
            }
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" :: "r"(cempty) : "memory");
        if (tid == 0 && p + 1 < P) {
            mb_wait(cempty, p & 1);
            produce_c(p + 1);
        }
        for (int ch = 0; ch < nch; ++ch, ++g) {
            if (tid == 0) produce(g + PREF);
            const int st = g % NSTG;
            mb_wait(bars + 8 * st, (g / NSTG) & 1);
            const unsigned sb = base + st * TS_STAGE_B;
            const unsigned xa = sb + (16 * wid + gr) * 128, yb = sb + 32768 + gr * 128;
#pragma unroll
            for (int k4 = 0; k4 < KC / 4; ++k4) {
                const unsigned hx = (k4 >> 2) * 16384 + sw[k4 & 3], hy = (k4 >> 2) * 8192 + sw[k4 & 3];
                double a0, a1;
                asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(a0) : "r"(xa + hx));
                asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(a1) : "r"(xa + 1024 + hx));
#pragma unroll
                for (int nb = 0; nb < 8; ++nb) {
                    double bv;
                    asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(bv) : "r"(yb + nb * 1024 + hy));
                    dmma(acc[0][nb][0], acc[0][nb][1], a0, bv);
                    dmma(acc[1][nb][0], acc[1][nb][1], a1, bv);
                }
            }
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" :: "r"(bars + 8 * (NSTG + st)) : "memory");
        }
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int nb = 0; nb < 8; ++nb) {
                const int r = 16 * wid + 8 * h + gr, c = 8 * nb + 2 * gc;
                if (r < rows && c < cols) Sh[(size_t)(r0 + r) * ldh + c0 + c] = -acc[h][nb][0];
                if (r < rows && c + 1 < cols) Sh[(size_t)(r0 + r) * ldh + c0 + c + 1] = -acc[h][nb][1];
            }
    }
    CYC1
}

template <int PREF>
void run_tma(double *Sh, int ldh, int ma, int nsm, double clk_ghz) {
    static PFN_cuTensorMapEncodeTiled enc = nullptr;
    if (!enc) {
        cudaDriverEntryPointQueryResult q;
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
    }
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)ldh, (cuuint64_t)ma};
    cuuint64_t strides[1] = {(cuuint64_t)ldh * 8};
    cuuint32_t box[2] = {16, 64}, es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, Sh, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return; }
    cudaFuncSetAttribute(k_tma<PREF>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEMT);
    const int P = 24, nrow_pairs = (ma / TB - 4) / 2;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int it = 0; it < 4; ++it) {
        cudaEventRecord(e0);
        k_tma<PREF><<<nsm, NT, SMEMT>>>(tm, Sh, ldh, ma, P, nrow_pairs);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaError_t err = cudaGetLastError();
    const double us = best * 1e3 / P;
    const double ideal_us = 2.0 * 128 * 64 * 256 / (128.0 * clk_ghz * 1e3);
    printf("TMA 4-stage, %d chunks ahead: %.2f us per block, %.1f %% of the DMMA rate %s\n", PREF, us, 100.0 * ideal_us / us,
           err == cudaSuccess ? "" : cudaGetErrorString(err));
}

template <int NSTG, int PREF>
void run_tma_c(double *Sh, int ldh, int ma, int nsm, double clk_ghz) {
    static PFN_cuTensorMapEncodeTiled enc = nullptr;
    if (!enc) {
        cudaDriverEntryPointQueryResult q;
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
    }
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)ldh, (cuuint64_t)ma};
    cuuint64_t strides[1] = {(cuuint64_t)ldh * 8};
    cuuint32_t box[2] = {16, 64}, es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, Sh, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return; }
    cudaFuncSetAttribute(k_tma_c<NSTG, PREF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (NSTG * TS_STAGE_B + 65536 + 1024 + 64));
    const int P = 24, nrow_pairs = (ma / TB - 4) / 2;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int it = 0; it < 4; ++it) {
        cudaEventRecord(e0);
        k_tma_c<NSTG, PREF><<<nsm, NT, (NSTG * TS_STAGE_B + 65536 + 1024 + 64)>>>(tm, Sh, ldh, ma, P, nrow_pairs);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaError_t err = cudaGetLastError();
    const double us = best * 1e3 / P;
    const double ideal_us = 2.0 * 128 * 64 * 256 / (128.0 * clk_ghz * 1e3);
    printf("TMA %d-stage + C staging, %d chunks ahead: %.2f us per block, %.1f %% of the DMMA rate %s\n", NSTG, PREF, us, 100.0 * ideal_us / us,
           err == cudaSuccess ? "" : cudaGetErrorString(err));
}

int main() {
    int nsm, clk_khz;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    const int ma = 9024, ldh = 9024 + 8;
    double *Sh, *out;
    cudaMalloc(&Sh, sizeof(double) * (size_t)ma * ldh);
    cudaMemset(Sh, 0, sizeof(double) * (size_t)ma * ldh);
    cudaMalloc(&out, sizeof(double) * nsm * NT);
    const double ghz = clk_khz * 1e-6;
    printf("%d SMs, clock %.3f GHz, m %d\n", nsm, ghz, ma);
    run<0>(Sh, ldh, ma, nsm, out, ghz);
    run<1>(Sh, ldh, ma, nsm, out, ghz);
    run<2>(Sh, ldh, ma, nsm, out, ghz);
    run<4>(Sh, ldh, ma, nsm, out, ghz);
    run<3>(Sh, ldh, ma, nsm, out, ghz);
    run<7>(Sh, ldh, ma, nsm, out, ghz);
    run_tma<2>(Sh, ldh, ma, nsm, ghz);
    run_tma<3>(Sh, ldh, ma, nsm, ghz);
    run_tma_c<3, 2>(Sh, ldh, ma, nsm, ghz);
    return 0;
}
