// Device-wide primitives used by the contact pipeline: exclusive scan, LSD radix sort of
// 64-bit keys, unique.  Hand-written (no CUB); deterministic for a given input.
#include "prims.h"

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "dev_common.cuh"

namespace pdipc {

static long long g_launches = 0;     // handles are single-threaded (pd_ipc.h)
void note_launch() { ++g_launches; }
long long launch_count() { return g_launches; }
void add_launches(long long n) { g_launches += n; }
// ----------------------------------------------------------------------- fill / copy ------
// Stream-ordered zero fill and device copy as library kernels (not memset / memcpy nodes).
__global__ void k_zero32(unsigned *__restrict__ p, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = 0u;
}
__global__ void k_copy32(unsigned *__restrict__ d, const unsigned *__restrict__ s, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) d[i] = s[i];
}
static int fill_grid(size_t n) { return (int)std::min<size_t>((n + 255) / 256, 148 * 4); }
cudaError_t dev_zero(void *p, size_t bytes, cudaStream_t st) {
    const size_t n = bytes / 4;                  // callers pass multiples of 4 bytes
    if (n == 0) return cudaSuccess;
    PDI_LAUNCH(k_zero32, fill_grid(n), 256, 0, st)(static_cast<unsigned *>(p), n);
    return cudaGetLastError();
}
__global__ void k_zero32x3(unsigned *__restrict__ a, size_t na, unsigned *__restrict__ b, size_t nb,
                           unsigned *__restrict__ c, size_t nc) {
    const size_t i0 = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
    for (size_t i = i0; i < na; i += st) a[i] = 0u;
    for (size_t i = i0; i < nb; i += st) b[i] = 0u;
    for (size_t i = i0; i < nc; i += st) c[i] = 0u;
}
cudaError_t dev_zero3(void *a, size_t ba, void *b, size_t bb, void *c, size_t bc, cudaStream_t st) {
    const size_t n = std::max({ba, bb, bc}) / 4;
    if (n == 0) return cudaSuccess;
    PDI_LAUNCH(k_zero32x3, fill_grid(n), 256, 0, st)(static_cast<unsigned *>(a), ba / 4, static_cast<unsigned *>(b),
                                                     bb / 4, static_cast<unsigned *>(c), bc / 4);
    return cudaGetLastError();
}
cudaError_t dev_copy(void *d, const void *s, size_t bytes, cudaStream_t st) {
    const size_t n = bytes / 4;
    if (n == 0) return cudaSuccess;
    PDI_LAUNCH(k_copy32, fill_grid(n), 256, 0, st)(static_cast<unsigned *>(d), static_cast<const unsigned *>(s), n);
    return cudaGetLastError();
}

// ----------------------------------------------------------------------- exclusive scan ----
constexpr int kScanNT = 1024, kScanIPT = 4, kScanTile = kScanNT * kScanIPT;

template <int NT>
__device__ int block_exclusive_scan(int v, int *sh, int *total) {
    // warp inclusive scan
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sh[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int s = lane < NT / 32 ? sh[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < NT / 32) sh[lane] = s;
    }
    __syncthreads();
    int base = wid > 0 ? sh[wid - 1] : 0;
    if (total) *total = sh[NT / 32 - 1];
    __syncthreads();
    return base + x - v;
}

// n_dev != nullptr: the length is *n_dev (clamped to n, the capacity the grid was sized for)
__device__ __forceinline__ int scan_len(int n, const int *n_dev) { return n_dev ? min(*n_dev, n) : n; }

__global__ void __launch_bounds__(kScanNT) k_scan_partials(const int *in, int n, const int *n_dev, int *part) {
    __shared__ int sh[32];
    n = scan_len(n, n_dev);
    int base = blockIdx.x * kScanTile + threadIdx.x * kScanIPT;
    int s = 0;
#pragma unroll
    for (int i = 0; i < kScanIPT; ++i) s += (base + i < n) ? in[base + i] : 0;
    int tot;
    block_exclusive_scan<kScanNT>(s, sh, &tot);
    if (threadIdx.x == 0) part[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kScanNT) k_scan_tiles(int *in, int n, const int *n_dev, int *out,
                                                        const int *part, int nparts, int zero_in) {
    __shared__ int sh[32];
    __shared__ int off;
    n = scan_len(n, n_dev);
    if (threadIdx.x == 0) {
        int o = 0;
        for (int b = 0; b < (int)blockIdx.x; ++b) o += part[b];   // nparts is small
        off = o;
    }
    __syncthreads();
    int base = blockIdx.x * kScanTile + threadIdx.x * kScanIPT;
    int v[kScanIPT];
    int s = 0;
#pragma unroll
    for (int i = 0; i < kScanIPT; ++i) {
        v[i] = (base + i < n) ? in[base + i] : 0;
        s += v[i];
    }
    int tot;
    int ex = block_exclusive_scan<kScanNT>(s, sh, &tot) + off;
#pragma unroll
    for (int i = 0; i < kScanIPT; ++i) {
        if (base + i <= n) out[base + i] = ex;      // out[n] = total
        ex += v[i];
        if (zero_in && base + i < n) in[base + i] = 0;   // input consumed: cleared for reuse
    }
    (void)nparts;
}

__global__ void k_compact_marks(const int *__restrict__ mark, const int *__restrict__ pos, int n,
                                int *__restrict__ idx) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && mark[i]) idx[pos[i]] = i;
}
void scan_exclusive(const int *in, int *out, int n, int *scratch, cudaStream_t st);

// Small scans (capacity <= kScanSingleMax): ONE CTA walks tiles of kScanNT x 16 with a running
// carry -- one launch instead of two, no partials round trip.
constexpr int kScanSingleIPT = 16, kScanSingleTile = kScanNT * kScanSingleIPT, kScanSingleMax = 2 * kScanSingleTile;
__global__ void __launch_bounds__(kScanNT) k_scan_single(const int *__restrict__ in, int n, const int *n_dev,
                                                         int *__restrict__ out) {
    __shared__ int sh[32];
    n = scan_len(n, n_dev);
    int carry = 0;
    for (int t0 = 0; t0 <= n; t0 += kScanSingleTile) {   // covers index n (the total)
        const int base = t0 + threadIdx.x * kScanSingleIPT;
        int v[kScanSingleIPT];
        if (base + kScanSingleIPT <= n) {
            const int4 *p = reinterpret_cast<const int4 *>(in + base);
#pragma unroll
            for (int q = 0; q < kScanSingleIPT / 4; ++q) {
                const int4 x = p[q];
                v[4 * q] = x.x; v[4 * q + 1] = x.y; v[4 * q + 2] = x.z; v[4 * q + 3] = x.w;
            }
        } else {
#pragma unroll
            for (int i = 0; i < kScanSingleIPT; ++i) v[i] = base + i < n ? in[base + i] : 0;
        }
        int sum = 0;
#pragma unroll
        for (int i = 0; i < kScanSingleIPT; ++i) sum += v[i];
        int tot;
        int ex = block_exclusive_scan<kScanNT>(sum, sh, &tot) + carry;
#pragma unroll
        for (int i = 0; i < kScanSingleIPT; ++i) {
            if (base + i <= n) out[base + i] = ex;      // out[n] = total
            ex += v[i];
        }
        carry += tot;
    }
}

// exclusive scan of 0/1 marks that also compacts the marked indices: idx[out[i]] = i where
// in[i] != 0 (single block; n <= kScanSingleMax keeps it one or two tiles)
__global__ void __launch_bounds__(kScanNT) k_scan_compact(const int *__restrict__ in, int n, int *__restrict__ out,
                                                          int *__restrict__ idx) {
    __shared__ int sh[32];
    int carry = 0;
    for (int t0 = 0; t0 <= n; t0 += kScanSingleTile) {
        const int base = t0 + threadIdx.x * kScanSingleIPT;
        int v[kScanSingleIPT];
#pragma unroll
        for (int i = 0; i < kScanSingleIPT; ++i) v[i] = base + i < n ? in[base + i] : 0;
        int sum = 0;
#pragma unroll
        for (int i = 0; i < kScanSingleIPT; ++i) sum += v[i];
        int tot;
        int ex = block_exclusive_scan<kScanNT>(sum, sh, &tot) + carry;
#pragma unroll
        for (int i = 0; i < kScanSingleIPT; ++i) {
            if (base + i <= n) out[base + i] = ex;
            if (v[i]) idx[ex] = base + i;
            ex += v[i];
        }
        carry += tot;
    }
}
void scan_compact(const int *in, int *out, int *idx, int n, int *scratch, cudaStream_t st) {
    if (n <= kScanSingleMax) {
        PDI_LAUNCH(k_scan_compact, 1, kScanNT, 0, st)(in, n, out, idx);
        return;
    }
    scan_exclusive(in, out, n, scratch, st);
    PDI_LAUNCH(k_compact_marks, (n + 255) / 256, 256, 0, st)(in, out, n, idx);
}

void scan_exclusive(const int *in, int *out, int n, int *scratch, cudaStream_t st) {
    if (n <= 0) {
        dev_zero(out, sizeof(int), st);
        return;
    }
    if (n <= kScanSingleMax) {
        PDI_LAUNCH(k_scan_single, 1, kScanNT, 0, st)(in, n, nullptr, out);
        return;
    }
    int nb = n / kScanTile + 1;                      // covers index n (the total)
    PDI_LAUNCH(k_scan_partials, nb, kScanNT, 0, st)(in, n, nullptr, scratch);
    PDI_LAUNCH(k_scan_tiles, nb, kScanNT, 0, st)(const_cast<int *>(in), n, nullptr, out, scratch, nb, 0);
}

void scan_exclusive_dev(const int *in, int *out, const int *n_dev, int cap, int *scratch, cudaStream_t st) {
    if (cap <= kScanSingleMax) {
        PDI_LAUNCH(k_scan_single, 1, kScanNT, 0, st)(in, cap, n_dev, out);
        return;
    }
    int nb = cap / kScanTile + 1;
    PDI_LAUNCH(k_scan_partials, nb, kScanNT, 0, st)(in, cap, n_dev, scratch);
    PDI_LAUNCH(k_scan_tiles, nb, kScanNT, 0, st)(const_cast<int *>(in), cap, n_dev, out, scratch, nb, 0);
}

// exclusive scan that also clears its input (large arrays: the two-pass scan; n > 0)
void scan_exclusive_clear(int *in, int *out, int n, int *scratch, cudaStream_t st) {
    int nb = n / kScanTile + 1;
    PDI_LAUNCH(k_scan_partials, nb, kScanNT, 0, st)(in, n, nullptr, scratch);
    PDI_LAUNCH(k_scan_tiles, nb, kScanNT, 0, st)(in, n, nullptr, out, scratch, nb, 1);
}

int scan_scratch_ints(int n) { return n / kScanTile + 2; }

// ----------------------------------------------------------------------- radix sort -------
constexpr int kRsNT = 256, kRsIPT = 16, kRsTile = kRsNT * kRsIPT, kRsWarps = kRsNT / 32;

__global__ void __launch_bounds__(kRsNT) k_rs_hist(const uint64_t *keys, int n, int shift,
                                                   int *hist, int nblocks) {
    __shared__ int h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const int base = blockIdx.x * kRsTile;
#pragma unroll 4
    for (int i = 0; i < kRsIPT; ++i) {
        int idx = base + i * kRsNT + threadIdx.x;
        if (idx < n) atomicAdd(&h[(int)((keys[idx] >> shift) & 255u)], 1);
    }
    __syncthreads();
    hist[threadIdx.x * nblocks + blockIdx.x] = h[threadIdx.x];
}

__global__ void __launch_bounds__(kRsNT) k_rs_scatter(const uint64_t *in, uint64_t *out, int n,
                                                      int shift, const int *offs, int nblocks) {
    __shared__ int base[256];
    __shared__ int wcnt[kRsWarps][256];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    base[tid] = offs[tid * nblocks + blockIdx.x];
    const unsigned lt = (1u << lane) - 1u;
    const int tb = blockIdx.x * kRsTile;
    for (int i = 0; i < kRsIPT; ++i) {
        int idx = tb + i * kRsNT + tid;
        bool valid = idx < n;
        uint64_t k = valid ? in[idx] : 0;
        int d = valid ? (int)((k >> shift) & 255u) : 256 + lane;
#pragma unroll
        for (int w = 0; w < kRsWarps; ++w) wcnt[w][tid] = 0;
        __syncthreads();
        unsigned peers = __match_any_sync(0xffffffffu, d);
        int rank = __popc(peers & lt);
        if (valid && rank == 0) wcnt[wid][d] = __popc(peers);
        __syncthreads();
        {
            int run = base[tid];
#pragma unroll
            for (int w = 0; w < kRsWarps; ++w) {
                int c = wcnt[w][tid];
                wcnt[w][tid] = run;
                run += c;
            }
            base[tid] = run;
        }
        __syncthreads();
        if (valid) out[wcnt[wid][d] + rank] = k;
        __syncthreads();
    }
}

int radix_scratch_ints(int nmax) {
    int nb = (nmax + kRsTile - 1) / kRsTile;
    if (nb < 1) nb = 1;
    return 2 * 256 * nb + 1 + scan_scratch_ints(256 * nb);
}

// Sorts keys[0..n) ascending by their low `bits` bits (higher bits must be zero or are
// ignored); result in keys.  tmp: n uint64; scratch: radix_scratch_ints(n) ints.
void radix_sort_u64(uint64_t *keys, uint64_t *tmp, int n, int bits, int *scratch,
                    cudaStream_t st) {
    if (n <= 1 || bits <= 0) return;
    int nb = (n + kRsTile - 1) / kRsTile;
    int *hist = scratch;
    int *offs = scratch + 256 * nb;
    int *sscr = offs + 256 * nb + 1;
    uint64_t *src = keys, *dst = tmp;
    int passes = (bits + 7) / 8;
    for (int p = 0; p < passes; ++p) {
        int shift = 8 * p;
        PDI_LAUNCH(k_rs_hist, nb, kRsNT, 0, st)(src, n, shift, hist, nb);
        scan_exclusive(hist, offs, 256 * nb, sscr, st);
        PDI_LAUNCH(k_rs_scatter, nb, kRsNT, 0, st)(src, dst, n, shift, offs, nb);
        uint64_t *t = src;
        src = dst;
        dst = t;
    }
    if (src != keys) dev_copy(keys, src, sizeof(uint64_t) * n, st);
}

// ----------------------------------------------------------------------- unique -----------
__global__ void k_unique_flags(const uint64_t *k, int n, int *flag) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) flag[i] = (i == 0 || k[i] != k[i - 1]) ? 1 : 0;
}

__global__ void k_unique_write(const uint64_t *k, int n, const int *pos, uint64_t *out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && (i == 0 || k[i] != k[i - 1])) out[pos[i]] = k[i];
}

void unique_sorted_u64(const uint64_t *keys, int n, uint64_t *out, int *flags, int *pos,
                       int *scratch, cudaStream_t st) {
    if (n <= 0) {
        dev_zero(pos, sizeof(int), st);
        return;
    }
    int nb = (n + 255) / 256;
    PDI_LAUNCH(k_unique_flags, nb, 256, 0, st)(keys, n, flags);
    scan_exclusive(flags, pos, n, scratch, st);
    PDI_LAUNCH(k_unique_write, nb, 256, 0, st)(keys, n, pos, out);
}

// ----------------------------------------------------------------------- reductions -------
__global__ void k_sum_partials(const double *part, int n, double *out) {
    // one block, fixed order: deterministic
    __shared__ double sh[32];
    double s = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s += part[i];
    s = block_sum<1024>(s, sh);
    if (threadIdx.x == 0) *out = s;
}

void sum_partials(const double *part, int n, double *out, cudaStream_t st) {
    PDI_LAUNCH(k_sum_partials, 1, 1024, 0, st)(part, n, out);
}

}  // namespace pdipc
