#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace pdipc {
// stream-ordered zero fill / device copy as library kernels (bytes: multiples of 4)
cudaError_t dev_zero(void *p, size_t bytes, cudaStream_t st);
cudaError_t dev_copy(void *d, const void *s, size_t bytes, cudaStream_t st);
// three zero fills in one launch
cudaError_t dev_zero3(void *a, size_t ba, void *b, size_t bb, void *c, size_t bc, cudaStream_t st);
// out[0..n] : exclusive scan of in[0..n), out[n] = total.  scratch: scan_scratch_ints(n).
void scan_exclusive(const int *in, int *out, int n, int *scratch, cudaStream_t st);
// same with the length read on the device (*n_dev, at most cap; grid sized for cap)
void scan_exclusive_dev(const int *in, int *out, const int *n_dev, int cap, int *scratch, cudaStream_t st);
int scan_scratch_ints(int n);
// scan_exclusive of 0/1 marks that also writes the marked indices: idx[out[i]] = i, in[i] != 0
void scan_compact(const int *in, int *out, int *idx, int n, int *scratch, cudaStream_t st);
// scan_exclusive that also zeroes in[0..n) after reading it (n > 0)
void scan_exclusive_clear(int *in, int *out, int n, int *scratch, cudaStream_t st);
// ascending LSD radix sort of the low `bits` bits; tmp: n keys; scratch: radix_scratch_ints(n)
void radix_sort_u64(uint64_t *keys, uint64_t *tmp, int n, int bits, int *scratch,
                    cudaStream_t st);
int radix_scratch_ints(int nmax);
// out = unique(keys) for sorted keys; count at pos[n]; flags, pos: n+1 ints
void unique_sorted_u64(const uint64_t *keys, int n, uint64_t *out, int *flags, int *pos,
                       int *scratch, cudaStream_t st);
// *out = sum(part[0..n)) in a fixed order (one block)
void sum_partials(const double *part, int n, double *out, cudaStream_t st);
}  // namespace pdipc
