// Zero-copy PCIe probe (tools/ only): SM loads from / stores to pinned host
// memory, to size a plugin kernel that streams lattices without DMA copies.
#include <cstdint>
extern "C" __global__ void zc(const uint4* __restrict__ hin, uint4* __restrict__ hout,
                              const uint4* __restrict__ din, uint4* __restrict__ dout, long n, int mode) {
    const long stride = (long)gridDim.x * blockDim.x;
    for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += 4 * stride) {
        uint4 a[4], b[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const long j = i + q * stride;
            if (j < n) {
                if (mode & 1) a[q] = __ldcs(hin + j);
                if (mode & 2) b[q] = __ldcs(din + j);
            }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const long j = i + q * stride;
            if (j < n) {
                if (mode & 1) __stcs(dout + j, a[q]);
                if (mode & 2) __stcs(hout + j, b[q]);
            }
        }
    }
}
