// init.cu -- the reference's exact-count Fisher-Yates init (kernels.py:26-45),
// computed in parallel with a bit-identical result.
//
// Sequential definition: a[k] = +1 for k < up, else -1; for i = n-1 .. 1:
// j_i = int(u_i * (i+1)) with u_i the draw at position pos0 + (n-1-i), then
// swap(a[i], a[j_i]).  Step i finalises a[i] (later steps only touch indices
// below i), so
//
//   final[i] = value at position j_i just before step i,
//   value at position p just before step t = val(w) where w is the most
//     recent earlier-executed writer of p -- the smallest step index w > t
//     with j_w = p -- or initial[p] if there is none,
//   val(x) = value at position x just before step x
//          = val(W(x)) with W(x) = smallest w > x with j_w = x, or initial[x].
//
// So with, per position p, the sorted list of steps that write p:
//   final[i] = val(succ(i)) or initial[j_i]   (succ: next larger step of the
//                                              same list as i)
//   final[0] = val(0),
// and val(x) follows W until it stops.  Steps: draw every j in parallel,
// count / scan / scatter them into per-position lists, sort each (short)
// list, resolve.  tests/test_gpu_init.py checks it against the sequential
// kernel and the oracle.
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"
#include "launchers.cuh"
#include "philox.cuh"

namespace ptmh {

struct FillBatch {
    int8_t* spins;        // rows of this batch, n sites each
    int64_t n, up;
    uint64_t seed, stream0, pos0;  // row b uses stream stream0 + b
    int32_t* j;           // (nb, n)      j[i], i >= 1
    int32_t* cnt;         // (nb, n)      counts, then scatter cursors
    int32_t* off;         // (nb, n + 1)  exclusive prefix of cnt
    int32_t* lst;         // (nb, n)      steps grouped by target position
    int32_t* succ;        // (nb, n)
    int32_t* wr;          // (nb, n)      W(p)
    int8_t* val;          // (nb, n)
    int32_t* bsum;        // (nb, nblk)   scan block sums
    int64_t nblk;
};

constexpr int kScanBlock = 1024;

__global__ void fy_draw(FillBatch F) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t b = blockIdx.y;
    if (i < 1 || i >= F.n) return;
    const uint64_t pos = F.pos0 + (uint64_t)(F.n - 1 - i);
    const double u = stream_uniform(F.seed, F.stream0 + (uint64_t)b, pos);
    const int32_t jj = (int32_t)__dmul_rn(u, (double)(i + 1));  // kernels.py:41
    F.j[b * F.n + i] = jj;
    atomicAdd(&F.cnt[b * F.n + jj], 1);
}

// exclusive scan of cnt (per row) into off; block-local pass
__global__ void fy_scan_blocks(FillBatch F) {
    __shared__ int32_t ws[32];
    const int64_t b = blockIdx.y;
    const int64_t k = (int64_t)blockIdx.x * kScanBlock + threadIdx.x;
    const int32_t v = (k < F.n) ? F.cnt[b * F.n + k] : 0;
    int32_t x = v;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) ws[w] = x;
    __syncthreads();
    if (w == 0) {
        int32_t t = ws[lane];
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
        }
        ws[lane] = t;
    }
    __syncthreads();
    const int32_t incl = x + (w > 0 ? ws[w - 1] : 0);
    if (k < F.n) F.off[b * (F.n + 1) + k] = incl - v;
    if (threadIdx.x == kScanBlock - 1) F.bsum[b * F.nblk + blockIdx.x] = incl;
}

__global__ void fy_scan_sums(FillBatch F) {  // one block per row: scan block sums
    const int64_t b = blockIdx.x;
    int32_t* bs = F.bsum + b * F.nblk;
    if (threadIdx.x == 0) {
        int32_t run = 0;
        for (int64_t q = 0; q < F.nblk; ++q) {
            const int32_t t = bs[q];
            bs[q] = run;
            run += t;
        }
        F.off[b * (F.n + 1) + F.n] = run;  // == n - 1
    }
}

__global__ void fy_scan_add(FillBatch F) {
    const int64_t b = blockIdx.y;
    const int64_t k = (int64_t)blockIdx.x * kScanBlock + threadIdx.x;
    if (k < F.n) F.off[b * (F.n + 1) + k] += F.bsum[b * F.nblk + blockIdx.x];
    if (k < F.n) F.cnt[b * F.n + k] = 0;  // reuse as scatter cursor
}

__global__ void fy_scatter(FillBatch F) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t b = blockIdx.y;
    if (i < 1 || i >= F.n) return;
    const int32_t p = F.j[b * F.n + i];
    const int32_t slot = F.off[b * (F.n + 1) + p] + atomicAdd(&F.cnt[b * F.n + p], 1);
    F.lst[b * F.n + slot] = (int32_t)i;
}

// per position: sort its (short) list, record successors and W(p)
__global__ void fy_lists(FillBatch F) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t b = blockIdx.y;
    if (p >= F.n) return;
    const int32_t* off = F.off + b * (F.n + 1);
    int32_t* l = F.lst + b * F.n;
    const int32_t lo = off[p], hi = off[p + 1];
    for (int32_t k = lo + 1; k < hi; ++k) {  // insertion sort
        const int32_t v = l[k];
        int32_t q = k - 1;
        while (q >= lo && l[q] > v) {
            l[q + 1] = l[q];
            --q;
        }
        l[q + 1] = v;
    }
    int32_t w = -1;
    for (int32_t k = lo; k < hi; ++k) {
        const int32_t v = l[k];
        F.succ[b * F.n + v] = (k + 1 < hi) ? l[k + 1] : -1;
        if (w < 0 && v > p) w = v;
    }
    F.wr[b * F.n + p] = w;
}

__global__ void fy_val(FillBatch F) {
    const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t b = blockIdx.y;
    if (x >= F.n) return;
    const int32_t* wr = F.wr + b * F.n;
    int64_t y = x;
    for (int32_t w = wr[y]; w >= 0; w = wr[y]) y = w;  // W(x) > x: terminates
    F.val[b * F.n + x] = (y < F.up) ? 1 : -1;
}

__global__ void fy_final(FillBatch F) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t b = blockIdx.y;
    if (i >= F.n) return;
    int8_t out;
    if (i == 0) {
        out = F.val[b * F.n];
    } else {
        const int32_t s = F.succ[b * F.n + i];
        out = (s >= 0) ? F.val[b * F.n + s] : ((F.j[b * F.n + i] < F.up) ? 1 : -1);
    }
    F.spins[b * F.n + i] = out;
}

int64_t fill_ws_bytes(int64_t n, int64_t rows_per_batch) {
    const int64_t nblk = (n + kScanBlock - 1) / kScanBlock;
    return rows_per_batch * (n * 4 * 5 + (n + 1) * 4 + n + nblk * 4) + 256;
}

int launch_fill_parallel(int8_t* spins, int64_t rows, int64_t n, int64_t up_count, uint64_t seed,
                         uint64_t stream0, uint64_t pos0, void* ws, int64_t ws_bytes, cudaStream_t s) {
    if (rows == 0) return PTMH_OK;
    if (n >= (int64_t(1) << 31)) {
        set_error("parallel fill: n must be < 2^31");
        return PTMH_ERR_ARG;
    }
    const int64_t per_row = fill_ws_bytes(n, 1);
    const int64_t nb = std::min<int64_t>(rows, ws_bytes / per_row);
    if (nb < 1) {
        set_error("parallel fill: workspace too small for one row");
        return PTMH_ERR_ARG;
    }
    const int64_t nblk = (n + kScanBlock - 1) / kScanBlock;
    char* p = static_cast<char*>(ws);
    auto take = [&](int64_t bytes) {
        char* q = p;
        p += (bytes + 255) & ~int64_t(255);
        return q;
    };
    FillBatch F{};
    F.n = n;
    F.up = up_count;
    F.seed = seed;
    F.nblk = nblk;
    F.j = reinterpret_cast<int32_t*>(take(nb * n * 4));
    F.cnt = reinterpret_cast<int32_t*>(take(nb * n * 4));
    F.off = reinterpret_cast<int32_t*>(take(nb * (n + 1) * 4));
    F.lst = reinterpret_cast<int32_t*>(take(nb * n * 4));
    F.succ = reinterpret_cast<int32_t*>(take(nb * n * 4));
    F.wr = reinterpret_cast<int32_t*>(take(nb * n * 4));
    F.val = reinterpret_cast<int8_t*>(take(nb * n));
    F.bsum = reinterpret_cast<int32_t*>(take(nb * nblk * 4));
    for (int64_t r0 = 0; r0 < rows; r0 += nb) {
        const int64_t m = std::min(nb, rows - r0);
        F.spins = spins + r0 * n;
        F.stream0 = stream0 + (uint64_t)r0;
        F.pos0 = pos0;
        const dim3 g(ceil_div(n, 256), (unsigned)m);
        PTMH_CUDA(cudaMemsetAsync(F.cnt, 0, (size_t)(m * n * 4), s));
        fy_draw<<<g, 256, 0, s>>>(F);
        fy_scan_blocks<<<dim3((unsigned)nblk, (unsigned)m), kScanBlock, 0, s>>>(F);
        fy_scan_sums<<<(unsigned)m, 32, 0, s>>>(F);
        fy_scan_add<<<dim3((unsigned)nblk, (unsigned)m), kScanBlock, 0, s>>>(F);
        fy_scatter<<<g, 256, 0, s>>>(F);
        fy_lists<<<g, 256, 0, s>>>(F);
        fy_val<<<g, 256, 0, s>>>(F);
        fy_final<<<g, 256, 0, s>>>(F);
        PTMH_LAUNCH_CHECK();
    }
    return PTMH_OK;
}

}  // namespace ptmh
