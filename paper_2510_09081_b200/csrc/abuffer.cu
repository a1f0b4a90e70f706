// abuffer.cu -- per-frame acceleration structure: per-voxel segment lists restricted to visible
// voxels.  Replaces lv/abuffer.py:104-114 (scan_offsets) and 195-255, 281-328 (_chunk_count_kernel,
// _write_kernel, _second_pass).
//
//   count (already in base>>16)  ->  single-pass decoupled-look-back scan  ->  scatter with an
//   atomic cursor  ->  per-voxel ordering pass.
// The reference's per-chunk cursors make every list ascending in segment index
// (lv/abuffer.py:313-317; pinned by its tests, test_abuffer.py:114-122).  A segment visits a voxel
// at most once, so sorting each list reproduces the reference's `fragments` array bit for bit
// (SURVEY.md §7 H2).  The reference's extra counting traversal (_chunk_count_kernel) exists only
// to rebuild deterministic cursors and to assert determinism; here the assertion is the
// cursor==end check in the ordering pass (LVX_ST_MISMATCH -> ABufferError on the host).
#include "lvx_device.cuh"

namespace lvx {

// ----------------------------------------------------------------------------- scan
constexpr int SCAN_THREADS = 512;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;
constexpr uint64_t FLAG_AGG = 1ull << 62, FLAG_INC = 2ull << 62, VAL_MASK = (1ull << 62) - 1;

__global__ void __launch_bounds__(SCAN_THREADS)
k_scan(const uint32_t *__restrict__ base, const uint8_t *__restrict__ cull, int64_t V,
       uint32_t *__restrict__ offsets, unsigned long long *__restrict__ state, uint64_t *__restrict__ stats) {
    __shared__ uint32_t s_tile;
    __shared__ uint32_t s_warp[SCAN_THREADS / 32];
    __shared__ uint64_t s_prefix;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // tiles are numbered in the order they start running, so a tile only ever waits for tiles
    // that are already resident (forward progress without co-residency assumptions)
    if (tid == 0) s_tile = (uint32_t)atomicAdd(&state[0], 1ull);
    __syncthreads();
    const int64_t tile = s_tile;
    unsigned long long *st = state + 1;
    const int64_t i0 = tile * SCAN_TILE + (int64_t)tid * SCAN_ITEMS;

    uint32_t c[SCAN_ITEMS];
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; k++) c[k] = 0;
    if (i0 < V) {   // V is a multiple of 8, so a thread's 8 items are all in or all out
        const uint4 w0 = *reinterpret_cast<const uint4 *>(base + i0);
        const uint4 w1 = *reinterpret_cast<const uint4 *>(base + i0 + 4);
        c[0] = w0.x >> 16; c[1] = w0.y >> 16; c[2] = w0.z >> 16; c[3] = w0.w >> 16;
        c[4] = w1.x >> 16; c[5] = w1.y >> 16; c[6] = w1.z >> 16; c[7] = w1.w >> 16;
        if (cull) {   // lv/abuffer.py:107-108
            const uint2 m = *reinterpret_cast<const uint2 *>(cull + i0);
#pragma unroll
            for (int k = 0; k < 4; k++) {
                if (((m.x >> (8 * k)) & 0xFFu) == 0) c[k] = 0;
                if (((m.y >> (8 * k)) & 0xFFu) == 0) c[4 + k] = 0;
            }
        }
    }
    uint32_t tsum = 0;
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; k++) tsum += c[k];
    // block-level exclusive scan of the per-thread sums (max 4096*65535 < 2^32)
    uint32_t inc = tsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t n = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += n;
    }
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < SCAN_THREADS / 32 ? s_warp[lane] : 0;
        uint32_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t n = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += n;
        }
        if (lane < SCAN_THREADS / 32) s_warp[lane] = wi - w;   // exclusive warp prefix
        const uint64_t agg = __shfl_sync(0xffffffffu, wi, SCAN_THREADS / 32 - 1);
        uint64_t excl = 0;
        if (tile == 0) {
            if (lane == 0) atomicExch(&st[0], FLAG_INC | agg);
        } else {
            if (lane == 0) atomicExch(&st[tile], FLAG_AGG | agg);
            int64_t j = tile - 1;
            for (;;) {
                const int64_t jj = j - lane;
                uint64_t v = FLAG_INC;   // virtual tile -1: inclusive prefix 0
                if (jj >= 0) v = *reinterpret_cast<volatile unsigned long long *>(&st[jj]);
                const uint32_t flag = (uint32_t)(v >> 62);
                const uint32_t bal_inc = __ballot_sync(0xffffffffu, flag == 2);
                const uint32_t bal_inv = __ballot_sync(0xffffffffu, flag == 0);
                const int first_inc = bal_inc ? __ffs(bal_inc) - 1 : 32;
                const uint32_t need = first_inc >= 31 ? 0xffffffffu : ((2u << first_inc) - 1u);
                if (bal_inv & need) continue;   // a predecessor we need has not published yet
                uint64_t contrib = lane <= first_inc ? (v & VAL_MASK) : 0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) contrib += __shfl_xor_sync(0xffffffffu, contrib, o);
                excl += contrib;
                if (first_inc < 32) break;
                j -= 32;
            }
            if (lane == 0) atomicExch(&st[tile], FLAG_INC | ((excl + agg) & VAL_MASK));
        }
        if (lane == 0) {
            s_prefix = excl;
            if ((tile + 1) * SCAN_TILE >= V) {   // last tile: total
                offsets[V] = (uint32_t)(excl + agg);
                stats[LVX_ST_FRAG_TOTAL] = excl + agg;
            }
        }
    }
    __syncthreads();
    if (i0 < V) {
        uint32_t run = (uint32_t)s_prefix + s_warp[warp] + (inc - tsum);
        uint32_t o[SCAN_ITEMS];
#pragma unroll
        for (int k = 0; k < SCAN_ITEMS; k++) { o[k] = run; run += c[k]; }
        *reinterpret_cast<uint4 *>(offsets + i0) = make_uint4(o[0], o[1], o[2], o[3]);
        *reinterpret_cast<uint4 *>(offsets + i0 + 4) = make_uint4(o[4], o[5], o[6], o[7]);
    }
}

// ----------------------------------------------------------------------------- scatter
// lv/abuffer.py:226-255 _write_kernel.  The hierarchical segment rejection (_segment_visible,
// 145-181) is an acceleration only -- culled voxels are skipped per cell (252-253) -- so the
// output does not depend on it.
__global__ void __launch_bounds__(128)
k_scatter(const double *__restrict__ verts, const int32_t *__restrict__ segs, int64_t n_seg, double rt,
          int res, int method, const uint8_t *__restrict__ cull0, uint32_t *__restrict__ cursor,
          uint32_t *__restrict__ frags, int64_t cap) {
    const int64_t si = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (si >= n_seg) return;
    const int64_t i = segs[si];
    const d3 a = ld3(verts + 3 * i), b = ld3(verts + 3 * i + 3);
    const int64_t res64 = res;
    for_each_cell(method, a, b, rt, res, [&](int x, int y, int z) {
        const int64_t idx = x + res64 * (y + res64 * z);
        if (cull0 && cull0[idx] == 0) return;
        const uint32_t pos = atomicAdd(&cursor[idx], 1u);
        if ((int64_t)pos < cap) frags[pos] = (uint32_t)i;
    });
}

// ----------------------------------------------------------------------------- ordering

// all-ascending bitonic network on f[0..n) executed by one warp; indices >= n act as +inf
__device__ void warp_bitonic(uint32_t *f, uint32_t n, int lane) {
    int lg = 1;
    while ((1u << lg) < n) lg++;
    const uint32_t half = 1u << (lg - 1);
    for (int lk = 1; lk <= lg; lk++) {                 // merge size k = 2^lk
        const uint32_t k = 1u << lk, hk = k >> 1;
        for (uint32_t t = lane; t < half; t += 32) {   // flip: i <-> mirror inside the k-block
            const uint32_t blk = (t >> (lk - 1)) << lk, o = t & (hk - 1);
            const uint32_t i = blk + o, l = blk + k - 1 - o;
            if (l < n) {
                const uint32_t a = f[i], b = f[l];
                if (a > b) { f[i] = b; f[l] = a; }
            }
        }
        __syncwarp();
        for (int lj = lk - 2; lj >= 0; lj--) {         // disperse: i <-> i + 2^lj
            const uint32_t j = 1u << lj;
            for (uint32_t t = lane; t < half; t += 32) {
                const uint32_t i = ((t >> lj) << (lj + 1)) + (t & (j - 1)), l = i + j;
                if (l < n) {
                    const uint32_t a = f[i], b = f[l];
                    if (a > b) { f[i] = b; f[l] = a; }
                }
            }
            __syncwarp();
        }
    }
}

// Ordering pass over the compacted list of visible voxels (the only voxels that own fragments).
// One warp sorts one list at a time, two lists in flight per iteration for memory-level
// parallelism:
//   n <= 32 : one coalesced 128-byte load, a bitonic network in registers (warp shuffles, depth
//             chosen from n), one coalesced store -- skipped when the list is already ascending;
//   n  > 32 : staged through shared memory (or sorted in place when it exceeds the stage) with
//             the all-ascending bitonic network above.
// HBM traffic is <= 8 B per fragment, every access coalesced.
constexpr int ORDER_WARPS = 8;
constexpr int ORDER_CAP = 512;   // fragments staged per warp for long lists (2 KiB)

// bitonic sort of one value per lane (ascending by lane), network truncated to LG stages:
// sorts the first 2^LG lanes when the rest hold +inf
template <int LG>
__device__ __forceinline__ uint32_t warp_sort(uint32_t v, int lane) {
#pragma unroll
    for (int lk = 1; lk <= LG; lk++) {
#pragma unroll
        for (int lj = lk - 1; lj >= 0; lj--) {
            const uint32_t o = __shfl_xor_sync(0xffffffffu, v, 1 << lj);
            // keep the smaller value on the lower lane of an ascending block
            const bool keep_min = (((lane >> lk) ^ (lane >> lj)) & 1) == 0;
            v = keep_min ? min(v, o) : max(v, o);
        }
    }
    return v;
}

__device__ __forceinline__ void sort_short(uint32_t *f, uint32_t nn, uint32_t val, int lane) {
    const uint32_t next = __shfl_down_sync(0xffffffffu, val, 1);
    if (__ballot_sync(0xffffffffu, lane + 1 < nn && val > next) == 0) return;   // already ascending
    if (nn <= 4) val = warp_sort<2>(val, lane);
    else if (nn <= 8) val = warp_sort<3>(val, lane);
    else if (nn <= 16) val = warp_sort<4>(val, lane);
    else val = warp_sort<5>(val, lane);
    if (lane < nn) f[lane] = val;
}

__global__ void __launch_bounds__(ORDER_WARPS * 32)
k_order(const uint32_t *__restrict__ offsets, const uint32_t *__restrict__ cursor,
        const uint32_t *__restrict__ vis_list, uint32_t *__restrict__ frags, int64_t cap,
        uint64_t *__restrict__ stats) {
    __shared__ uint32_t stage[ORDER_WARPS][ORDER_CAP];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t n_lists = (int64_t)*reinterpret_cast<const unsigned long long *>(vis_list);
    const int64_t warp_id = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    uint32_t n_long = 0;
    // each warp takes a contiguous chunk of 32 list entries per step: lane k reads entry k's bounds
    for (int64_t e0 = warp_id * 32; e0 < n_lists; e0 += n_warps * 32) {
        uint32_t b = 0, n = 0;
        if (e0 + lane < n_lists) {
            const uint32_t v = vis_list[LVX_LIST_HDR + e0 + lane];
            b = offsets[v];
            const uint32_t e = offsets[v + 1];
            n = e - b;
            if (cursor[v] != e) stats[LVX_ST_MISMATCH] = 1;   // lv/abuffer.py:310-311
            if ((int64_t)e > cap) n = 0;                      // never touch memory past the buffer
        }
        uint32_t work = __ballot_sync(0xffffffffu, n > 1);
        n_long += __popc(__ballot_sync(0xffffffffu, n > 32));
        while (work) {
            // two lists per iteration: both loads are issued before either sort
            const int s0 = __ffs(work) - 1;
            work &= work - 1;
            const int s1 = work ? __ffs(work) - 1 : -1;
            if (s1 >= 0) work &= work - 1;
            const uint32_t b0 = __shfl_sync(0xffffffffu, b, s0), n0 = __shfl_sync(0xffffffffu, n, s0);
            const uint32_t b1 = __shfl_sync(0xffffffffu, b, s1 < 0 ? 0 : s1);
            const uint32_t n1 = s1 < 0 ? 0 : __shfl_sync(0xffffffffu, n, s1 < 0 ? 0 : s1);
            uint32_t v0 = 0xffffffffu, v1 = 0xffffffffu;
            if (n0 <= 32 && lane < n0) v0 = frags[b0 + lane];
            if (n1 <= 32 && lane < n1) v1 = frags[b1 + lane];
#pragma unroll
            for (int k = 0; k < 2; k++) {
                const uint32_t bb = k ? b1 : b0, nn = k ? n1 : n0;
                if (nn < 2) continue;
                uint32_t *f = frags + bb;
                if (nn <= 32) sort_short(f, nn, k ? v1 : v0, lane);
                else if (nn <= ORDER_CAP) {
                    uint32_t *buf = stage[warp];
                    for (uint32_t i = lane; i < nn; i += 32) buf[i] = f[i];
                    __syncwarp();
                    warp_bitonic(buf, nn, lane);
                    for (uint32_t i = lane; i < nn; i += 32) f[i] = buf[i];
                    __syncwarp();
                } else {
                    warp_bitonic(f, nn, lane);
                }
            }
        }
    }
    if (lane == 0 && n_long)
        atomicAdd((unsigned long long *)&stats[LVX_ST_LONG_LISTS], (unsigned long long)n_long);
}

__global__ void __launch_bounds__(256)
k_copy_u32(const uint32_t *__restrict__ src, uint32_t *__restrict__ dst, int64_t n) {
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
    if (i + 3 < n) *reinterpret_cast<uint4 *>(dst + i) = *reinterpret_cast<const uint4 *>(src + i);
    else for (int64_t k = i; k < n; k++) dst[k] = src[k];
}

}  // namespace lvx

using namespace lvx;

extern "C" {

int64_t lvx_scan_scratch_bytes(int64_t n_voxels) {
    const int64_t tiles = (n_voxels + SCAN_TILE - 1) / SCAN_TILE;
    return (tiles + 1) * 8;
}

int lvx_scan(const uint32_t *base, const uint8_t *cull_base, int64_t n_voxels, uint32_t *offsets,
             void *scratch, uint64_t *stats, void *stream) {
    if (n_voxels < 8 || (n_voxels & 7)) return LVX_E_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t tiles = (n_voxels + SCAN_TILE - 1) / SCAN_TILE;
    LVX_CUDA(cudaMemsetAsync(scratch, 0, (size_t)lvx_scan_scratch_bytes(n_voxels), s));
    k_scan<<<(unsigned)tiles, SCAN_THREADS, 0, s>>>(base, cull_base, n_voxels, offsets,
                                                   (unsigned long long *)scratch, stats);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

int lvx_scatter(const double *verts, const int32_t *segs, int64_t n_seg, double rt, int res, int method,
                const uint8_t *cull_flat, const uint32_t *vis_list, const uint32_t *offsets, uint32_t *cursor,
                uint32_t *frags, int64_t frag_capacity, uint64_t *stats, void *stream) {
    if (!vis_list) return LVX_E_ARG;
    if (!pow2(res) || method < 0 || method > 2) return LVX_E_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t V = (int64_t)res * res * res;
    k_copy_u32<<<blocks_for((V + 3) / 4, 256), 256, 0, s>>>(offsets, cursor, V);
    if (n_seg > 0)
        k_scatter<<<blocks_for(n_seg, 128), 128, 0, s>>>(verts, segs, n_seg, rt, res, method, cull_flat, cursor,
                                                        frags, frag_capacity);
    {
        unsigned nb = 148 * 8;   // persistent: 148 SMs x 8 CTAs of 8 warps
        const unsigned need = blocks_for((V + 31) / 32, ORDER_WARPS);
        if (nb > need) nb = need;
        k_order<<<nb, ORDER_WARPS * 32, 0, s>>>(offsets, cursor, vis_list, frags, frag_capacity, stats);
    }
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

}  // extern "C"
