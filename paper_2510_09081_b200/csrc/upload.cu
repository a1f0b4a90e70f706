// upload.cu -- line-set upload: voxel-unit vertices, segment ids, clip normals, AABB.
// Replaces lv/voxelizer.py:435-447 (segment_arrays), lv/lineset.py:74-79, 81-82, 213-242.
#include "lvx_device.cuh"

namespace lvx {

thread_local char g_err[256] = {0};
int cuda_fail(cudaError_t e, const char *where) {
    snprintf(g_err, sizeof(g_err), "%s: %s", where, cudaGetErrorString(e));
    return LVX_E_CUDA;
}

// polyline containing vertex i: largest p with off[p] <= i
__device__ __forceinline__ int64_t find_polyline(const int64_t *__restrict__ off, int64_t n_poly, int64_t i) {
    int64_t lo = 0, hi = n_poly;  // invariant off[lo] <= i < off[hi]
    while (hi - lo > 1) {
        int64_t mid = (lo + hi) >> 1;
        if (off[mid] <= i) lo = mid; else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ d3 wv(const float *__restrict__ v, int64_t i) {
    return d3{(double)v[3 * i], (double)v[3 * i + 1], (double)v[3 * i + 2]};
}
__device__ __forceinline__ d3 sub(const d3 &a, const d3 &b) { return d3{a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ double len3(const d3 &d) { return sqrt(d.x * d.x + d.y * d.y + d.z * d.z); }

// One thread per vertex.  Uniform polylines (the common case: off[p] = p*L) skip the search.
__global__ void __launch_bounds__(256)
k_upload(const float *__restrict__ v32, const int64_t *__restrict__ off, int64_t n_verts, int64_t n_poly,
         double wx, double wy, double wz, double vs, int64_t uniform_len,
         double *__restrict__ verts, float *__restrict__ verts_f, double *__restrict__ normals,
         int32_t *__restrict__ segs, uint64_t *__restrict__ stats) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_verts) return;
    const d3 w = wv(v32, i);
    // lv/voxelizer.py:438
    const double vx = (w.x - wx) / vs, vy = (w.y - wy) / vs, vz = (w.z - wz) / vs;
    verts[3 * i] = vx; verts[3 * i + 1] = vy; verts[3 * i + 2] = vz;
    if (verts_f) { verts_f[3 * i] = (float)vx; verts_f[3 * i + 1] = (float)vy; verts_f[3 * i + 2] = (float)vz; }
    const int64_t p = uniform_len > 0 ? i / uniform_len : find_polyline(off, n_poly, i);
    const int64_t s = off[p], e = off[p + 1];
    // lv/lineset.py:74-79: vertex i starts segment number i - p unless it ends its polyline
    if (i != e - 1) segs[i - p] = (int32_t)i;
    if (normals == nullptr) return;
    // lv/lineset.py:222-242
    d3 d;
    if (i == s) d = sub(wv(v32, s + 1), w);
    else if (i == e - 1) d = sub(w, wv(v32, e - 2));
    else d = sub(wv(v32, i + 1), wv(v32, i - 1));
    double len = len3(d);
    if (len == 0.0) {
        const int64_t m = e - s, li = i - s;
        const int64_t k = li < m - 2 ? li : m - 2;
        d = sub(wv(v32, s + k + 1), wv(v32, s + k));
        len = len3(d);
        if (len == 0.0) {
            bool found = false;
            for (int64_t j = 0; j < m - 1 && !found; j++) {
                d = sub(wv(v32, s + j + 1), wv(v32, s + j));
                len = len3(d);
                found = len > 0.0;
            }
            if (!found) {
                atomicMax((unsigned long long *)&stats[LVX_ST_DEGENERATE], (unsigned long long)(p + 1));
                d = d3{0, 0, 0};
                len = 1.0;
            }
        }
    }
    normals[3 * i] = d.x / len;
    normals[3 * i + 1] = d.y / len;
    normals[3 * i + 2] = d.z / len;
}

// order-preserving float <-> uint mapping so that min/max can use integer atomics
__device__ __forceinline__ uint32_t f2o(float f) {
    uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float o2f(uint32_t u) {
    return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

__global__ void k_aabb_init(uint32_t *acc) {
    if (threadIdx.x < 3) acc[threadIdx.x] = 0xffffffffu;
    else if (threadIdx.x < 6) acc[threadIdx.x] = 0u;
}

__global__ void __launch_bounds__(256)
k_aabb(const float *__restrict__ v, int64_t n_verts, uint32_t *__restrict__ acc) {
    float mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_verts;
         i += (int64_t)gridDim.x * blockDim.x)
        for (int a = 0; a < 3; a++) {
            float f = v[3 * i + a];
            mn[a] = fminf(mn[a], f);
            mx[a] = fmaxf(mx[a], f);
        }
    for (int a = 0; a < 3; a++)
        for (int o = 16; o > 0; o >>= 1) {
            mn[a] = fminf(mn[a], __shfl_xor_sync(0xffffffffu, mn[a], o));
            mx[a] = fmaxf(mx[a], __shfl_xor_sync(0xffffffffu, mx[a], o));
        }
    // one set of six atomics per block (the six target words are shared by the whole grid)
    __shared__ float s_mn[8][3], s_mx[8][3];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0)
        for (int a = 0; a < 3; a++) { s_mn[warp][a] = mn[a]; s_mx[warp][a] = mx[a]; }
    __syncthreads();
    if (threadIdx.x < 3) {
        const int a = threadIdx.x;
        float lo = s_mn[0][a], hi = s_mx[0][a];
        for (int w = 1; w < 8; w++) { lo = fminf(lo, s_mn[w][a]); hi = fmaxf(hi, s_mx[w][a]); }
        atomicMin(&acc[a], f2o(lo));
        atomicMax(&acc[3 + a], f2o(hi));
    }
}

__global__ void k_aabb_finish(uint32_t *acc) {
    if (threadIdx.x < 6) ((float *)acc)[threadIdx.x] = o2f(acc[threadIdx.x]);
}

__global__ void k_stats_reset(uint64_t *stats) {
    if (threadIdx.x < LVX_STATS_WORDS) stats[threadIdx.x] = 0;
}


// ----------------------------------------------------------------------------- processing order
// Voxelization and the A-buffer scatter produce the same output for any processing order of the
// segments (integer atomics; the ordering pass sorts every list).  Handing neighbouring threads
// segments of the same brick makes their atomics and 4-byte fragment stores fall into the same
// sectors at the same time: on C4 (10 M segments, 3.7 GB of fragments) the scatter's DRAM traffic
// was 11x the fragment bytes in polyline order.  One counting sort per frame: rank inside the
// brick from the histogram atomic, a single-block scan of the (few thousand) bins, a scatter.
__device__ __forceinline__ uint32_t brick_of(const double *__restrict__ verts, int64_t v, int res, int brick, int nb) {
    const int bx = min(max((int)floor(verts[3 * v]), 0), res - 1) / brick;
    const int by = min(max((int)floor(verts[3 * v + 1]), 0), res - 1) / brick;
    const int bz = min(max((int)floor(verts[3 * v + 2]), 0), res - 1) / brick;
    return (uint32_t)bx + (uint32_t)nb * ((uint32_t)by + (uint32_t)nb * (uint32_t)bz);
}

__global__ void __launch_bounds__(256)
k_order_hist(const double *__restrict__ verts, const int32_t *__restrict__ segs, int64_t n_seg, int res, int brick,
             int nb, uint32_t *__restrict__ hist, uint32_t *__restrict__ rank) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    // consecutive segments of a polyline mostly share their brick: one atomic per group of equal keys
    const uint32_t key = i < n_seg ? brick_of(verts, segs[i], res, brick, nb) : 0xffffffffu;
    const uint32_t same = __match_any_sync(0xffffffffu, key);
    const int lane = threadIdx.x & 31, leader = __ffs(same) - 1;
    uint32_t base = 0;
    if (lane == leader && i < n_seg) base = atomicAdd(&hist[key], (uint32_t)__popc(same));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (i < n_seg) rank[i] = base + __popc(same & ((1u << lane) - 1u));
}

// exclusive scan of n <= 2^20 bins by one block of 1024 threads (n is a few thousand)
__global__ void __launch_bounds__(1024)
k_order_scan(uint32_t *__restrict__ hist, int n) {
    __shared__ uint32_t s_warp[32];
    __shared__ uint32_t s_carry;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (int base = 0; base < n; base += 1024) {
        const int i = base + threadIdx.x;
        const uint32_t v = i < n ? hist[i] : 0u;
        uint32_t inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += u;
        }
        if (lane == 31) s_warp[warp] = inc;
        __syncthreads();
        if (warp == 0) {
            uint32_t w = s_warp[lane], wi = w;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t u = __shfl_up_sync(0xffffffffu, wi, o);
                if (lane >= o) wi += u;
            }
            s_warp[lane] = wi - w;
        }
        __syncthreads();
        const uint32_t carry = s_carry;
        if (i < n) hist[i] = carry + s_warp[warp] + inc - v;
        __syncthreads();
        if (threadIdx.x == 1023) s_carry = carry + s_warp[warp] + inc;
        __syncthreads();
    }
}

__global__ void __launch_bounds__(256)
k_order_scatter(const double *__restrict__ verts, const int32_t *__restrict__ segs, int64_t n_seg, int res, int brick,
                int nb, const uint32_t *__restrict__ start, const uint32_t *__restrict__ rank, int32_t *__restrict__ order) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_seg) return;
    const int32_t v = segs[i];
    order[start[brick_of(verts, v, res, brick, nb)] + rank[i]] = v;
}

}  // namespace lvx

using namespace lvx;

extern "C" {

const char *lvx_last_cuda_error(void) { return g_err; }
int lvx_version(void) { return 100; }

int lvx_num_levels(int res) {
    if (!pow2(res)) return LVX_E_ARG;
    return make_level_offsets(res).n_levels;
}
int64_t lvx_pyramid_elems(int res) {
    if (!pow2(res)) return LVX_E_ARG;
    LevelOffsets L = make_level_offsets(res);
    return L.off[L.n_levels];
}

int lvx_stats_reset(uint64_t *stats, void *stream) {
    k_stats_reset<<<1, 32, 0, (cudaStream_t)stream>>>(stats);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

int lvx_clear(void *ptr, int64_t bytes, void *stream) {
    LVX_CUDA(cudaMemsetAsync(ptr, 0, (size_t)bytes, (cudaStream_t)stream));
    return LVX_OK;
}

int lvx_upload(const float *verts_f32, const int64_t *poly_off, int64_t n_verts, int64_t n_poly,
               const double *world_min_host, double voxel_size, double *verts, float *verts_f,
               double *normals, int32_t *segs, uint64_t *stats, void *stream) {
    if (n_verts < 2 || n_poly < 1 || !(voxel_size > 0) || n_verts > 0x7fffffffLL) return LVX_E_ARG;
    // uniform-length hint: valid only if n_verts divides evenly; the kernel still reads off[p], so
    // a wrong hint cannot happen silently -- the host wrapper passes it only when verified.
    int64_t uniform = 0;
    k_upload<<<blocks_for(n_verts, 256), 256, 0, (cudaStream_t)stream>>>(
        verts_f32, poly_off, n_verts, n_poly, world_min_host[0], world_min_host[1], world_min_host[2],
        voxel_size, uniform, verts, verts_f, normals, segs, stats);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

int lvx_aabb(const float *verts_f32, int64_t n_verts, float *out6, void *stream) {
    if (n_verts < 1) return LVX_E_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    k_aabb_init<<<1, 32, 0, s>>>((uint32_t *)out6);
    unsigned nb = blocks_for(n_verts, 256 * 4);       // >= 4 vertices per thread
    if (nb > 148 * 4) nb = 148 * 4;
    if (nb < 1) nb = 1;
    k_aabb<<<nb, 256, 0, s>>>(verts_f32, n_verts, (uint32_t *)out6);
    k_aabb_finish<<<1, 32, 0, s>>>((uint32_t *)out6);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

int64_t lvx_segment_order_scratch_words(int64_t n_seg, int res, int brick) {
    if (!pow2(res) || brick < 1 || !pow2(brick) || brick > res) return LVX_E_ARG;
    const int64_t nb = res / brick;
    return nb * nb * nb + n_seg;
}

int lvx_segment_order(const double *verts, const int32_t *segs, int64_t n_seg, int res, int brick, int32_t *order,
                      uint32_t *scratch, void *stream) {
    if (!pow2(res) || brick < 1 || (brick & (brick - 1)) || brick > res || n_seg < 0 || n_seg > 0x7fffffffLL) return LVX_E_ARG;
    if (n_seg == 0) return LVX_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const int nb = res / brick;
    const int64_t bins = (int64_t)nb * nb * nb;
    if (bins > (1 << 20)) return LVX_E_ARG;
    uint32_t *hist = scratch, *rank = scratch + bins;
    LVX_CUDA(cudaMemsetAsync(hist, 0, (size_t)bins * 4, s));
    k_order_hist<<<blocks_for(n_seg, 256), 256, 0, s>>>(verts, segs, n_seg, res, brick, nb, hist, rank);
    k_order_scan<<<1, 1024, 0, s>>>(hist, (int)bins);
    k_order_scatter<<<blocks_for(n_seg, 256), 256, 0, s>>>(verts, segs, n_seg, res, brick, nb, hist, rank, order);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

}  // extern "C"
