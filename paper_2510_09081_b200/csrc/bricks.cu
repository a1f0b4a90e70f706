// bricks.cu -- the A-buffer build through per-brick segment lists (capsule traversal).
// Replaces lv/abuffer.py:195-255 (_chunk_count_kernel, _write_kernel) and the per-chunk cursors of
// 281-328 (_second_pass) like abuffer.cu's scatter + ordering pass, with the same outputs bit for bit.
//
// Why.  The scatter pass pays one RETURNING global atomic and one scattered 4-byte store per incidence
// (segment x voxel) and the ordering pass then sorts every list: on B200 both sit at per-incidence floors
// (LSU round trips, instruction issue) that do not move with the grid size -- 20 ms for the 922 M
// incidences of the 10 M-segment / 512^3 set.  Here no global atomic and no sort touches an incidence:
//
//   1. k_bin<count>   every segment counts itself into the 8^3-voxel bricks its inflated box overlaps
//                     (fire-and-forget atomics, ~3-4 per segment instead of ~60-90 per segment);
//   2. k_bin_alloc    every brick reserves a range of the pair array (warp-aggregated allocator);
//   3. k_bin<fill>    the segments write their ids into the ranges;
//   4. k_brick_build  one WARP per brick.  It sorts the brick's segment ids (a few hundred; shared
//                     memory) and takes them 32 at a time in ascending order, one per lane.  A lane PLANS
//                     its segment's traversal restricted to the brick (the slabs of lv/voxelizer.py:180-206
//                     are random-access, see SlabPlan / slab_at); the slabs of all 32 segments are pooled and
//                     worked off 32 at a time, each -- an axis-aligned box of cells one cell thick -- ORed
//                     into its owner's 512-bit map of the brick (16 words in shared memory, column
//                     `owner`).  The warp then transposes the 32 x 32 bit matrix of every non-empty word
//                     with five shuffle stages: lane b now holds, for voxel 32 w + b, the mask of the lanes
//                     (= segments) that visit it, and appends them to the voxel's list bit by bit:
//                     ascending lane = ascending segment id, so every list comes out in the reference's
//                     order (lv/abuffer.py:313-317) by construction.  The tight index (see abuffer.cu) is
//                     written in the same sweep from a second map, filled row by row (rows pooled too).
//
// (A first version -- one 256-thread CTA per brick, lanes setting their bit of per-voxel masks with
// shared-memory atomicOr cell by cell, then one thread per voxel emitting -- was slower than scatter + order:
// 1.50 against 1.28 ms on C2, 24.8 against 20.1 ms on C4; 15 warp instructions per incidence at 14 of 32
// threads, the nested slab / row / cell loops of 32 different segments do not converge.)
//
// Tight fragments.  abuffer.cu proves "capsule of radius R misses the voxel's cube" per incidence with a
// separating-direction search (~70 flops).  Here the test is made once per ROW of the traversal: the cube
// grown by R in the maximum norm (a box, which contains the cube grown by R in the Euclidean norm) is hit
// by the segment for an interval of cells of the row, found with two slab clips (~35 flops per row of 3-4
// cells).  The box is a superset of the rounded cube (2-3 % more tight fragments at R = 0.2); the index
// stays conservative: a fragment left out can never yield an accepted hit (lv/raytracer.py:446-452).
#include "lvx_device.cuh"

namespace lvx {

constexpr int BR = 8, BR_LOG = 3, BR_VOX = BR * BR * BR;
constexpr int BM_WORDS = BR_VOX / 32;                       // words of a lane's bit map of the brick: word = (y >> 2) + 2 z, bit = x + 8 (y & 3)
constexpr uint32_t BB_SORT_CAP = 2 * BM_WORDS * 32;         // ids sorted in shared memory (the bit-map area, before use)
constexpr int BIN_HDR = 4;                                  // scratch words 0..1: pairs needed (u64); 2: brick count

// scratch layout (u32 words): header | cnt[nb] | start[nb] | cur[nb] | pairs[capacity]
struct BrickScratch {
    unsigned long long *total;
    uint32_t *cnt, *start, *cur, *pairs;
    int64_t cap;
};
static inline int64_t brick_count(int res) { const int64_t rb = (res + BR - 1) / BR; return rb * rb * rb; }
static inline BrickScratch carve(uint32_t *scratch, int res, int64_t pair_capacity) {
    const int64_t nb = (brick_count(res) + 3) & ~3LL;
    BrickScratch S;
    S.total = reinterpret_cast<unsigned long long *>(scratch);
    S.cnt = scratch + BIN_HDR;
    S.start = S.cnt + nb;
    S.cur = S.start + nb;
    S.pairs = S.cur + nb;
    S.cap = pair_capacity;
    return S;
}

// inflated voxel box of a segment, clamped to the grid; false = no cell at all.  The capsule traversal never
// leaves it: its minor ranges are clamped to exactly these bounds (lv/voxelizer.py:171-176) and its slabs run
// from floor(min - r) to ceil(max + r) - 1 along the major axis.
__device__ __forceinline__ bool seg_box(const d3 &a, const d3 &b, double rt, int res, int lo[3], int hi[3]) {
    lo[0] = (int)floor(fmin(a.x, b.x) - rt); hi[0] = (int)floor(fmax(a.x, b.x) + rt);
    lo[1] = (int)floor(fmin(a.y, b.y) - rt); hi[1] = (int)floor(fmax(a.y, b.y) + rt);
    lo[2] = (int)floor(fmin(a.z, b.z) - rt); hi[2] = (int)floor(fmax(a.z, b.z) + rt);
#pragma unroll
    for (int k = 0; k < 3; k++) {
        lo[k] = max(lo[k], 0); hi[k] = min(hi[k], res - 1);
        if (hi[k] < lo[k]) return false;
    }
    return true;
}

// Pass 1 / 3.  `vis3`: level 3 (8^3-voxel nodes) of the pyramid of the voxels that own fragments, or NULL:
// a brick without a single owner gets no pair (culled bundles' interiors, other ranks' screen tiles).
template <bool FILL>
__global__ void __launch_bounds__(256)
k_bin(const double *__restrict__ verts, const int32_t *__restrict__ segs, int64_t n_seg, double rt, int res,
      const uint8_t *__restrict__ vis3, BrickScratch S) {
    const int64_t si = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (si >= n_seg) return;
    const int64_t i = segs[si];
    const d3 a = ld3(verts + 3 * i), b = ld3(verts + 3 * i + 3);
    int lo[3], hi[3];
    if (!seg_box(a, b, rt, res, lo, hi)) return;
    const int rb = (res + BR - 1) >> BR_LOG;
    for (int bz = lo[2] >> BR_LOG; bz <= hi[2] >> BR_LOG; bz++)
        for (int by = lo[1] >> BR_LOG; by <= hi[1] >> BR_LOG; by++)
            for (int bx = lo[0] >> BR_LOG; bx <= hi[0] >> BR_LOG; bx++) {
                const uint32_t bi = (uint32_t)bx + (uint32_t)rb * ((uint32_t)by + (uint32_t)rb * (uint32_t)bz);
                if (vis3 && !vis3[bi]) continue;
                if (!FILL) atomicAdd(&S.cnt[bi], 1u);
                else {
                    const uint32_t pos = atomicAdd(&S.cur[bi], 1u);
                    if ((int64_t)pos < S.cap) S.pairs[pos] = (uint32_t)i;
                }
            }
}

// Pass 2: ranges of the pair array, in whatever order the warps arrive (a list's place does not matter).
__global__ void __launch_bounds__(256)
k_bin_alloc(int64_t nb, BrickScratch S) {
    const int64_t bi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const uint32_t c = bi < nb ? S.cnt[bi] : 0u;
    uint32_t inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += v;
    }
    unsigned long long base = 0;
    const uint32_t sum = __shfl_sync(0xffffffffu, inc, 31);
    if (lane == 31 && sum) base = atomicAdd(S.total, (unsigned long long)sum);
    base = __shfl_sync(0xffffffffu, base, 31);
    if (bi < nb) {
        // a start beyond 2^32 cannot be stored; the build refuses such a frame anyway (total > capacity)
        const unsigned long long st = base + (inc - c);
        const uint32_t s32 = st > 0xffffffffull ? 0xffffffffu : (uint32_t)st;
        S.start[bi] = s32;
        S.cur[bi] = s32;
    }
}

// The slabs of rows_capsule (lvx_device.cuh; zero-length segments: the box of rows_aabb) that lie inside the brick
// [bx0, bx0 + 8) x ..., each clamped to it, from the same arithmetic: f(lo[3], hi[3], axis) receives the cells
// lo .. hi (inclusive, grid coordinates by axis x, y, z) of one slab -- a box one cell thick along the major axis
// -- and the axis along which the reference's innermost loop runs (rows of the traversal).
// The reference walks the slabs of the major axis with the recurrence t0 <- t1, p0 <- p1
// (lv/voxelizer.py:189-206), but nothing in a slab depends on the walk: the first slab is [t_min, T1],
// T1 = min(t_max, floor(t_min + 1)); every later one starts at an integer t0 = c (its cell index) < t_max, ends
// at min(t_max, c + 1), and its entry point p0 is the previous slab's p1 = e + s * (t0 - t_min) -- the same
// expression on the same operands.  So the slabs of one brick are computed directly.
// SlabPlan = what a lane knows about its segment's slabs inside the brick: the constants of the traversal, where the
// walk enters the brick (t_start) and where its first slab there ends (T1), and how many slabs follow.  Slab q is
// computed from these alone (slab_at), by ANY lane: the slabs of the warp's 32 segments are pooled and worked off 32
// at a time, because a pair has anything from 1 to 8 of them and a lane-per-segment loop runs at a quarter of the
// warp's width.
struct SlabPlan {
    double t_min, t_max, e1, e2, s1, s2, r1, r2, t_start, T1;
    int lo_j, hi_j, lo_k, hi_k;     // minor ranges, grid coordinates, already clamped to the brick
    int c0;                         // box traversal: first slab
    int code;                       // a0 | a1 << 2 | a2 << 4 | box << 6
    int n_slab;

    __device__ __forceinline__ void init(const d3 &a, const d3 &b, double r, int res, int bx0, int by0, int bz0) {
        const d3 d{b.x - a.x, b.y - a.y, b.z - a.z};
        const bool box = d.x == 0.0 && d.y == 0.0 && d.z == 0.0;
        t_min = t_max = e1 = e2 = s1 = s2 = r1 = r2 = t_start = T1 = 0.0;
        c0 = 0; n_slab = 0;
        if (box) {      // lv/voxelizer.py:116-140 (zero-length segment): slabs along z, rows along x, fixed ranges
            code = 2 | (1 << 2) | (0 << 4) | (1 << 6);
            lo_k = max((int)floor(fmin(a.x, b.x) - r), bx0); hi_k = min((int)floor(fmax(a.x, b.x) + r), min(res, bx0 + BR) - 1);
            lo_j = max((int)floor(fmin(a.y, b.y) - r), by0); hi_j = min((int)floor(fmax(a.y, b.y) + r), min(res, by0 + BR) - 1);
            c0 = max((int)floor(fmin(a.z, b.z) - r), bz0);
            const int c_end = min((int)floor(fmax(a.z, b.z) + r), min(res, bz0 + BR) - 1) + 1;
            if (hi_k >= lo_k && hi_j >= lo_j) n_slab = max(c_end - c0, 0);
            return;
        }
        int a0, a1, a2;
        rank3(fabs(d.x), fabs(d.y), fabs(d.z), a0, a1, a2);
        code = a0 | (a1 << 2) | (a2 << 4);
        double d0 = sel(d, a0), d1 = sel(d, a1), d2 = sel(d, a2);
        double v0_0 = sel(a, a0), v0_1 = sel(a, a1), v0_2 = sel(a, a2);
        double v1_0 = sel(b, a0), v1_1 = sel(b, a1), v1_2 = sel(b, a2);
        if (d0 < 0.0) {
            double t;
            t = v0_0; v0_0 = v1_0; v1_0 = t;
            t = v0_1; v0_1 = v1_1; v1_1 = t;
            t = v0_2; v0_2 = v1_2; v1_2 = t;
            d0 = -d0; d1 = -d1; d2 = -d2;
        }
        s1 = d1 / d0; s2 = d2 / d0;
        t_min = v0_0 - 1.0 * r;
        t_max = v1_0 + 1.0 * r;
        e1 = v0_1 - s1 * r; e2 = v0_2 - s2 * r;
        r1 = r * sqrt(1.0 + s1 * s1);
        r2 = r * sqrt(1.0 + s2 * s2);
        const int B0 = a0 == 0 ? bx0 : (a0 == 1 ? by0 : bz0);
        const int B1 = a1 == 0 ? bx0 : (a1 == 1 ? by0 : bz0);
        const int B2 = a2 == 0 ? bx0 : (a2 == 1 ? by0 : bz0);
        lo_j = max((int)floor(fmin(v0_1, v1_1) - r), B1); hi_j = min((int)floor(fmax(v0_1, v1_1) + r), min(res, B1 + BR) - 1);
        lo_k = max((int)floor(fmin(v0_2, v1_2) - r), B2); hi_k = min((int)floor(fmax(v0_2, v1_2) + r), min(res, B2 + BR) - 1);
        const int c_end = min(res, B0 + BR);                                       // slabs B0 .. c_end - 1
        if (hi_j < lo_j || hi_k < lo_k) return;
        // enter the walk at the brick: at t_min if the first slab is not below the brick, else at the first integer
        // t0 >= B0 the walk reaches (every slab after the first starts at an integer)
        t_start = t_min;
        if (floor(t_min) < (double)B0) {
            const double T1r = fmin(t_max, floor(t_min + 1.0));
            t_start = T1r < t_max ? fmax(T1r, (double)B0) : t_max;
        }
        if (!(t_start < t_max) || !(floor(t_start) < (double)c_end)) return;
        T1 = fmin(t_max, floor(t_start + 1.0));                                    // end of the first slab in the brick
        n_slab = 1;
        if (T1 < t_max) n_slab += max(min((int)ceil(t_max), c_end) - (int)T1, 0);  // then one per integer T1, T1 + 1, ... < t_max
    }
};

// Slab q of a plan (its fields passed one by one: they come out of shuffles): cells [lo, hi] per axis, grid
// coordinates; false = the slab holds no cell of the brick.  The body of the reference's while loop.
__device__ __forceinline__ bool slab_at(int q, double t_min, double t_max, double e1, double e2, double s1, double s2,
                                        double r1, double r2, double t_start, double T1, int lo_j, int hi_j, int lo_k,
                                        int hi_k, int c0, int code, int lo[3], int hi[3]) {
    int j_min, j_max, k_min, k_max, c;
    if (code >> 6) {
        c = c0 + q;
        j_min = lo_j; j_max = hi_j; k_min = lo_k; k_max = hi_k;
    } else {
        const double t0 = q == 0 ? t_start : T1 + (double)(q - 1);
        c = (int)floor(t0);
        const double t1 = fmin(t_max, floor(t0 + 1.0));
        const double dt0 = t0 - t_min, dt = t1 - t_min;
        const double p0_1 = e1 + s1 * dt0, p0_2 = e2 + s2 * dt0;       // (= e1, e2 at t0 = t_min)
        const double p1_1 = e1 + s1 * dt, p1_2 = e2 + s2 * dt;
        j_min = max((int)floor(fmin(p0_1, p1_1) - r1), lo_j);
        j_max = min((int)floor(fmax(p0_1, p1_1) + r1), hi_j);
        k_min = max((int)floor(fmin(p0_2, p1_2) - r2), lo_k);
        k_max = min((int)floor(fmax(p0_2, p1_2) + r2), hi_k);
    }
    if (k_max < k_min || j_max < j_min) return false;
    const int a0 = code & 3, a1 = (code >> 2) & 3;
#pragma unroll
    for (int ax = 0; ax < 3; ax++) {
        lo[ax] = ax == a0 ? c : (ax == a1 ? j_min : k_min);
        hi[ax] = ax == a0 ? c : (ax == a1 ? j_max : k_max);
    }
    return true;
}

// Cells u in [u_lo, u_hi] of the row (cx, cy, cz) + u * e_axis (cell centres, in the segment's f32 frame) whose
// cube grown by h - 0.5 in the maximum norm is met by the segment; u_lo > u_hi = none.
struct SegBox {
    float a[3], e[3], inv[3];
};
// single-precision view of a segment in the frame of its brick (coordinates of a few voxels: rounded at ~1e-6), for
// the conservative tight test only
__device__ __forceinline__ SegBox make_segbox(const d3 &a, const d3 &b, int bx0, int by0, int bz0) {
    SegBox q;
    q.a[0] = (float)(a.x - bx0); q.a[1] = (float)(a.y - by0); q.a[2] = (float)(a.z - bz0);
    q.e[0] = (float)(b.x - a.x); q.e[1] = (float)(b.y - a.y); q.e[2] = (float)(b.z - a.z);
#pragma unroll
    for (int k = 0; k < 3; k++) q.inv[k] = fabsf(q.e[k]) > 1e-9f ? __fdividef(1.f, q.e[k]) : 1e30f;   // (a still coordinate: inside its slab or not)
    return q;
}
__device__ __forceinline__ void tight_cells(const SegBox &q, float cx, float cy, float cz, int axis, float h, int &u_lo, int &u_hi) {
    const float c[3] = {cx, cy, cz};
    float tA = 0.f, tB = 1.f, ar = 0.f, er = 0.f, cr = 0.f;
#pragma unroll
    for (int k = 0; k < 3; k++) {
        if (k == axis) { ar = q.a[k]; er = q.e[k]; cr = c[k]; }
        else {
            const float t1 = (c[k] - h - q.a[k]) * q.inv[k], t2 = (c[k] + h - q.a[k]) * q.inv[k];
            tA = fmaxf(tA, fminf(t1, t2));
            tB = fminf(tB, fmaxf(t1, t2));
        }
    }
    if (!(tA <= tB)) { u_lo = 1; u_hi = 0; return; }
    const float s1 = tA * er, s2 = tB * er;
    u_lo = (int)ceilf(ar + fminf(s1, s2) - h - cr);
    u_hi = (int)floorf(ar + fmaxf(s1, s2) + h - cr);
}

// all-ascending bitonic network on f[0..n) executed by the whole CTA; indices >= n act as +inf
__device__ void cta_bitonic(uint32_t *f, uint32_t n) {
    if (n < 2) return;
    int lg = 1;
    while ((1u << lg) < n) lg++;
    const uint32_t half = 1u << (lg - 1);
    for (int lk = 1; lk <= lg; lk++) {
        const uint32_t k = 1u << lk, hk = k >> 1;
        for (uint32_t t = threadIdx.x; t < half; t += blockDim.x) {
            const uint32_t blk = (t >> (lk - 1)) << lk, o = t & (hk - 1);
            const uint32_t i = blk + o, l = blk + k - 1 - o;
            if (l < n) {
                const uint32_t a = f[i], b = f[l];
                if (a > b) { f[i] = b; f[l] = a; }
            }
        }
        __syncthreads();
        for (int lj = lk - 2; lj >= 0; lj--) {
            const uint32_t j = 1u << lj;
            for (uint32_t t = threadIdx.x; t < half; t += blockDim.x) {
                const uint32_t i = ((t >> lj) << (lj + 1)) + (t & (j - 1)), l = i + j;
                if (l < n) {
                    const uint32_t a = f[i], b = f[l];
                    if (a > b) { f[i] = b; f[l] = a; }
                }
            }
            __syncthreads();
        }
    }
}

struct TightOut {
    uint32_t *frags;
    uint16_t *slot;
    uint16_t *cnt;
};

// transpose of the 32 x 32 bit matrix whose row `lane` is x: the result's bit i in lane b = bit b of lane i's x
__device__ __forceinline__ uint32_t transpose32(uint32_t x, int lane) {
    uint32_t m = 0x0000ffffu;
#pragma unroll
    for (int j = 16; j >= 1; j >>= 1) {
        const uint32_t y = __shfl_xor_sync(0xffffffffu, x, j);
        x = (lane & j) ? ((x & ~m) | ((y >> j) & m)) : ((x & m) | ((y << j) & ~m));
        m ^= m << (j >> 1);
    }
    return x;
}

// bits of the cells [x0, x1] x [y0, y1] (brick-local, 0..7) of one z-layer in the layer's two words (y < 4, y >= 4)
__device__ __forceinline__ void layer_bits(int x0, int x1, int y0, int y1, uint32_t &w_lo, uint32_t &w_hi) {
    const uint32_t xm = ((2u << (x1 - x0)) - 1u) << x0;                 // bits x0..x1 of one row
    const uint32_t rows = xm * 0x01010101u;                             // ... in all four rows of a word
    const int a0 = y0, a1 = min(y1, 3), b0 = max(y0, 4) - 4, b1 = y1 - 4;
    w_lo = a1 >= a0 ? rows & ((0xffffffffu >> (8 * (3 - (a1 - a0)))) << (8 * a0)) : 0u;
    w_hi = b1 >= b0 ? rows & ((0xffffffffu >> (8 * (3 - (b1 - b0)))) << (8 * b0)) : 0u;
}

#ifndef LVX_BRICK_MINB
#define LVX_BRICK_MINB 24
#endif
__global__ void __launch_bounds__(32, LVX_BRICK_MINB)
k_brick_build(const double *__restrict__ verts, double rt, float r_tight, int res, const uint32_t *__restrict__ offsets,
              uint32_t *__restrict__ frags, int64_t cap, const TightOut T, BrickScratch S, uint64_t *__restrict__ stats) {
    __shared__ uint32_t s_bm[2][BM_WORDS][32];      // [all | tight][word][lane]; before the chunks: the sort buffer
    __shared__ uint32_t s_base[BM_WORDS][32];       // per voxel (word w, bit = lane): list start
    __shared__ uint16_t s_nv[BM_WORDS][32], s_k[BM_WORDS][32], s_tk[BM_WORDS][32];   // list length, fragments / tight fragments so far
    __shared__ uint32_t s_ids[32];
    __shared__ uint32_t s_slab[BR][32];             // per lane: its slabs inside the brick (local box + row axis), see below
    __shared__ uint8_t s_cum[BR][32];               // ... and the running number of their rows
    const int lane = threadIdx.x;
    const unsigned long long need = *S.total;
    if (blockIdx.x == 0 && lane == 0) stats[LVX_ST_BRICK_PAIRS] = need;
    if ((int64_t)need > S.cap) return;               // the pair array was too small: the caller grows it and redoes the frame
    const uint32_t n = S.cnt[blockIdx.x];
    if (n == 0) return;
    const int rb = (res + BR - 1) >> BR_LOG;
    const int bx0 = (int)(blockIdx.x % rb) << BR_LOG, by0 = (int)((blockIdx.x / rb) % rb) << BR_LOG,
              bz0 = (int)(blockIdx.x / (rb * rb)) << BR_LOG;

    // ---- the voxels of this lane (bit `lane` of every word): list bounds
    const int vx = bx0 + (lane & 7), vy_lo = by0 + (lane >> 3);
    bool any = false;
    {
        // all 32 loads of the lane in flight together (the walk up the brick is a chain of dependent phases run by
        // ~20 warps per SM: 7 % of its stall samples sat on these loads when they went out four at a time)
        uint32_t bb[BM_WORDS], ee[BM_WORDS];
#pragma unroll
        for (int w = 0; w < BM_WORDS; w++) {
            const int y = vy_lo + 4 * (w & 1), z = bz0 + (w >> 1);
            bb[w] = 0; ee[w] = 0;
            if (vx < res && y < res && z < res) {
                const uint32_t idx = (uint32_t)vx + (uint32_t)res * ((uint32_t)y + (uint32_t)res * (uint32_t)z);
                bb[w] = offsets[idx];
                ee[w] = offsets[idx + 1];
            }
        }
#pragma unroll
        for (int w = 0; w < BM_WORDS; w++) {
            uint32_t nv = ee[w] - bb[w];
            if ((int64_t)ee[w] > cap) {               // never touch memory past the buffer: the frame is redone with a
                nv = 0;                               // larger one, but the tracer of THIS frame still runs
                if (T.cnt) {
                    const int y = vy_lo + 4 * (w & 1), z = bz0 + (w >> 1);
                    T.cnt[(uint32_t)vx + (uint32_t)res * ((uint32_t)y + (uint32_t)res * (uint32_t)z)] = 0;
                }
            }
            s_base[w][lane] = bb[w]; s_nv[w][lane] = (uint16_t)nv; s_k[w][lane] = 0; s_tk[w][lane] = 0;
            any |= nv != 0;
        }
    }
    if (!__any_sync(0xffffffffu, any)) return;       // nothing in this brick owns a fragment (culled / other tile)

    // ---- ascending segment ids
    uint32_t *ids = S.pairs + S.start[blockIdx.x];
    uint32_t *sortbuf = &s_bm[0][0][0];
    if (n <= 32) {                                    // one bitonic network in registers
        uint32_t v = (uint32_t)lane < n ? ids[lane] : 0xffffffffu;
#pragma unroll
        for (int lk = 1; lk <= 5; lk++)
#pragma unroll
            for (int lj = lk - 1; lj >= 0; lj--) {
                const uint32_t o = __shfl_xor_sync(0xffffffffu, v, 1 << lj);
                const bool keep_min = (((lane >> lk) ^ (lane >> lj)) & 1) == 0;
                v = keep_min ? min(v, o) : max(v, o);
            }
        if ((uint32_t)lane < n) ids[lane] = v;
    } else if (n <= BB_SORT_CAP) {
        for (uint32_t i = lane; i < n; i += 32) sortbuf[i] = ids[i];
        __syncwarp();
        cta_bitonic(sortbuf, n);
        for (uint32_t i = lane; i < n; i += 32) ids[i] = sortbuf[i];
    } else {
        cta_bitonic(ids, n);
    }
    __syncwarp();
#pragma unroll
    for (int w = 0; w < BM_WORDS; w++) { s_bm[0][w][lane] = 0; s_bm[1][w][lane] = 0; }

    const float h = 0.5f + r_tight + 1e-4f;
    const bool want_tight = T.frags != nullptr;

    for (uint32_t c0 = 0; c0 < n; c0 += 32) {
        const uint32_t me = c0 + lane;
        const uint32_t id = me < n ? ids[me] : 0xffffffffu;
        s_ids[lane] = id;
        if (me + 32 < n) {                            // the next chunk's end points: asked for a whole chunk ahead
            const uint32_t nid = ids[me + 32];
            asm volatile("prefetch.global.L2 [%0];" ::"l"(verts + 3 * (int64_t)nid));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(verts + 3 * (int64_t)nid + 5));
        }
        // ---- the slabs of the 32 segments, pooled: every lane plans its own segment, then the warp works the slabs
        // off 32 at a time whoever's they are.  A slab is ORed into its OWNER's bit map of all cells and kept
        // (20 bits) for the tight test.
        SegBox sb;
        uint32_t n_rows = 0;
        {
            d3 a{0, 0, 0}, b{0, 0, 0};
            if (me < n) { a = ld3(verts + 3 * (int64_t)id); b = ld3(verts + 3 * (int64_t)id + 3); }
            sb = make_segbox(a, b, bx0, by0, bz0);
            SlabPlan P;
            P.init(a, b, rt, res, bx0, by0, bz0);
            if (me >= n) P.n_slab = 0;
            uint32_t incl_s = (uint32_t)P.n_slab;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t v = __shfl_up_sync(0xffffffffu, incl_s, o);
                if (lane >= o) incl_s += v;
            }
            const uint32_t total_s = __shfl_sync(0xffffffffu, incl_s, 31);
            for (uint32_t g0 = 0; g0 < total_s; g0 += 32) {
                const uint32_t g = g0 + lane;
                int o = 0;                                        // owner = number of lanes whose slabs end at or before g
#pragma unroll
                for (int step = 16; step; step >>= 1) {
                    const uint32_t v = __shfl_sync(0xffffffffu, incl_s, o + step - 1);
                    if (v <= g) o += step;
                }
                const bool valid = g < total_s;
                o = min(o, 31);
                const uint32_t o_incl = __shfl_sync(0xffffffffu, incl_s, o);
                const int o_n = __shfl_sync(0xffffffffu, P.n_slab, o);
                const double t_min = __shfl_sync(0xffffffffu, P.t_min, o), t_max = __shfl_sync(0xffffffffu, P.t_max, o);
                const double e1 = __shfl_sync(0xffffffffu, P.e1, o), e2 = __shfl_sync(0xffffffffu, P.e2, o);
                const double s1 = __shfl_sync(0xffffffffu, P.s1, o), s2 = __shfl_sync(0xffffffffu, P.s2, o);
                const double r1 = __shfl_sync(0xffffffffu, P.r1, o), r2 = __shfl_sync(0xffffffffu, P.r2, o);
                const double t_start = __shfl_sync(0xffffffffu, P.t_start, o), T1 = __shfl_sync(0xffffffffu, P.T1, o);
                const int lo_j = __shfl_sync(0xffffffffu, P.lo_j, o), hi_j = __shfl_sync(0xffffffffu, P.hi_j, o);
                const int lo_k = __shfl_sync(0xffffffffu, P.lo_k, o), hi_k = __shfl_sync(0xffffffffu, P.hi_k, o);
                const int c0 = __shfl_sync(0xffffffffu, P.c0, o), code = __shfl_sync(0xffffffffu, P.code, o);
                if (valid) {
                    const int q = (int)(g - (o_incl - (uint32_t)o_n));
                    int lo[3], hi[3];
                    uint32_t desc = 0, rows = 0;
                    if (slab_at(q, t_min, t_max, e1, e2, s1, s2, r1, r2, t_start, T1, lo_j, hi_j, lo_k, hi_k, c0, code, lo, hi)) {
                        const int x0 = lo[0] - bx0, x1 = hi[0] - bx0, y0 = lo[1] - by0, y1 = hi[1] - by0, z0 = lo[2] - bz0, z1 = hi[2] - bz0;
                        uint32_t w_lo, w_hi;
                        layer_bits(x0, x1, y0, y1, w_lo, w_hi);
                        for (int z = z0; z <= z1; z++) {
                            if (w_lo) atomicOr(&s_bm[0][2 * z][o], w_lo);
                            if (w_hi) atomicOr(&s_bm[0][2 * z + 1][o], w_hi);
                        }
                        // rows of the slab = the reference's innermost loops, along a2: one per cell of the two other axes
                        const int axis = (code >> 4) & 3;
                        const int ex = axis == 0 ? 1 : x1 - x0 + 1, ey = axis == 1 ? 1 : y1 - y0 + 1, ez = axis == 2 ? 1 : z1 - z0 + 1;
                        rows = (uint32_t)(ex * ey * ez);
                        desc = (uint32_t)x0 | (uint32_t)x1 << 3 | (uint32_t)y0 << 6 | (uint32_t)y1 << 9 | (uint32_t)z0 << 12 |
                               (uint32_t)z1 << 15 | (uint32_t)axis << 18;
                    }
                    s_slab[q][o] = desc;
                    s_cum[q][o] = (uint8_t)rows;
                }
            }
            __syncwarp();
            for (int q = 0; q < P.n_slab; q++) {                  // running row counts of this lane's slabs
                n_rows += s_cum[q][lane];
                s_cum[q][lane] = (uint8_t)n_rows;
            }
        }
        __syncwarp();
        // ---- the rows of all 32 segments, 32 at a time whoever's they are: the cells of a row whose cube, grown by
        // r_tight in the maximum norm, the segment meets -> the owner's tight map
        if (want_tight) {
            uint32_t incl = n_rows;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += v;
            }
            const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
            for (uint32_t g0 = 0; g0 < total; g0 += 32) {
                const uint32_t g = g0 + lane;
                int o = 0;                                        // owner = number of lanes whose rows end at or before g
#pragma unroll
                for (int step = 16; step; step >>= 1) {
                    const uint32_t v = __shfl_sync(0xffffffffu, incl, o + step - 1);
                    if (v <= g) o += step;
                }
                const bool valid = g < total;
                o = min(o, 31);
                const uint32_t o_incl = __shfl_sync(0xffffffffu, incl, o), o_rows = __shfl_sync(0xffffffffu, n_rows, o);
                SegBox ob;
#pragma unroll
                for (int k = 0; k < 3; k++) {
                    ob.a[k] = __shfl_sync(0xffffffffu, sb.a[k], o);
                    ob.e[k] = __shfl_sync(0xffffffffu, sb.e[k], o);
                    ob.inv[k] = __shfl_sync(0xffffffffu, sb.inv[k], o);
                }
                if (valid) {
                    uint32_t local = g - (o_incl - o_rows);       // row of the owner
                    int sl = 0;
                    uint32_t before = 0;
                    for (;;) {
                        const uint32_t c = s_cum[sl][o];
                        if (local < c) break;
                        before = c; sl++;
                    }
                    local -= before;
                    const uint32_t d = s_slab[sl][o];
                    const int x0 = d & 7, x1 = (d >> 3) & 7, y0 = (d >> 6) & 7, y1 = (d >> 9) & 7, z0 = (d >> 12) & 7, z1 = (d >> 15) & 7;
                    const int axis = (int)(d >> 18);
                    // the slab is one cell thick along the major axis: its rows differ in ONE other coordinate
                    int cx = x0, cy = y0, cz = z0;
                    if (axis != 0 && x1 > x0) cx += (int)local;
                    else if (axis != 1 && y1 > y0) cy += (int)local;
                    else cz += (int)local;
                    const int n_row = axis == 0 ? x1 - x0 + 1 : (axis == 1 ? y1 - y0 + 1 : z1 - z0 + 1);
                    int u_lo, u_hi;
                    tight_cells(ob, (float)cx + 0.5f, (float)cy + 0.5f, (float)cz + 0.5f, axis, h, u_lo, u_hi);
                    u_lo = max(u_lo, 0); u_hi = min(u_hi, n_row - 1);
                    for (int u = u_lo; u <= u_hi; u++) {
                        const int ux = cx + (axis == 0 ? u : 0), uy = cy + (axis == 1 ? u : 0), uz = cz + (axis == 2 ? u : 0);
                        atomicOr(&s_bm[1][2 * uz + (uy >> 2)][o], 1u << (ux + 8 * (uy & 3)));
                    }
                }
            }
        }
        __syncwarp();
        // ---- per word: transpose, then lane b appends the segments of voxel 32 w + b in lane (= id) order
#pragma unroll 1
        for (int w = 0; w < BM_WORDS; w++) {
            const uint32_t v = s_bm[0][w][lane];
            if (!__any_sync(0xffffffffu, v != 0)) continue;
            const uint32_t tv = s_bm[1][w][lane];
            s_bm[0][w][lane] = 0; s_bm[1][w][lane] = 0;
            uint32_t vm = transpose32(v, lane);
            const uint32_t tm = transpose32(tv, lane);
            const uint32_t nv = s_nv[w][lane];
            if (!vm || !nv) continue;
            const uint32_t base = s_base[w][lane];
            uint32_t k = s_k[w][lane], tk = s_tk[w][lane];
            while (vm) {
                const int bpos = __ffs(vm) - 1;
                vm &= vm - 1;
                const uint32_t seg = s_ids[bpos];
                if (k < nv) {
                    frags[base + k] = seg;
                    if ((tm >> bpos) & 1u) {
                        T.frags[base + tk] = seg;
                        T.slot[base + tk] = (uint16_t)k;
                        tk++;
                    }
                }
                k++;
            }
            s_k[w][lane] = (uint16_t)min(k, 0xffffu); s_tk[w][lane] = (uint16_t)tk;
        }
        __syncwarp();
    }
    // ---- per voxel: tight count, the reference's count check (lv/abuffer.py:310-311)
    uint32_t n_long = 0;
    bool bad = false;
#pragma unroll 4
    for (int w = 0; w < BM_WORDS; w++) {
        const uint32_t nv = s_nv[w][lane];
        if (!nv) continue;
        const int y = vy_lo + 4 * (w & 1), z = bz0 + (w >> 1);
        const uint32_t idx = (uint32_t)vx + (uint32_t)res * ((uint32_t)y + (uint32_t)res * (uint32_t)z);
        if (T.cnt) T.cnt[idx] = s_tk[w][lane];
        bad |= s_k[w][lane] != nv;
        n_long += nv > 32;
    }
    if (bad) stats[LVX_ST_MISMATCH] = 1;
    n_long = __reduce_add_sync(0xffffffffu, n_long);
    if (lane == 0 && n_long) atomicAdd((unsigned long long *)&stats[LVX_ST_LONG_LISTS], (unsigned long long)n_long);
}

}  // namespace lvx

using namespace lvx;

extern "C" {

int64_t lvx_brick_scratch_words(int res, int64_t pair_capacity) {
    const int64_t nb = (brick_count(res) + 3) & ~3LL;
    return BIN_HDR + 3 * nb + (pair_capacity > 0 ? pair_capacity : 0);
}

int lvx_build_lists(const double *verts, const int32_t *segs, int64_t n_seg, double rt, double r_tight, int res,
                    const uint8_t *cull_flat, const uint32_t *offsets, uint32_t *frags, int64_t frag_capacity,
                    uint32_t *tight_frags, uint16_t *tight_slot, uint16_t *tight_cnt,
                    uint32_t *scratch, int64_t pair_capacity, uint64_t *stats, void *stream) {
    if (!pow2(res) || res < BR || !scratch || pair_capacity < 0 || pair_capacity > 0xfffffff0LL) return LVX_E_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    const bool want_tight = tight_frags != nullptr;
    if (want_tight != (tight_slot != nullptr) || want_tight != (tight_cnt != nullptr)) return LVX_E_ARG;
    const int64_t nb = brick_count(res);
    const BrickScratch S = carve(scratch, res, pair_capacity);
    const uint8_t *vis3 = nullptr;
    if (cull_flat) {
        const LevelOffsets L = make_level_offsets(res);
        vis3 = cull_flat + L.off[BR_LOG];
    }
    LVX_CUDA(cudaMemsetAsync(scratch, 0, (size_t)(BIN_HDR + ((nb + 3) & ~3LL)) * 4, s));
    if (n_seg > 0) k_bin<false><<<blocks_for(n_seg, 256), 256, 0, s>>>(verts, segs, n_seg, rt, res, vis3, S);
    k_bin_alloc<<<blocks_for(nb, 256), 256, 0, s>>>(nb, S);
    if (n_seg > 0) k_bin<true><<<blocks_for(n_seg, 256), 256, 0, s>>>(verts, segs, n_seg, rt, res, vis3, S);
    const TightOut T{tight_frags, tight_slot, tight_cnt};
    k_brick_build<<<(unsigned)nb, 32, 0, s>>>(verts, rt, want_tight ? (float)r_tight : -1.f, res, offsets, frags,
                                                     frag_capacity, T, S, stats);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

}  // extern "C"
