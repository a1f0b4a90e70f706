// lvx_device.cuh -- device-side building blocks shared by the sm_100a kernels.
//
// Everything that decides voxel membership runs in IEEE f64 and is compiled with
// -fmad=false, in the reference's operation order, so integer outputs are
// bit-identical to the numba reference.  Reference citations: lv/ = pkg/src/linevox/.
#pragma once
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>

#include "../../include/lvx.h"

namespace lvx {

// ----------------------------------------------------------------------------- host helpers
extern thread_local char g_err[256];
int cuda_fail(cudaError_t e, const char *where);
#define LVX_CUDA(call)                                         \
    do {                                                       \
        cudaError_t e_ = (call);                               \
        if (e_ != cudaSuccess) return lvx::cuda_fail(e_, #call); \
    } while (0)
#define LVX_LAUNCH_CHECK() LVX_CUDA(cudaGetLastError())

static inline bool pow2(int r) { return r >= 2 && (r & (r - 1)) == 0; }
static inline unsigned blocks_for(int64_t n, int threads) { return (unsigned)((n + threads - 1) / threads); }

// ----------------------------------------------------------------------------- small math
struct d3 { double x, y, z; };
__device__ __forceinline__ double sel(const d3 &v, int a) { return a == 0 ? v.x : (a == 1 ? v.y : v.z); }
__device__ __forceinline__ d3 ld3(const double *p) { return d3{p[0], p[1], p[2]}; }

// lv/voxelizer.py:89-106 _rank3: major axis first, ties keep x before y before z
__device__ __forceinline__ void rank3(double ax, double ay, double az, int &a0, int &a1, int &a2) {
    int m = 0, r1, r2;
    if (ay > ax && ay >= az) m = 1;
    else if (az > ax && az > ay) m = 2;
    if (m == 0) { r1 = 1; r2 = 2; }
    else if (m == 1) { r1 = 0; r2 = 2; }
    else { r1 = 0; r2 = 1; }
    double vr2 = (r2 == 1) ? ay : az;
    double vr1 = (r1 == 0) ? ax : ay;
    a0 = m;
    if (vr2 > vr1) { a1 = r2; a2 = r1; } else { a1 = r1; a2 = r2; }
}

// ----------------------------------------------------------------------------- traversal
// Calls f(x, y, z) for every IN-GRID cell of the segment's traversal, each exactly once.
// Nothing is materialised: slabs are enumerated arithmetically (the reference builds a heap
// list per segment, lv/voxelizer.py:180-206).  Out-of-grid cells are skipped by clamping the
// loop bounds, which is what the callers' `continue` does (lv/voxelizer.py:321-322).

// Row form: f(x, y, z, axis, len) receives the cells (x, y, z) + u * e_axis, u in [0, len), of one
// innermost loop of the traversal, so that callers can issue the memory operations of a whole row
// (typically 3-4 cells) back to back instead of one dependent atomic at a time.

template <class F>
__device__ __forceinline__ void rows_aabb(const d3 &v0, const d3 &v1, double r, int res, F &&f) {
    // lv/voxelizer.py:116-140
    int x0 = (int)floor(fmin(v0.x, v1.x) - r), x1 = (int)floor(fmax(v0.x, v1.x) + r);
    int y0 = (int)floor(fmin(v0.y, v1.y) - r), y1 = (int)floor(fmax(v0.y, v1.y) + r);
    int z0 = (int)floor(fmin(v0.z, v1.z) - r), z1 = (int)floor(fmax(v0.z, v1.z) + r);
    x0 = max(x0, 0); y0 = max(y0, 0); z0 = max(z0, 0);
    x1 = min(x1, res - 1); y1 = min(y1, res - 1); z1 = min(z1, res - 1);
    if (x1 < x0) return;
    for (int z = z0; z <= z1; z++)
        for (int y = y0; y <= y1; y++) f(x0, y, z, 0, x1 - x0 + 1);
}

template <class F>
__device__ __forceinline__ void rows_capsule(const d3 &a, const d3 &b, double r, int res, F &&f) {
    // lv/voxelizer.py:143-206 (Algorithm 1 of the paper)
    d3 d{b.x - a.x, b.y - a.y, b.z - a.z};
    if (d.x == 0.0 && d.y == 0.0 && d.z == 0.0) { rows_aabb(a, b, r, res, f); return; }
    int a0, a1, a2;
    rank3(fabs(d.x), fabs(d.y), fabs(d.z), a0, a1, a2);
    double d0 = sel(d, a0), d1 = sel(d, a1), d2 = sel(d, a2);
    // v0 = start in the +major direction
    double v0_0 = sel(a, a0), v0_1 = sel(a, a1), v0_2 = sel(a, a2);
    double v1_0 = sel(b, a0), v1_1 = sel(b, a1), v1_2 = sel(b, a2);
    if (d0 < 0.0) {
        double t;
        t = v0_0; v0_0 = v1_0; v1_0 = t;
        t = v0_1; v0_1 = v1_1; v1_1 = t;
        t = v0_2; v0_2 = v1_2; v1_2 = t;
        d0 = -d0; d1 = -d1; d2 = -d2;
    }
    const double s1 = d1 / d0, s2 = d2 / d0;      // s[a0] == 1 exactly
    const double t_min = v0_0 - 1.0 * r;          // v0e[a0] = v0 - s*r with s = d0/d0 = 1
    const double t_max = v1_0 + 1.0 * r;
    const double e1 = v0_1 - s1 * r, e2 = v0_2 - s2 * r;  // v0e minor components
    const double r1 = r * sqrt(1.0 + s1 * s1);
    const double r2 = r * sqrt(1.0 + s2 * s2);
    int lo_j = (int)floor(fmin(v0_1, v1_1) - r), hi_j = (int)floor(fmax(v0_1, v1_1) + r);
    int lo_k = (int)floor(fmin(v0_2, v1_2) - r), hi_k = (int)floor(fmax(v0_2, v1_2) + r);
    lo_j = max(lo_j, 0); lo_k = max(lo_k, 0);
    hi_j = min(hi_j, res - 1); hi_k = min(hi_k, res - 1);
    double t0 = t_min, p0_1 = e1, p0_2 = e2;
    while (t0 < t_max) {
        const double t1 = fmin(t_max, floor(t0 + 1.0));
        const double dt = t1 - t_min;
        const double p1_1 = e1 + s1 * dt, p1_2 = e2 + s2 * dt;
        const int ci = (int)floor(t0);
        if (ci >= 0 && ci < res) {
            int j_min = max((int)floor(fmin(p0_1, p1_1) - r1), lo_j);
            int j_max = min((int)floor(fmax(p0_1, p1_1) + r1), hi_j);
            int k_min = max((int)floor(fmin(p0_2, p1_2) - r2), lo_k);
            int k_max = min((int)floor(fmax(p0_2, p1_2) + r2), hi_k);
            if (k_max >= k_min)
                for (int j = j_min; j <= j_max; j++) {
                    const int x = a0 == 0 ? ci : (a1 == 0 ? j : k_min);
                    const int y = a0 == 1 ? ci : (a1 == 1 ? j : k_min);
                    const int z = a0 == 2 ? ci : (a1 == 2 ? j : k_min);
                    f(x, y, z, a2, k_max - k_min + 1);
                }
        }
        t0 = t1; p0_1 = p1_1; p0_2 = p1_2;
    }
}

// The same traversal as a state machine: next() hands out the rows of rows_capsule (zero-length
// segments: rows_aabb) one at a time, in the same order, from the same arithmetic.  A warp can so step
// the traversals of its 32 segments in lockstep and pool their rows (k_scatter_rows).
struct RowGen {
    double t_min, t_max, e1, e2, s1, s2, r1, r2;     // constants of the segment (capsule form)
    double t0, p0_1, p0_2;                           // slab state
    int lo_j, hi_j, lo_k, hi_k, res;
    int a0, a1, a2;
    int ci, j, j_max, k_min, len;                    // rows j..j_max of the current slab
    bool box, done;

    __device__ __forceinline__ void init(const d3 &a, const d3 &b, double r, int res_) {
        res = res_; done = false; j = 1; j_max = 0; ci = 0; k_min = 0; len = 0;
        const d3 d{b.x - a.x, b.y - a.y, b.z - a.z};
        box = d.x == 0.0 && d.y == 0.0 && d.z == 0.0;
        if (box) {      // rows_aabb: slabs = z, rows = y, cells along x
            int x0 = (int)floor(fmin(a.x, b.x) - r), x1 = (int)floor(fmax(a.x, b.x) + r);
            int y0 = (int)floor(fmin(a.y, b.y) - r), y1 = (int)floor(fmax(a.y, b.y) + r);
            int z0 = (int)floor(fmin(a.z, b.z) - r), z1 = (int)floor(fmax(a.z, b.z) + r);
            x0 = max(x0, 0); y0 = max(y0, 0); z0 = max(z0, 0);
            x1 = min(x1, res - 1); y1 = min(y1, res - 1); z1 = min(z1, res - 1);
            a0 = 2; a1 = 1; a2 = 0;
            lo_j = y0; hi_j = y1; lo_k = x0; hi_k = x1;
            ci = z0 - 1; t0 = (double)z1;            // (t0 doubles as the last slab here)
            if (x1 < x0) done = true;
            t_min = t_max = e1 = e2 = s1 = s2 = r1 = r2 = p0_1 = p0_2 = 0.0;
            return;
        }
        rank3(fabs(d.x), fabs(d.y), fabs(d.z), a0, a1, a2);
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
        lo_j = (int)floor(fmin(v0_1, v1_1) - r); hi_j = (int)floor(fmax(v0_1, v1_1) + r);
        lo_k = (int)floor(fmin(v0_2, v1_2) - r); hi_k = (int)floor(fmax(v0_2, v1_2) + r);
        lo_j = max(lo_j, 0); lo_k = max(lo_k, 0);
        hi_j = min(hi_j, res - 1); hi_k = min(hi_k, res - 1);
        t0 = t_min; p0_1 = e1; p0_2 = e2;
    }
    __device__ __forceinline__ bool finished() const { return done && j > j_max; }
    __device__ __forceinline__ void advance() {
        j = 1; j_max = 0;
        if (box) {
            if ((double)ci >= t0) { done = true; return; }
            ci++;
            if (hi_j >= lo_j) { j = lo_j; j_max = hi_j; k_min = lo_k; len = hi_k - lo_k + 1; }
            return;
        }
        if (!(t0 < t_max)) { done = true; return; }
        const double t1 = fmin(t_max, floor(t0 + 1.0));
        const double dt = t1 - t_min;
        const double p1_1 = e1 + s1 * dt, p1_2 = e2 + s2 * dt;
        ci = (int)floor(t0);
        if (ci >= 0 && ci < res) {
            const int j_min = max((int)floor(fmin(p0_1, p1_1) - r1), lo_j);
            const int jm = min((int)floor(fmax(p0_1, p1_1) + r1), hi_j);
            const int km = max((int)floor(fmin(p0_2, p1_2) - r2), lo_k);
            const int k_max = min((int)floor(fmax(p0_2, p1_2) + r2), hi_k);
            if (k_max >= km) { j = j_min; j_max = jm; k_min = km; len = k_max - km + 1; }
        }
        t0 = t1; p0_1 = p1_1; p0_2 = p1_2;
    }
    // one step: at most one slab advance, at most one row (x, y, z) + u * e_axis, u in [0, n)
    __device__ __forceinline__ bool next(int &x, int &y, int &z, int &axis, int &n) {
        if (j > j_max && !done) advance();
        if (j > j_max) return false;
        x = a0 == 0 ? ci : (a1 == 0 ? j : k_min);
        y = a0 == 1 ? ci : (a1 == 1 ? j : k_min);
        z = a0 == 2 ? ci : (a1 == 2 ? j : k_min);
        axis = a2; n = len;
        j++;
        return true;
    }
};

template <class F>
__device__ __forceinline__ void cells_aabb(const d3 &v0, const d3 &v1, double r, int res, F &&f) {
    rows_aabb(v0, v1, r, res, [&](int x, int y, int z, int, int len) { for (int u = 0; u < len; u++) f(x + u, y, z); });
}

template <class F>
__device__ __forceinline__ void cells_capsule(const d3 &a, const d3 &b, double r, int res, F &&f) {
    rows_capsule(a, b, r, res, [&](int x, int y, int z, int axis, int len) {
        for (int u = 0; u < len; u++) f(x + (axis == 0 ? u : 0), y + (axis == 1 ? u : 0), z + (axis == 2 ? u : 0));
    });
}

template <class F>
__device__ __forceinline__ void cells_dda(const d3 &v0, const d3 &v1, int res, F &&f) {
    // lv/voxelizer.py:209-251
    int x = (int)floor(v0.x), y = (int)floor(v0.y), z = (int)floor(v0.z);
    const int ex = (int)floor(v1.x), ey = (int)floor(v1.y), ez = (int)floor(v1.z);
    const int steps = abs(ex - x) + abs(ey - y) + abs(ez - z);
    auto emit = [&](int X, int Y, int Z) {
        if (X >= 0 && Y >= 0 && Z >= 0 && X < res && Y < res && Z < res) f(X, Y, Z);
    };
    emit(x, y, z);
    if (steps == 0) return;
    const double dx = v1.x - v0.x, dy = v1.y - v0.y, dz = v1.z - v0.z;
    const int sx = dx > 0 ? 1 : -1, sy = dy > 0 ? 1 : -1, sz = dz > 0 ? 1 : -1;
    const double big = 1e30;
    double tmx = dx != 0.0 ? ((double)(x + (sx > 0 ? 1 : 0)) - v0.x) / dx : big;
    double tmy = dy != 0.0 ? ((double)(y + (sy > 0 ? 1 : 0)) - v0.y) / dy : big;
    double tmz = dz != 0.0 ? ((double)(z + (sz > 0 ? 1 : 0)) - v0.z) / dz : big;
    const double tdx = dx != 0.0 ? fabs(1.0 / dx) : big;
    const double tdy = dy != 0.0 ? fabs(1.0 / dy) : big;
    const double tdz = dz != 0.0 ? fabs(1.0 / dz) : big;
    for (int i = 1; i <= steps; i++) {
        if (tmx <= tmy && tmx <= tmz) { x += sx; tmx += tdx; }
        else if (tmy <= tmz) { y += sy; tmy += tdy; }
        else { z += sz; tmz += tdz; }
        emit(x, y, z);
    }
}

template <class F>
__device__ __forceinline__ void for_each_cell(int method, const d3 &a, const d3 &b, double rt, int res, F &&f) {
    if (method == 1) cells_capsule(a, b, rt, res, f);
    else if (method == 0) cells_dda(a, b, res, f);
    else cells_aabb(a, b, rt, res, f);
}

// f(x, y, z, axis, len); the dda method yields rows of one cell
template <class F>
__device__ __forceinline__ void for_each_row(int method, const d3 &a, const d3 &b, double rt, int res, F &&f) {
    if (method == 1) rows_capsule(a, b, rt, res, f);
    else if (method == 0) cells_dda(a, b, res, [&](int x, int y, int z) { f(x, y, z, 0, 1); });
    else rows_aabb(a, b, rt, res, f);
}

// ----------------------------------------------------------------------------- capsule
struct Capsule {
    d3 a, b, n0, n1;
    double r;
    bool clip;
};

// lv/voxelizer.py:254-283 _sdf
__device__ __forceinline__ double capsule_sdf(double px, double py, double pz, const Capsule &c, double r) {
    const double dx = c.b.x - c.a.x, dy = c.b.y - c.a.y, dz = c.b.z - c.a.z;
    const double p0x = px - c.a.x, p0y = py - c.a.y, p0z = pz - c.a.z;
    const double dd = dx * dx + dy * dy + dz * dz;
    double h = 0.0;
    if (dd > 0.0) {
        h = (p0x * dx + p0y * dy + p0z * dz) / dd;
        if (h < 0.0) h = 0.0; else if (h > 1.0) h = 1.0;
    }
    const double qx = p0x - dx * h, qy = p0y - dy * h, qz = p0z - dz * h;
    double sdf = sqrt(qx * qx + qy * qy + qz * qz) - r;
    if (c.clip) {
        const double s0 = -(p0x * c.n0.x + p0y * c.n0.y + p0z * c.n0.z);
        const double s1 = (px - c.b.x) * c.n1.x + (py - c.b.y) * c.n1.y + (pz - c.b.z) * c.n1.z;
        if (s0 > sdf) sdf = s0;
        if (s1 > sdf) sdf = s1;
    }
    return sdf;
}

// Single-precision view of one segment in a frame whose origin is an integer voxel near its start,
// for CONSERVATIVE pre-tests only: cell centres are exact in it (small integers + 0.5) and the end
// points are rounded at magnitudes of a few voxels (~1e-6 absolute), far below the margins the
// callers use.  Exact results never depend on it.
struct SegF {
    int ox, oy, oz;
    float ax, ay, az, ex, ey, ez, inv_ee;
};
__device__ __forceinline__ SegF make_segf(const d3 &a, const d3 &b) {
    SegF s;
    s.ox = (int)floor(a.x); s.oy = (int)floor(a.y); s.oz = (int)floor(a.z);
    s.ax = (float)(a.x - s.ox); s.ay = (float)(a.y - s.oy); s.az = (float)(a.z - s.oz);
    s.ex = (float)(b.x - a.x); s.ey = (float)(b.y - a.y); s.ez = (float)(b.z - a.z);
    const float ee = fmaf(s.ex, s.ex, fmaf(s.ey, s.ey, s.ez * s.ez));
    s.inv_ee = ee > 0.f ? __fdividef(1.f, ee) : 0.f;
    return s;
}
// squared distance from the point (px, py, pz) (same frame) to the segment, accurate to ~1e-5 relative
__device__ __forceinline__ float segf_dist2(const SegF &s, float px, float py, float pz) {
    const float wx = px - s.ax, wy = py - s.ay, wz = pz - s.az;
    const float h = fminf(fmaxf(fmaf(wx, s.ex, fmaf(wy, s.ey, wz * s.ez)) * s.inv_ee, 0.f), 1.f);
    const float qx = fmaf(-h, s.ex, wx), qy = fmaf(-h, s.ey, wy), qz = fmaf(-h, s.ez, wz);
    return fmaf(qx, qx, fmaf(qy, qy, qz * qz));
}

// lv/voxelizer.py:286-298 _occupancy followed by q = int(round(occ * 4096)) (328)
__device__ __forceinline__ uint32_t occupancy_q(double px, double py, double pz, const Capsule &c,
                                                double rc, double corr) {
    const double sdf = capsule_sdf(px, py, pz, c, rc);
    double occ = 0.5 - sdf;
    if (occ < 0.0) occ = 0.0; else if (occ > 1.0) occ = 1.0;
    return (uint32_t)(int)rint(occ * corr * 4096.0);   // rint = round-half-even, like python round()
}

__device__ __forceinline__ Capsule load_capsule(const double *__restrict__ verts, const double *__restrict__ normals,
                                                int64_t i, double r, bool clip) {
    Capsule c;
    c.a = ld3(verts + 3 * i);
    c.b = ld3(verts + 3 * i + 3);
    if (clip) { c.n0 = ld3(normals + 3 * i); c.n1 = ld3(normals + 3 * i + 3); }
    else { c.n0 = d3{0, 0, 0}; c.n1 = d3{0, 0, 0}; }
    c.r = r;
    c.clip = clip;
    return c;
}

// pyramid level offsets (elements), level 0 first
struct LevelOffsets {
    int64_t off[16];
    int n_levels;
};
static inline LevelOffsets make_level_offsets(int res) {
    LevelOffsets L;
    int n = 0;
    int64_t o = 0;
    for (int r = res; r >= 1; r >>= 1) { L.off[n++] = o; o += (int64_t)r * r * r; }
    L.off[n] = o;
    L.n_levels = n;
    return L;
}

// List buffers: word 0..1 hold the entry count (u64), entries start at word LVX_LIST_HDR.
#define LVX_LIST_HDR 16

__device__ __forceinline__ void list_append_warp(uint32_t *list, bool pred, uint32_t value) {
    const uint32_t m = __ballot_sync(0xffffffffu, pred);
    if (!m) return;
    const int lane = threadIdx.x & 31;
    unsigned long long b = 0;
    if (lane == __ffs(m) - 1) b = atomicAdd(reinterpret_cast<unsigned long long *>(list), (unsigned long long)__popc(m));
    b = __shfl_sync(0xffffffffu, b, __ffs(m) - 1);
    if (pred) list[LVX_LIST_HDR + b + __popc(m & ((1u << lane) - 1u))] = value;
}

// Block-wide version for kernels that append from every thread (called by ALL threads of the
// block, blockDim.x <= 1024): one global atomic per block instead of one per warp -- the list
// counter is a single address, and half a million same-address atomics per pass were the cost of
// the per-voxel culling passes.  `counter2` (optional) receives the same count (a stats word).
__device__ __forceinline__ void list_append_block(uint32_t *list, bool pred, uint32_t value,
                                                  unsigned long long *counter2 = nullptr) {
    __shared__ uint32_t s_cnt[32];
    __shared__ unsigned long long s_base;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, n_warps = (blockDim.x + 31) >> 5;
    const uint32_t m = __ballot_sync(0xffffffffu, pred);
    if (lane == 0) s_cnt[warp] = __popc(m);
    __syncthreads();
    if (warp == 0) {
        const uint32_t c = lane < n_warps ? s_cnt[lane] : 0;
        uint32_t inc = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += v;
        }
        if (lane < n_warps) s_cnt[lane] = inc - c;            // exclusive prefix per warp
        if (lane == 31 && inc) {
            s_base = atomicAdd(reinterpret_cast<unsigned long long *>(list), (unsigned long long)inc);
            if (counter2) atomicAdd(counter2, (unsigned long long)inc);
        }
    }
    __syncthreads();
    if (pred) list[LVX_LIST_HDR + s_base + s_cnt[warp] + __popc(m & ((1u << lane) - 1u))] = value;
    __syncthreads();          // s_cnt / s_base may be reused by the next call
}

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
}

}  // namespace lvx
