// render.cu -- image-order voxel ray tracing: grid clip, hierarchical empty-space skip, face-to-face
// DDA, analytic clipped ray-capsule intersection, opaque first hit or exact ordered k-buffer
// transparency, AO/shadow lookup.  Replaces lv/raytracer.py:113-256 (_ray_capsule,
// _capsule_normal), 272-347 (marching helpers), 368-423 (_tri3d, _shade, _pixel_ray), 430-515
// (_voxel_best_hit, _opaque_kernel), 518-645 (_transparent_kernel) and 94-97 (_to_srgb).
#include "lvx_device.cuh"

namespace lvx {

struct RenderArgs {
    const double *verts, *normals;
    const float *verts_f;      // voxel-unit vertices rounded to f32 (conservative pre-test only)
    const uint32_t *offsets, *frags;
    const uint8_t *bits;
    const float *ao, *sh;
    uint32_t bits_off[16];
    int res, n_levels;
    lvx_camera cam;
    lvx_render_params p;
    double *rgb;
    uint8_t *srgb;
    int32_t *hit_id;
    uint64_t *stats;
    // shading on demand (lvx_trace_hits / lvx_resolve)
    double *hit_t;           // per pixel: t of the first hit, < 0 = miss
    uint32_t *need_bits;     // V/32 words: voxels whose AO/shadow some hit pixel interpolates
    uint32_t *need_list;     // compacted list of those voxels (list layout of lvx_device.cuh)
    int guard_volumes;       // ao/sh hold values only where requested: read 1.0 where bits[] == 0
};

__device__ __forceinline__ bool clip_ok(const Capsule &c, double px, double py, double pz) {
    if (!c.clip) return true;
    if ((px - c.a.x) * c.n0.x + (py - c.a.y) * c.n0.y + (pz - c.a.z) * c.n0.z < -1e-9) return false;
    if ((px - c.b.x) * c.n1.x + (py - c.b.y) * c.n1.y + (pz - c.b.z) * c.n1.z > 1e-9) return false;
    return true;
}

// Conservative miss test: every surface _ray_capsule can return a point on (cylinder body, end
// spheres, clip disks incl. their 1e-9 slacks) lies within r + ~1e-9/r of the segment's axis
// LINE, so a ray whose line-to-line distance from the axis exceeds r + 1e-4 cannot hit and the
// full f64 routine would return -1.  ~25 flops, no division or square root; it removes most of
// the tests (lists hold every segment within the 1-voxel traversal footprint, the capsule
// itself is much thinner).  Near-parallel and degenerate cases are never rejected here.
__device__ __forceinline__ bool surely_misses(double ox, double oy, double oz, double dx, double dy, double dz,
                                              const d3 &a, const d3 &b, double r) {
    const double bax = b.x - a.x, bay = b.y - a.y, baz = b.z - a.z;
    const double baba = bax * bax + bay * bay + baz * baz;
    const double nx = dy * baz - dz * bay, ny = dz * bax - dx * baz, nz = dx * bay - dy * bax;
    const double nn = nx * nx + ny * ny + nz * nz;
    if (!(baba > 1e-12) || !(nn > 1e-6 * baba)) return false;
    const double h = (ox - a.x) * nx + (oy - a.y) * ny + (oz - a.z) * nz;
    const double R = r + 1e-4;
    return h * h > R * R * nn;
}

// Single-precision version used by the cooperative kernels.  It bounds the distance between the
// ray LINE through P (a point of the ray inside the current voxel, so all differences are a few
// voxels long) and the SEGMENT [a, b]: every surface the f64 routine can return lies within
// r + 3.2e-5 of the segment, the f32 evaluation (inputs rounded to f32 at magnitudes <= 1024,
// i.e. <= 6.1e-5 absolute) is accurate to a few 1e-4, so "distance > r + 2e-3" proves a miss.
// ~40 full-rate FMA-able operations instead of ~60 half-rate f64 ones, and it also rejects rays that
// pass the infinite cylinder beyond the segment's ends.
__device__ __forceinline__ bool surely_misses_f32(float Px, float Py, float Pz, float Dx, float Dy, float Dz,
                                                  const float *__restrict__ vf, int64_t i, float R2) {
    const float ax = vf[3 * i], ay = vf[3 * i + 1], az = vf[3 * i + 2];
    const float bx = vf[3 * i + 3], by = vf[3 * i + 4], bz = vf[3 * i + 5];
    const float wx = ax - Px, wy = ay - Py, wz = az - Pz;
    const float ex = bx - ax, ey = by - ay, ez = bz - az;
    // (explicit fmaf: the translation unit is compiled with -fmad=false for the f64 code)
    const float dw = fmaf(Dx, wx, fmaf(Dy, wy, Dz * wz)), de = fmaf(Dx, ex, fmaf(Dy, ey, Dz * ez));
    const float wpx = fmaf(-Dx, dw, wx), wpy = fmaf(-Dy, dw, wy), wpz = fmaf(-Dz, dw, wz);   // w, e perpendicular to D
    const float epx = fmaf(-Dx, de, ex), epy = fmaf(-Dy, de, ey), epz = fmaf(-Dz, de, ez);
    const float ee = fmaf(epx, epx, fmaf(epy, epy, epz * epz));
    float sgm = 0.f;
    if (ee > 1e-12f) sgm = fminf(fmaxf(__fdividef(-fmaf(wpx, epx, fmaf(wpy, epy, wpz * epz)), ee), 0.f), 1.f);
    const float qx = fmaf(sgm, epx, wpx), qy = fmaf(sgm, epy, wpy), qz = fmaf(sgm, epz, wpz);
    return fmaf(qx, qx, fmaf(qy, qy, qz * qz)) > R2;
}

__device__ __forceinline__ Capsule load_capsule_lazy(const double *__restrict__ normals, int64_t i, const d3 &a,
                                                     const d3 &b, double r, bool clip) {
    Capsule c;
    c.a = a; c.b = b; c.r = r; c.clip = clip;
    if (clip) { c.n0 = ld3(normals + 3 * i); c.n1 = ld3(normals + 3 * i + 3); }
    else { c.n0 = d3{0, 0, 0}; c.n1 = d3{0, 0, 0}; }
    return c;
}

// lv/raytracer.py:113-222: smallest t >= 0 on the clipped capsule surface, or -1
__device__ double ray_capsule(double ox, double oy, double oz, double dx, double dy, double dz, const Capsule &c) {
    const double ax = c.a.x, ay = c.a.y, az = c.a.z, bx = c.b.x, by = c.b.y, bz = c.b.z, r = c.r;
    const double bax = bx - ax, bay = by - ay, baz = bz - az;
    const double oax = ox - ax, oay = oy - ay, oaz = oz - az;
    const double baba = bax * bax + bay * bay + baz * baz;
    const double eps = 1e-12;
    double best = -1.0;
    if (baba > eps) {
        const double bard = bax * dx + bay * dy + baz * dz;
        const double baoa = bax * oax + bay * oay + baz * oaz;
        const double rdoa = dx * oax + dy * oay + dz * oaz;
        const double oaoa = oax * oax + oay * oay + oaz * oaz;
        const double a_ = baba - bard * bard;
        const double b_ = baba * rdoa - baoa * bard;
        const double c_ = baba * oaoa - baoa * baoa - r * r * baba;
        if (fabs(a_) > eps) {
            const double disc = b_ * b_ - a_ * c_;
            if (disc >= 0.0) {
                const double sq = sqrt(disc);
#pragma unroll
                for (int k = 0; k < 2; k++) {
                    const double t = (-b_ + (k ? sq : -sq)) / a_;
                    if (t >= 0.0) {
                        const double y = baoa + t * bard;
                        if (-1e-9 <= y && y <= baba + 1e-9) {
                            const double px = ox + dx * t, py = oy + dy * t, pz = oz + dz * t;
                            if (clip_ok(c, px, py, pz) && (best < 0.0 || t < best)) best = t;
                        }
                    }
                }
            }
        }
    }
#pragma unroll
    for (int cap = 0; cap < 2; cap++) {
        const double cx = cap ? bx : ax, cy = cap ? by : ay, cz = cap ? bz : az;
        const double ocx = ox - cx, ocy = oy - cy, ocz = oz - cz;
        const double bq = ocx * dx + ocy * dy + ocz * dz;
        const double cq = ocx * ocx + ocy * ocy + ocz * ocz - r * r;
        const double disc = bq * bq - cq;
        if (disc < 0.0) continue;
        const double sq = sqrt(disc);
#pragma unroll
        for (int k = 0; k < 2; k++) {
            const double t = -bq + (k ? sq : -sq);
            if (t < 0.0) continue;
            const double px = ox + dx * t, py = oy + dy * t, pz = oz + dz * t;
            const double y = (px - ax) * bax + (py - ay) * bay + (pz - az) * baz;
            bool on_cap = cap == 0 ? (y <= 1e-9) : (y >= baba - 1e-9);
            if (baba <= eps) on_cap = cap == 0;
            if (on_cap && clip_ok(c, px, py, pz) && (best < 0.0 || t < best)) best = t;
        }
    }
    if (c.clip) {
#pragma unroll
        for (int pl = 0; pl < 2; pl++) {
            const double nx = pl ? c.n1.x : c.n0.x, ny = pl ? c.n1.y : c.n0.y, nz = pl ? c.n1.z : c.n0.z;
            const double qx = pl ? bx : ax, qy = pl ? by : ay, qz = pl ? bz : az;
            const double dn = dx * nx + dy * ny + dz * nz;
            if (fabs(dn) < eps) continue;
            const double t = ((qx - ox) * nx + (qy - oy) * ny + (qz - oz) * nz) / dn;
            if (t < 0.0) continue;
            const double px = ox + dx * t, py = oy + dy * t, pz = oz + dz * t;
            double h = 0.0;
            if (baba > eps) h = ((px - ax) * bax + (py - ay) * bay + (pz - az) * baz) / baba;
            if (h < 0.0) h = 0.0; else if (h > 1.0) h = 1.0;
            const double wx = px - (ax + bax * h), wy = py - (ay + bay * h), wz = pz - (az + baz * h);
            if (wx * wx + wy * wy + wz * wz > r * r + 1e-9) continue;
            if (clip_ok(c, px, py, pz) && (best < 0.0 || t < best)) best = t;
        }
    }
    return best;
}

// lv/raytracer.py:225-256
__device__ void capsule_normal(double px, double py, double pz, const Capsule &c, double &ox, double &oy, double &oz) {
    const double bax = c.b.x - c.a.x, bay = c.b.y - c.a.y, baz = c.b.z - c.a.z;
    const double baba = bax * bax + bay * bay + baz * baz;
    double h = 0.0;
    if (baba > 1e-12) {
        h = ((px - c.a.x) * bax + (py - c.a.y) * bay + (pz - c.a.z) * baz) / baba;
        if (h < 0.0) h = 0.0; else if (h > 1.0) h = 1.0;
    }
    const double wx = px - (c.a.x + bax * h), wy = py - (c.a.y + bay * h), wz = pz - (c.a.z + baz * h);
    const double s_cap = sqrt(wx * wx + wy * wy + wz * wz) - c.r;
    double nx = wx, ny = wy, nz = wz;
    if (c.clip) {
        const double s0 = -((px - c.a.x) * c.n0.x + (py - c.a.y) * c.n0.y + (pz - c.a.z) * c.n0.z);
        const double s1 = (px - c.b.x) * c.n1.x + (py - c.b.y) * c.n1.y + (pz - c.b.z) * c.n1.z;
        if (s0 >= s_cap && s0 >= s1) { nx = -c.n0.x; ny = -c.n0.y; nz = -c.n0.z; }
        else if (s1 >= s_cap) { nx = c.n1.x; ny = c.n1.y; nz = c.n1.z; }
    }
    const double nn = sqrt(nx * nx + ny * ny + nz * nz);
    if (nn == 0.0) { ox = 0.0; oy = 0.0; oz = 1.0; return; }
    ox = nx / nn; oy = ny / nn; oz = nz / nn;
}

// lv/raytracer.py:294-313.  The reference takes the minimum of up to three quotients.  Here the
// quotients are first estimated with precomputed reciprocals (error < 3e-16 relative); only axes
// whose estimate is within 1e-13 of the smallest can own the exact minimum, so the exact IEEE
// division is evaluated for those (almost always one) and the result is bit-identical.
struct RayInv { double ix, iy, iz; };
__device__ __forceinline__ RayInv make_inv(double dx, double dy, double dz) {
    return RayInv{dx != 0.0 ? 1.0 / dx : 0.0, dy != 0.0 ? 1.0 / dy : 0.0, dz != 0.0 ? 1.0 / dz : 0.0};
}
__device__ __forceinline__ double voxel_exit(double ox, double oy, double oz, double dx, double dy, double dz,
                                             const RayInv &inv, int x, int y, int z, int lvl) {
    const int size = 1 << lvl;
    const int bx = (x >> lvl) << lvl, by = (y >> lvl) << lvl, bz = (z >> lvl) << lvl;
    const double big = 1e30;
    const double nx = (double)(dx > 0.0 ? bx + size : bx) - ox;
    const double ny = (double)(dy > 0.0 ? by + size : by) - oy;
    const double nz = (double)(dz > 0.0 ? bz + size : bz) - oz;
    const double ax = dx != 0.0 ? nx * inv.ix : big;
    const double ay = dy != 0.0 ? ny * inv.iy : big;
    const double az = dz != 0.0 ? nz * inv.iz : big;
    const double m = fmin(ax, fmin(ay, az));
    const double lim = m + fabs(m) * 1e-13 + 1e-290;
    double t = big;
    if (ax <= lim) t = fmin(t, nx / dx);
    if (ay <= lim) t = fmin(t, ny / dy);
    if (az <= lim) t = fmin(t, nz / dz);
    return t;
}

// lv/raytracer.py:316-326: largest level whose node containing (x,y,z) is clear.  A parent is the OR
// of its children, so "clear" is monotone in the level and the answer can be found from any
// starting level (`hint`, normally the previous step's answer) instead of always climbing from 1.
__device__ __forceinline__ bool node_clear(const RenderArgs &A, int l, int x, int y, int z) {
    const uint32_t rl = (uint32_t)A.res >> l;
    return A.bits[A.bits_off[l] + ((uint32_t)x >> l) + rl * (((uint32_t)y >> l) + rl * ((uint32_t)z >> l))] == 0;
}
__device__ __forceinline__ int empty_level(const RenderArgs &A, int x, int y, int z, int hint) {
    const int top = A.n_levels - 1;
    int l = hint < 1 ? 1 : (hint > top ? top : hint);
    if (top < 1) return 0;
    if (node_clear(A, l, x, y, z)) {
        while (l < top && node_clear(A, l + 1, x, y, z)) l++;
        return l;
    }
    do { l--; } while (l >= 1 && !node_clear(A, l, x, y, z));
    return l;
}

// lv/raytracer.py:368-390 (volumes are f32, widened exactly like the reference's astype(f64))
__device__ __forceinline__ double tri3d(const float *__restrict__ vol, const uint8_t *__restrict__ guard, int res,
                                        double px, double py, double pz) {
    const double ux = px - 0.5, uy = py - 0.5, uz = pz - 0.5;
    const int ix = (int)floor(ux), iy = (int)floor(uy), iz = (int)floor(uz);
    const double fx = ux - ix, fy = uy - iy, fz = uz - iz;
    double acc = 0.0;
#pragma unroll
    for (int dz = 0; dz < 2; dz++) {
        const int z = min(max(iz + dz, 0), res - 1);
        const double wz = dz ? fz : 1.0 - fz;
#pragma unroll
        for (int dy = 0; dy < 2; dy++) {
            const int y = min(max(iy + dy, 0), res - 1);
            const double wy = dy ? fy : 1.0 - fy;
#pragma unroll
            for (int dx = 0; dx < 2; dx++) {
                const int x = min(max(ix + dx, 0), res - 1);
                const double wx = dx ? fx : 1.0 - fx;
                const int64_t idx = x + (int64_t)res * (y + (int64_t)res * z);
                // non-visible voxels keep ao = shadow = 1 (lv/shading.py:177-178)
                const double val = (guard && guard[idx] == 0) ? 1.0 : (double)vol[idx];
                acc += wx * wy * wz * val;
            }
        }
    }
    return acc;
}

// lv/raytracer.py:393-411
__device__ __forceinline__ void shade(const RenderArgs &A, const Capsule &c, double nx, double ny, double nz,
                                      double px, double py, double pz, double &cr, double &cg, double &cb) {
    const double sx = c.b.x - c.a.x, sy = c.b.y - c.a.y, sz = c.b.z - c.a.z;
    const double sn = sqrt(sx * sx + sy * sy + sz * sz);
    if (sn == 0.0) { cr = cg = cb = 0.5; }
    else { cr = fabs(sx) / sn; cg = fabs(sy) / sn; cb = fabs(sz) / sn; }
    const uint8_t *guard = A.guard_volumes ? A.bits : nullptr;
    const double ao = A.ao ? tri3d(A.ao, guard, A.res, px, py, pz) : 1.0;
    const double sh = A.sh ? tri3d(A.sh, guard, A.res, px, py, pz) : 1.0;
    double ndl = nx * A.p.light_to_source[0] + ny * A.p.light_to_source[1] + nz * A.p.light_to_source[2];
    if (ndl < 0.0) ndl = 0.0;
    const double k = 0.4 * ao + 0.6 * sh * ndl;
    cr = cr * k; cg = cg * k; cb = cb * k;
}

__device__ __forceinline__ uint8_t to_srgb8(double v) {   // lv/raytracer.py:94-97
    const double c = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
    const double s = c <= 0.0031308 ? 12.92 * c : 1.055 * pow(c, 1.0 / 2.4) - 0.055;
    return (uint8_t)(int)rint(s * 255.0);
}

template <int MODE>
__global__ void __launch_bounds__(128)
k_render(const RenderArgs A) {
    const int px = A.p.tile_x0 + blockIdx.x * 8 + (threadIdx.x & 7);
    const int py = A.p.tile_y0 + blockIdx.y * 16 + (threadIdx.x >> 3);
    const bool live = px < A.p.tile_x1 && py < A.p.tile_y1;
    uint32_t n_tests = 0;
    if (live) {
        const int w = A.cam.width, h = A.cam.height, res = A.res;
        // lv/raytracer.py:414-423
        const double aspect = (double)w / (double)h;
        const double u = (2.0 * (px + 0.5) / w - 1.0) * aspect * A.cam.tan_half_fov;
        const double v = (1.0 - 2.0 * (py + 0.5) / h) * A.cam.tan_half_fov;
        double dx = A.cam.fwd[0] + u * A.cam.right[0] + v * A.cam.up[0];
        double dy = A.cam.fwd[1] + u * A.cam.right[1] + v * A.cam.up[1];
        double dz = A.cam.fwd[2] + u * A.cam.right[2] + v * A.cam.up[2];
        const double dn = sqrt(dx * dx + dy * dy + dz * dz);
        dx = dx / dn; dy = dy / dn; dz = dz / dn;
        const double ox = A.cam.pos[0], oy = A.cam.pos[1], oz = A.cam.pos[2];
        // lv/raytracer.py:272-291
        double t0 = 0.0, t1 = 1e30;
        {
            const double o[3] = {ox, oy, oz}, d[3] = {dx, dy, dz};
#pragma unroll
            for (int a = 0; a < 3; a++) {
                if (d[a] == 0.0) {
                    if (o[a] < 0.0 || o[a] > (double)res) { t0 = 1.0; t1 = -1.0; break; }
                } else {
                    double ta = (0.0 - o[a]) / d[a], tb = ((double)res - o[a]) / d[a];
                    if (ta > tb) { const double tmp = ta; ta = tb; tb = tmp; }
                    if (ta > t0) t0 = ta;
                    if (tb < t1) t1 = tb;
                }
            }
        }
        const bool clip = A.p.use_clip != 0;
        const double r = A.p.radius;
        const RayInv inv = make_inv(dx, dy, dz);
        int lvl_hint = 1;
        double out_r, out_g, out_b;
        int32_t out_id;
        if (MODE == 0) {
            out_r = A.p.background[0]; out_g = A.p.background[1]; out_b = A.p.background[2];
            out_id = -1;
            if (t1 >= t0) {
                double t = t0 > 0.0 ? t0 : 0.0;
                while (t < t1) {
                    const double tm = t + 1e-6;
                    const int x = (int)floor(ox + dx * tm), y = (int)floor(oy + dy * tm), z = (int)floor(oz + dz * tm);
                    if (x < 0 || y < 0 || z < 0 || x >= res || y >= res || z >= res) break;
                    const int64_t idx = x + (int64_t)res * (y + (int64_t)res * z);
                    double te;
                    if (A.bits[idx] != 0) {
                        // lv/raytracer.py:430-456
                        double best = -1.0;
                        int64_t best_i = -1;
                        const uint32_t fo = A.offsets[idx], fe = A.offsets[idx + 1];
                        for (uint32_t s = fo; s < fe; s++) {
                            const int64_t i = A.frags[s];
                            n_tests++;
                            const d3 va = ld3(A.verts + 3 * i), vb = ld3(A.verts + 3 * i + 3);
                            if (surely_misses(ox, oy, oz, dx, dy, dz, va, vb, r)) continue;
                            const Capsule c = load_capsule_lazy(A.normals, i, va, vb, r, clip);
                            const double tt = ray_capsule(ox, oy, oz, dx, dy, dz, c);
                            if (tt < 0.0) continue;
                            const int hx = (int)floor(ox + dx * tt), hy = (int)floor(oy + dy * tt), hz = (int)floor(oz + dz * tt);
                            if (hx != x || hy != y || hz != z) continue;   // belongs to another voxel's list
                            if (best < 0.0 || tt < best) { best = tt; best_i = i; }
                        }
                        if (best >= 0.0) {
                            const double hx = ox + dx * best, hy = oy + dy * best, hz = oz + dz * best;
                            const Capsule c = load_capsule(A.verts, A.normals, best_i, r, clip);
                            double nx, ny, nz;
                            capsule_normal(hx, hy, hz, c, nx, ny, nz);
                            shade(A, c, nx, ny, nz, hx, hy, hz, out_r, out_g, out_b);
                            out_id = (int32_t)best_i;
                            break;
                        }
                        te = voxel_exit(ox, oy, oz, dx, dy, dz, inv, x, y, z, 0);
                    } else {
                        const int l = lvl_hint = empty_level(A, x, y, z, lvl_hint);
                        te = voxel_exit(ox, oy, oz, dx, dy, dz, inv, x, y, z, l);
                    }
                    t = te > t ? te : t + 1e-6;
                }
            }
        } else {
            double col_r = 0.0, col_g = 0.0, col_b = 0.0, acc_a = 0.0;
            int64_t first_hit = -1;
            int64_t keybuf[64];
            double tbuf[64];
            int32_t ibuf[64];
            const int kslots = A.p.k;
            const bool early = A.p.early_termination != 0;
            const double alpha = A.p.alpha;
            if (t1 >= t0) {
                double t = t0 > 0.0 ? t0 : 0.0;
                while (t < t1) {
                    if (early && acc_a >= 0.999) break;
                    const double tm = t + 1e-6;
                    const int x = (int)floor(ox + dx * tm), y = (int)floor(oy + dy * tm), z = (int)floor(oz + dz * tm);
                    if (x < 0 || y < 0 || z < 0 || x >= res || y >= res || z >= res) break;
                    const int64_t idx = x + (int64_t)res * (y + (int64_t)res * z);
                    if (A.bits[idx] == 0) {
                        const int l = lvl_hint = empty_level(A, x, y, z, lvl_hint);
                        const double te = voxel_exit(ox, oy, oz, dx, dy, dz, inv, x, y, z, l);
                        t = te > t ? te : t + 1e-6;
                        continue;
                    }
                    const double te = voxel_exit(ox, oy, oz, dx, dy, dz, inv, x, y, z, 0);
                    const double t_enter = t, span = te - t_enter;
                    const double inv_span = span > 0.0 ? 65535.0 / span : 0.0;
                    const uint32_t fo = A.offsets[idx], fn = A.offsets[idx + 1] - fo;
                    int64_t last_key = -1;
                    for (;;) {
                        int kept = 0;
                        uint32_t accepted = 0;
                        for (uint32_t s = 0; s < fn; s++) {
                            const int64_t i = A.frags[fo + s];
                            n_tests++;
                            const d3 va = ld3(A.verts + 3 * i), vb = ld3(A.verts + 3 * i + 3);
                            if (surely_misses(ox, oy, oz, dx, dy, dz, va, vb, r)) continue;
                            const Capsule c = load_capsule_lazy(A.normals, i, va, vb, r, clip);
                            const double tt = ray_capsule(ox, oy, oz, dx, dy, dz, c);
                            if (tt < 0.0) continue;
                            const int hx = (int)floor(ox + dx * tt), hy = (int)floor(oy + dy * tt), hz = (int)floor(oz + dz * tt);
                            if (hx != x || hy != y || hz != z) continue;
                            int64_t q = (int64_t)((tt - t_enter) * inv_span);   // int(): truncation
                            if (q < 0) q = 0; else if (q > 65535) q = 65535;
                            const int64_t key = (q << 16) | (int64_t)s;
                            if (key <= last_key) continue;
                            accepted++;
                            int j;
                            if (kept < kslots) { j = kept; kept++; }
                            else if (key < keybuf[kslots - 1]) j = kslots - 1;
                            else continue;
                            while (j > 0 && keybuf[j - 1] > key) {
                                keybuf[j] = keybuf[j - 1]; tbuf[j] = tbuf[j - 1]; ibuf[j] = ibuf[j - 1];
                                j--;
                            }
                            keybuf[j] = key; tbuf[j] = tt; ibuf[j] = (int32_t)i;
                        }
                        for (int j = 0; j < kept; j++) {
                            if (early && acc_a >= 0.999) break;
                            const double tt = tbuf[j];
                            const int64_t i = ibuf[j];
                            const double hx = ox + dx * tt, hy = oy + dy * tt, hz = oz + dz * tt;
                            const Capsule c = load_capsule(A.verts, A.normals, i, r, clip);
                            double nx, ny, nz, cr, cg, cb;
                            capsule_normal(hx, hy, hz, c, nx, ny, nz);
                            shade(A, c, nx, ny, nz, hx, hy, hz, cr, cg, cb);
                            const double wgt = (1.0 - acc_a) * alpha;
                            col_r += wgt * cr; col_g += wgt * cg; col_b += wgt * cb;
                            acc_a += wgt;
                            if (first_hit < 0) first_hit = i;
                        }
                        if (accepted <= (uint32_t)kslots) break;
                        if (early && acc_a >= 0.999) break;
                        last_key = keybuf[kslots - 1];
                    }
                    t = te > t ? te : t + 1e-6;
                }
            }
            out_r = col_r + (1.0 - acc_a) * A.p.background[0];
            out_g = col_g + (1.0 - acc_a) * A.p.background[1];
            out_b = col_b + (1.0 - acc_a) * A.p.background[2];
            out_id = (int32_t)first_hit;
        }
        const int64_t pix = (int64_t)py * w + px;
        if (A.rgb) { A.rgb[3 * pix] = out_r; A.rgb[3 * pix + 1] = out_g; A.rgb[3 * pix + 2] = out_b; }
        if (A.srgb) { A.srgb[3 * pix] = to_srgb8(out_r); A.srgb[3 * pix + 1] = to_srgb8(out_g); A.srgb[3 * pix + 2] = to_srgb8(out_b); }
        A.hit_id[pix] = out_id;
    }
    uint64_t tests = warp_sum_u64(n_tests);
    if ((threadIdx.x & 31) == 0 && tests)
        atomicAdd((unsigned long long *)&A.stats[LVX_ST_RAY_TESTS], (unsigned long long)tests);
}

// ----------------------------------------------------------------------------- opaque, warp-cooperative
// The per-pixel loop above spends most of its instructions in the heavy f64 intersection with 2-3
// of 32 lanes active (ncu: profiles/r01c).  This kernel keeps the reference's per-ray semantics
// (lv/raytracer.py:459-515) but shares the work of a warp's 8x4 pixel tile:
//   1. every unfinished ray marches (hierarchical skip) to its next occupied voxel;
//   2. the (ray, fragment) pairs of all 32 rays are flattened with a warp prefix sum and dealt
//      round-robin to the lanes -> the cheap conservative reject runs fully converged, fragment
//      ids are read coalesced;
//   3. pairs that survive the reject are compacted into a shared-memory queue; whenever 32 are
//      queued the full clipped ray-capsule routine runs on all 32 lanes at once;
//   4. hits are folded on the owning lane by (t, slot) -- "min t, first slot wins ties" (453) --
//      and rays without a hit step to the voxel exit.
// Shading runs once, after the loop, for all hit rays together.
constexpr int RC_WARPS = 4;

struct WarpShared {
    double dir[3][32];
    float dirf[3][32], pf[3][32];   // f32 direction and a ray point inside the current voxel
    int vox[3][32];
    uint32_t fo[32];
    uint32_t prefix[33];
    uint32_t q_i[64];
    uint32_t q_rs[64];
    double hit_t[32];
    uint32_t hit_s[32], hit_i[32];
};

#ifndef LVX_RC_MINB
#define LVX_RC_MINB 6
#endif
template <bool DEFER>
__global__ void __launch_bounds__(RC_WARPS * 32, LVX_RC_MINB)
k_render_opaque_coop(const RenderArgs A) {
    __shared__ WarpShared sh_all[RC_WARPS];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    WarpShared &S = sh_all[warp];
    // block = 4 warps side by side: 32 x 4 pixels, each warp an 8x4 tile
    const int px = A.p.tile_x0 + blockIdx.x * (8 * RC_WARPS) + warp * 8 + (lane & 7);
    const int py = A.p.tile_y0 + blockIdx.y * 4 + (lane >> 3);
    const bool live = px < A.p.tile_x1 && py < A.p.tile_y1;
    const int w = A.cam.width, h = A.cam.height, res = A.res;
    const double ox = A.cam.pos[0], oy = A.cam.pos[1], oz = A.cam.pos[2];
    const bool clip = A.p.use_clip != 0;
    const double r = A.p.radius;
    double dx = 0.0, dy = 0.0, dz = 1.0, t = 0.0, t1 = -1.0;
    bool active = false;
    if (live) {
        // lv/raytracer.py:414-423
        const double aspect = (double)w / (double)h;
        const double u = (2.0 * (px + 0.5) / w - 1.0) * aspect * A.cam.tan_half_fov;
        const double v = (1.0 - 2.0 * (py + 0.5) / h) * A.cam.tan_half_fov;
        dx = A.cam.fwd[0] + u * A.cam.right[0] + v * A.cam.up[0];
        dy = A.cam.fwd[1] + u * A.cam.right[1] + v * A.cam.up[1];
        dz = A.cam.fwd[2] + u * A.cam.right[2] + v * A.cam.up[2];
        const double dn = sqrt(dx * dx + dy * dy + dz * dz);
        dx = dx / dn; dy = dy / dn; dz = dz / dn;
        // lv/raytracer.py:272-291
        double t0 = 0.0;
        t1 = 1e30;
        const double o[3] = {ox, oy, oz}, d[3] = {dx, dy, dz};
#pragma unroll
        for (int a = 0; a < 3; a++) {
            if (d[a] == 0.0) {
                if (o[a] < 0.0 || o[a] > (double)res) { t0 = 1.0; t1 = -1.0; break; }
            } else {
                double ta = (0.0 - o[a]) / d[a], tb = ((double)res - o[a]) / d[a];
                if (ta > tb) { const double tmp = ta; ta = tb; tb = tmp; }
                if (ta > t0) t0 = ta;
                if (tb < t1) t1 = tb;
            }
        }
        active = t1 >= t0;
        t = t0 > 0.0 ? t0 : 0.0;
    }
    S.dir[0][lane] = dx; S.dir[1][lane] = dy; S.dir[2][lane] = dz;
    S.dirf[0][lane] = (float)dx; S.dirf[1][lane] = (float)dy; S.dirf[2][lane] = (float)dz;
    const float R2f = ((float)r + 2e-3f) * ((float)r + 2e-3f);
    const RayInv inv = make_inv(dx, dy, dz);
    int lvl_hint = 1;
    double best_t = -1.0;      // final hit of this lane's ray
    int64_t best_i = -1;
    uint64_t n_tests = 0;
    __syncwarp();

    for (;;) {
        // ---- 1. march to the next occupied voxel (lv/raytracer.py:475-482, 506-509)
        uint32_t n = 0;
        double te = 0.0;
        int x = 0, y = 0, z = 0;
        if (active) {
            for (;;) {
                if (!(t < t1)) { active = false; break; }
                const double tm = t + 1e-6;
                x = (int)floor(ox + dx * tm); y = (int)floor(oy + dy * tm); z = (int)floor(oz + dz * tm);
                if (x < 0 || y < 0 || z < 0 || x >= res || y >= res || z >= res) { active = false; break; }
                const int64_t idx = x + (int64_t)res * (y + (int64_t)res * z);
                if (A.bits[idx] != 0) {
                    const uint32_t fo = A.offsets[idx];
                    n = A.offsets[idx + 1] - fo;
                    S.fo[lane] = fo;
                    te = voxel_exit(ox, oy, oz, dx, dy, dz, inv, x, y, z, 0);
                    break;
                }
                const int l = lvl_hint = empty_level(A, x, y, z, lvl_hint);
                const double tl = voxel_exit(ox, oy, oz, dx, dy, dz, inv, x, y, z, l);
                t = tl > t ? tl : t + 1e-6;
            }
        }
        if (__ballot_sync(0xffffffffu, active) == 0) break;
        S.vox[0][lane] = x; S.vox[1][lane] = y; S.vox[2][lane] = z;
        {   // a point of the ray inside the voxel (its centre-most parameter), for the f32 pre-test
            const double tc = 0.5 * (t + te);
            S.pf[0][lane] = (float)(ox + dx * tc); S.pf[1][lane] = (float)(oy + dy * tc); S.pf[2][lane] = (float)(oz + dz * tc);
        }
        // ---- 2. flatten (ray, fragment) pairs
        uint32_t inc = active ? n : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += v;
        }
        S.prefix[lane + 1] = inc;
        if (lane == 0) S.prefix[0] = 0;
        const uint32_t T = __shfl_sync(0xffffffffu, inc, 31);
        if (lane == 0) n_tests += T;
        double cur_t = -1.0;           // best hit of this lane's ray in this voxel
        uint32_t cur_s = 0xffffffffu, cur_i = 0;
        uint32_t qn = 0, own = 0;
        __syncwarp();
        for (uint32_t p0 = 0; p0 < T || qn > 0; p0 += 32) {
            const uint32_t p = p0 + lane;
            bool pass = false;
            uint32_t rr = 0, ss = 0, ii = 0;
            if (p < T) {
                // owner ray: largest rr with prefix[rr] <= p
                while (S.prefix[own + 1] <= p) own++;       // owner ray: prefix[own] <= p < prefix[own+1]
                rr = own;
                ss = p - S.prefix[rr];
                ii = A.frags[S.fo[rr] + ss];
                pass = !surely_misses_f32(S.pf[0][rr], S.pf[1][rr], S.pf[2][rr], S.dirf[0][rr], S.dirf[1][rr],
                                          S.dirf[2][rr], A.verts_f, (int64_t)ii, R2f);
            }
            // ---- 3. compact survivors into the queue
            const uint32_t m = __ballot_sync(0xffffffffu, pass);
            if (pass) {
                const uint32_t pos = qn + __popc(m & ((1u << lane) - 1u));
                S.q_i[pos] = ii;
                S.q_rs[pos] = (rr << 16) | ss;
            }
            qn += __popc(m);
            __syncwarp();
            const bool flush = p0 + 32 >= T;          // last batch of pairs: drain what is left
            if (qn >= 32 || (flush && qn > 0)) {
                const uint32_t take = qn < 32 ? qn : 32;
                bool hit = false;
                double ht = 0.0;
                uint32_t hr = 0, hs = 0, hi_ = 0;
                if (lane < take) {
                    hi_ = S.q_i[lane];
                    const uint32_t rs = S.q_rs[lane];
                    hr = rs >> 16; hs = rs & 0xFFFFu;
                    const double ddx = S.dir[0][hr], ddy = S.dir[1][hr], ddz = S.dir[2][hr];
                    const Capsule c = load_capsule(A.verts, A.normals, (int64_t)hi_, r, clip);
                    ht = ray_capsule(ox, oy, oz, ddx, ddy, ddz, c);
                    if (ht >= 0.0) {   // lv/raytracer.py:446-452: the hit must lie in the ray's current voxel
                        const int hx = (int)floor(ox + ddx * ht), hy = (int)floor(oy + ddy * ht), hz = (int)floor(oz + ddz * ht);
                        hit = hx == S.vox[0][hr] && hy == S.vox[1][hr] && hz == S.vox[2][hr];
                    }
                }
                __syncwarp();
                // move the queue tail down
                uint32_t mv_i = 0, mv_rs = 0;
                const bool mv = lane + 32 < qn;
                if (mv) { mv_i = S.q_i[lane + 32]; mv_rs = S.q_rs[lane + 32]; }
                __syncwarp();
                if (mv) { S.q_i[lane] = mv_i; S.q_rs[lane] = mv_rs; }
                qn -= take;
                // ---- 4. fold hits on the owning lanes: min t, then lowest slot (lv/raytracer.py:453)
                uint32_t hm = __ballot_sync(0xffffffffu, hit);
                if (hit) { S.hit_t[lane] = ht; S.hit_s[lane] = hs; S.hit_i[lane] = hi_; }
                __syncwarp();
                while (hm) {
                    const int src = __ffs(hm) - 1;
                    hm &= hm - 1;
                    const uint32_t owner = __shfl_sync(0xffffffffu, hr, src);
                    if ((uint32_t)lane == owner) {
                        const double tt = S.hit_t[src];
                        const uint32_t s2 = S.hit_s[src];
                        if (cur_t < 0.0 || tt < cur_t || (tt == cur_t && s2 < cur_s)) {
                            cur_t = tt; cur_s = s2; cur_i = S.hit_i[src];
                        }
                    }
                }
                __syncwarp();
            }
            if (flush && qn == 0) break;
        }
        if (active) {
            if (cur_t >= 0.0) { best_t = cur_t; best_i = cur_i; active = false; }
            else t = te > t ? te : t + 1e-6;
        }
        __syncwarp();
    }

    if (!DEFER) {
        if (live) {
            double out_r = A.p.background[0], out_g = A.p.background[1], out_b = A.p.background[2];
            int32_t out_id = -1;
            if (best_t >= 0.0) {
                const double hx = ox + dx * best_t, hy = oy + dy * best_t, hz = oz + dz * best_t;
                const Capsule c = load_capsule(A.verts, A.normals, best_i, r, clip);
                double nx, ny, nz;
                capsule_normal(hx, hy, hz, c, nx, ny, nz);
                shade(A, c, nx, ny, nz, hx, hy, hz, out_r, out_g, out_b);
                out_id = (int32_t)best_i;
            }
            const int64_t pix = (int64_t)py * w + px;
            if (A.rgb) { A.rgb[3 * pix] = out_r; A.rgb[3 * pix + 1] = out_g; A.rgb[3 * pix + 2] = out_b; }
            if (A.srgb) { A.srgb[3 * pix] = to_srgb8(out_r); A.srgb[3 * pix + 1] = to_srgb8(out_g); A.srgb[3 * pix + 2] = to_srgb8(out_b); }
            A.hit_id[pix] = out_id;
        }
    } else {
        // Shading on demand: record the hit, and request AO/shadow for the (visible) voxels its
        // trilinear lookup will read (lv/raytracer.py:368-390).  New requests are gathered per
        // block in shared memory so the global list counter sees one atomic per block.
        // (warp-level only: a block-wide barrier here would park finished warps until the slowest
        // warp of the block leaves the trace loop)
        uint32_t items[8];
        int n_items = 0;
        if (live) {
            const int64_t pix = (int64_t)py * w + px;
            A.hit_t[pix] = best_t;
            A.hit_id[pix] = best_t >= 0.0 ? (int32_t)best_i : -1;
            if (best_t >= 0.0) {
                const double hx = ox + dx * best_t, hy = oy + dy * best_t, hz = oz + dz * best_t;
                const int ix = (int)floor(hx - 0.5), iy = (int)floor(hy - 0.5), iz = (int)floor(hz - 0.5);
#pragma unroll
                for (int k = 0; k < 8; k++) {
                    const int X = min(max(ix + (k & 1), 0), res - 1);
                    const int Y = min(max(iy + ((k >> 1) & 1), 0), res - 1);
                    const int Z = min(max(iz + (k >> 2), 0), res - 1);
                    const uint32_t idx = (uint32_t)X + (uint32_t)res * ((uint32_t)Y + (uint32_t)res * (uint32_t)Z);
                    bool fresh = false;
                    if (A.bits[idx] != 0) {
                        const uint32_t bit = 1u << (idx & 31);
                        fresh = (atomicOr(&A.need_bits[idx >> 5], bit) & bit) == 0;
                    }
                    items[k] = idx;
                    if (fresh) n_items |= 1 << k;
                }
            }
        }
        // one global atomic per warp: exclusive scan of the per-lane counts
        const uint32_t mine = __popc((uint32_t)n_items);
        uint32_t incl = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
        if (total) {
            unsigned long long b = 0;
            if (lane == 0)
                b = atomicAdd(reinterpret_cast<unsigned long long *>(A.need_list), (unsigned long long)total);
            b = __shfl_sync(0xffffffffu, b, 0);
            uint32_t pos = (uint32_t)b + incl - mine;
#pragma unroll
            for (int k = 0; k < 8; k++)
                if (n_items & (1 << k)) A.need_list[LVX_LIST_HDR + pos++] = items[k];
        }
    }
    if (lane == 0 && n_tests)
        atomicAdd((unsigned long long *)&A.stats[LVX_ST_RAY_TESTS], (unsigned long long)n_tests);
}

// ----------------------------------------------------------------------------- transparent, warp-cooperative
// Same work sharing as the opaque kernel for lv/raytracer.py:518-645.  Per round every active ray
// sits in one occupied voxel; the flattened (ray, fragment) pairs are rejected/intersected by all
// lanes; in-voxel hits become (key = depth16 << 16 | slot, t, segment) records in a per-warp list,
// which the owning lanes drain into their private k-slot buffers.  The k smallest keys above
// `last_key` are a set, so the insertion order does not matter (keys are unique: the slot is in
// the low bits) and the reference's result is reproduced exactly, including the re-scan of a
// voxel when more than k hits were accepted (the ray then stays in the voxel for another round,
// and its tests are counted again like the reference does).
constexpr int HL_CAP = 128;

struct WarpSharedT {
    double dir[3][32];
    float dirf[3][32], pf[3][32];
    double t_enter[32], inv_span[32];
    int vox[3][32];
    uint32_t fo[32];
    uint32_t prefix[33];
    uint32_t q_i[64];
    uint32_t q_rs[64];
    double hl_t[HL_CAP];
    uint32_t hl_key[HL_CAP], hl_i[HL_CAP];
    uint8_t hl_r[HL_CAP];
};

__global__ void __launch_bounds__(RC_WARPS * 32)
k_render_transparent_coop(const RenderArgs A) {
    __shared__ WarpSharedT sh_all[RC_WARPS];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    WarpSharedT &S = sh_all[warp];
    const int px = A.p.tile_x0 + blockIdx.x * (8 * RC_WARPS) + warp * 8 + (lane & 7);
    const int py = A.p.tile_y0 + blockIdx.y * 4 + (lane >> 3);
    const bool live = px < A.p.tile_x1 && py < A.p.tile_y1;
    const int w = A.cam.width, h = A.cam.height, res = A.res;
    const double ox = A.cam.pos[0], oy = A.cam.pos[1], oz = A.cam.pos[2];
    const bool clip = A.p.use_clip != 0;
    const double r = A.p.radius;
    const int kslots = A.p.k;
    const bool early = A.p.early_termination != 0;
    const double alpha = A.p.alpha;
    double dx = 0.0, dy = 0.0, dz = 1.0, t = 0.0, t1 = -1.0;
    bool active = false;
    if (live) {
        const double aspect = (double)w / (double)h;
        const double u = (2.0 * (px + 0.5) / w - 1.0) * aspect * A.cam.tan_half_fov;
        const double v = (1.0 - 2.0 * (py + 0.5) / h) * A.cam.tan_half_fov;
        dx = A.cam.fwd[0] + u * A.cam.right[0] + v * A.cam.up[0];
        dy = A.cam.fwd[1] + u * A.cam.right[1] + v * A.cam.up[1];
        dz = A.cam.fwd[2] + u * A.cam.right[2] + v * A.cam.up[2];
        const double dn = sqrt(dx * dx + dy * dy + dz * dz);
        dx = dx / dn; dy = dy / dn; dz = dz / dn;
        double t0 = 0.0;
        t1 = 1e30;
        const double o[3] = {ox, oy, oz}, d[3] = {dx, dy, dz};
#pragma unroll
        for (int a = 0; a < 3; a++) {
            if (d[a] == 0.0) {
                if (o[a] < 0.0 || o[a] > (double)res) { t0 = 1.0; t1 = -1.0; break; }
            } else {
                double ta = (0.0 - o[a]) / d[a], tb = ((double)res - o[a]) / d[a];
                if (ta > tb) { const double tmp = ta; ta = tb; tb = tmp; }
                if (ta > t0) t0 = ta;
                if (tb < t1) t1 = tb;
            }
        }
        active = t1 >= t0;
        t = t0 > 0.0 ? t0 : 0.0;
    }
    S.dir[0][lane] = dx; S.dir[1][lane] = dy; S.dir[2][lane] = dz;
    S.dirf[0][lane] = (float)dx; S.dirf[1][lane] = (float)dy; S.dirf[2][lane] = (float)dz;
    const float R2f = ((float)r + 2e-3f) * ((float)r + 2e-3f);
    const RayInv inv = make_inv(dx, dy, dz);
    int lvl_hint = 1;
    double col_r = 0.0, col_g = 0.0, col_b = 0.0, acc_a = 0.0;
    int64_t first_hit = -1;
    uint32_t keybuf[64], ibuf[64];
    double tbuf[64];
    uint64_t n_tests = 0;
    // per-voxel state of this lane's ray
    bool repeat = false;
    int64_t last_key = -1;
    uint32_t n = 0;
    double te = 0.0;
    int x = 0, y = 0, z = 0;
    __syncwarp();

    for (;;) {
        // ---- 1. next occupied voxel (or stay for a re-scan)
        if (active && !repeat) {
            for (;;) {
                if ((early && acc_a >= 0.999) || !(t < t1)) { active = false; break; }
                const double tm = t + 1e-6;
                x = (int)floor(ox + dx * tm); y = (int)floor(oy + dy * tm); z = (int)floor(oz + dz * tm);
                if (x < 0 || y < 0 || z < 0 || x >= res || y >= res || z >= res) { active = false; break; }
                const int64_t idx = x + (int64_t)res * (y + (int64_t)res * z);
                if (A.bits[idx] != 0) {
                    const uint32_t fo = A.offsets[idx];
                    n = A.offsets[idx + 1] - fo;
                    S.fo[lane] = fo;
                    te = voxel_exit(ox, oy, oz, dx, dy, dz, inv, x, y, z, 0);
                    const double span = te - t;                  // t_enter = t (lv/raytracer.py:557-560)
                    S.t_enter[lane] = t;
                    S.inv_span[lane] = span > 0.0 ? 65535.0 / span : 0.0;
                    last_key = -1;
                    break;
                }
                const int l = lvl_hint = empty_level(A, x, y, z, lvl_hint);
                const double tl = voxel_exit(ox, oy, oz, dx, dy, dz, inv, x, y, z, l);
                t = tl > t ? tl : t + 1e-6;
            }
        }
        if (__ballot_sync(0xffffffffu, active) == 0) break;
        S.vox[0][lane] = x; S.vox[1][lane] = y; S.vox[2][lane] = z;
        {   // a point of the ray inside the voxel (its centre-most parameter), for the f32 pre-test
            const double tc = 0.5 * (t + te);
            S.pf[0][lane] = (float)(ox + dx * tc); S.pf[1][lane] = (float)(oy + dy * tc); S.pf[2][lane] = (float)(oz + dz * tc);
        }
        // ---- 2. flatten (ray, fragment) pairs
        uint32_t inc = active ? n : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += v;
        }
        S.prefix[lane + 1] = inc;
        if (lane == 0) S.prefix[0] = 0;
        const uint32_t T = __shfl_sync(0xffffffffu, inc, 31);
        if (lane == 0) n_tests += T;
        int kept = 0;
        uint32_t accepted = 0;
        uint32_t qn = 0, hl_n = 0, own = 0;
        __syncwarp();

        // owners pull their records out of the hit list (insertion sort, lv/raytracer.py:589-607)
        auto drain = [&]() {
            for (uint32_t e = 0; e < hl_n; e++) {
                if (S.hl_r[e] != (uint8_t)lane) continue;
                const uint32_t key = S.hl_key[e];
                if ((int64_t)key <= last_key) continue;
                accepted++;
                int j;
                if (kept < kslots) { j = kept; kept++; }
                else if (key < keybuf[kslots - 1]) j = kslots - 1;
                else continue;
                while (j > 0 && keybuf[j - 1] > key) {
                    keybuf[j] = keybuf[j - 1]; tbuf[j] = tbuf[j - 1]; ibuf[j] = ibuf[j - 1];
                    j--;
                }
                keybuf[j] = key; tbuf[j] = S.hl_t[e]; ibuf[j] = S.hl_i[e];
            }
            hl_n = 0;
            __syncwarp();
        };

        for (uint32_t p0 = 0; p0 < T || qn > 0; p0 += 32) {
            const uint32_t p = p0 + lane;
            bool pass = false;
            uint32_t rr = 0, ss = 0, ii = 0;
            if (p < T) {
                while (S.prefix[own + 1] <= p) own++;       // owner ray: prefix[own] <= p < prefix[own+1]
                rr = own;
                ss = p - S.prefix[rr];
                ii = A.frags[S.fo[rr] + ss];
                pass = !surely_misses_f32(S.pf[0][rr], S.pf[1][rr], S.pf[2][rr], S.dirf[0][rr], S.dirf[1][rr],
                                          S.dirf[2][rr], A.verts_f, (int64_t)ii, R2f);
            }
            const uint32_t m = __ballot_sync(0xffffffffu, pass);
            if (pass) {
                const uint32_t pos = qn + __popc(m & ((1u << lane) - 1u));
                S.q_i[pos] = ii;
                S.q_rs[pos] = (rr << 16) | ss;
            }
            qn += __popc(m);
            __syncwarp();
            const bool flush = p0 + 32 >= T;
            if (qn >= 32 || (flush && qn > 0)) {
                const uint32_t take = qn < 32 ? qn : 32;
                bool hit = false;
                double ht = 0.0;
                uint32_t hr = 0, hs = 0, hi_ = 0, hkey = 0;
                if (lane < take) {
                    hi_ = S.q_i[lane];
                    const uint32_t rs = S.q_rs[lane];
                    hr = rs >> 16; hs = rs & 0xFFFFu;
                    const double ddx = S.dir[0][hr], ddy = S.dir[1][hr], ddz = S.dir[2][hr];
                    const Capsule c = load_capsule(A.verts, A.normals, (int64_t)hi_, r, clip);
                    ht = ray_capsule(ox, oy, oz, ddx, ddy, ddz, c);
                    if (ht >= 0.0) {
                        const int hx = (int)floor(ox + ddx * ht), hy = (int)floor(oy + ddy * ht), hz = (int)floor(oz + ddz * ht);
                        hit = hx == S.vox[0][hr] && hy == S.vox[1][hr] && hz == S.vox[2][hr];
                        if (hit) {   // lv/raytracer.py:583-588
                            int64_t q = (int64_t)((ht - S.t_enter[hr]) * S.inv_span[hr]);
                            if (q < 0) q = 0; else if (q > 65535) q = 65535;
                            hkey = ((uint32_t)q << 16) | hs;
                        }
                    }
                }
                __syncwarp();
                uint32_t mv_i = 0, mv_rs = 0;
                const bool mv = lane + 32 < qn;
                if (mv) { mv_i = S.q_i[lane + 32]; mv_rs = S.q_rs[lane + 32]; }
                __syncwarp();
                if (mv) { S.q_i[lane] = mv_i; S.q_rs[lane] = mv_rs; }
                qn -= take;
                const uint32_t hm = __ballot_sync(0xffffffffu, hit);
                if (hl_n + __popc(hm) > HL_CAP) drain();
                if (hit) {
                    const uint32_t pos = hl_n + __popc(hm & ((1u << lane) - 1u));
                    S.hl_t[pos] = ht; S.hl_key[pos] = hkey; S.hl_i[pos] = hi_; S.hl_r[pos] = (uint8_t)hr;
                }
                hl_n += __popc(hm);
                __syncwarp();
            }
            if (flush && qn == 0) break;
        }
        drain();
        // ---- blend the kept hits front to back (lv/raytracer.py:608-631)
        if (active) {
            for (int j = 0; j < kept; j++) {
                if (early && acc_a >= 0.999) break;
                const double tt = tbuf[j];
                const int64_t i = ibuf[j];
                const double hx = ox + dx * tt, hy = oy + dy * tt, hz = oz + dz * tt;
                const Capsule c = load_capsule(A.verts, A.normals, i, r, clip);
                double nx, ny, nz, cr, cg, cb;
                capsule_normal(hx, hy, hz, c, nx, ny, nz);
                shade(A, c, nx, ny, nz, hx, hy, hz, cr, cg, cb);
                const double wgt = (1.0 - acc_a) * alpha;
                col_r += wgt * cr; col_g += wgt * cg; col_b += wgt * cb;
                acc_a += wgt;
                if (first_hit < 0) first_hit = i;
            }
            // lv/raytracer.py:632-637
            if (accepted <= (uint32_t)kslots || (early && acc_a >= 0.999)) {
                repeat = false;
                t = te > t ? te : t + 1e-6;
            } else {
                last_key = keybuf[kslots - 1];
                repeat = true;
            }
        }
        __syncwarp();
    }

    if (live) {
        const double out_r = col_r + (1.0 - acc_a) * A.p.background[0];
        const double out_g = col_g + (1.0 - acc_a) * A.p.background[1];
        const double out_b = col_b + (1.0 - acc_a) * A.p.background[2];
        const int64_t pix = (int64_t)py * w + px;
        if (A.rgb) { A.rgb[3 * pix] = out_r; A.rgb[3 * pix + 1] = out_g; A.rgb[3 * pix + 2] = out_b; }
        if (A.srgb) { A.srgb[3 * pix] = to_srgb8(out_r); A.srgb[3 * pix + 1] = to_srgb8(out_g); A.srgb[3 * pix + 2] = to_srgb8(out_b); }
        A.hit_id[pix] = (int32_t)first_hit;
    }
    if (lane == 0 && n_tests)
        atomicAdd((unsigned long long *)&A.stats[LVX_ST_RAY_TESTS], (unsigned long long)n_tests);
}

// Second half of shading on demand: one thread per pixel re-derives its ray (same expressions,
// hence the same bits, as the trace kernel), and shades the recorded hit.
__global__ void __launch_bounds__(128)
k_resolve(const RenderArgs A) {
    const int px = A.p.tile_x0 + blockIdx.x * 32 + (threadIdx.x & 31);
    const int py = A.p.tile_y0 + blockIdx.y * 4 + (threadIdx.x >> 5);
    if (px >= A.p.tile_x1 || py >= A.p.tile_y1) return;
    const int w = A.cam.width, h = A.cam.height;
    const int64_t pix = (int64_t)py * w + px;
    double out_r = A.p.background[0], out_g = A.p.background[1], out_b = A.p.background[2];
    const double best_t = A.hit_t[pix];
    if (best_t >= 0.0) {
        const double aspect = (double)w / (double)h;
        const double u = (2.0 * (px + 0.5) / w - 1.0) * aspect * A.cam.tan_half_fov;
        const double v = (1.0 - 2.0 * (py + 0.5) / h) * A.cam.tan_half_fov;
        double dx = A.cam.fwd[0] + u * A.cam.right[0] + v * A.cam.up[0];
        double dy = A.cam.fwd[1] + u * A.cam.right[1] + v * A.cam.up[1];
        double dz = A.cam.fwd[2] + u * A.cam.right[2] + v * A.cam.up[2];
        const double dn = sqrt(dx * dx + dy * dy + dz * dz);
        dx = dx / dn; dy = dy / dn; dz = dz / dn;
        const double hx = A.cam.pos[0] + dx * best_t, hy = A.cam.pos[1] + dy * best_t, hz = A.cam.pos[2] + dz * best_t;
        const Capsule c = load_capsule(A.verts, A.normals, (int64_t)A.hit_id[pix], A.p.radius, A.p.use_clip != 0);
        double nx, ny, nz;
        capsule_normal(hx, hy, hz, c, nx, ny, nz);
        shade(A, c, nx, ny, nz, hx, hy, hz, out_r, out_g, out_b);
    }
    if (A.rgb) { A.rgb[3 * pix] = out_r; A.rgb[3 * pix + 1] = out_g; A.rgb[3 * pix + 2] = out_b; }
    if (A.srgb) { A.srgb[3 * pix] = to_srgb8(out_r); A.srgb[3 * pix + 1] = to_srgb8(out_g); A.srgb[3 * pix + 2] = to_srgb8(out_b); }
}

}  // namespace lvx

using namespace lvx;

static int fill_args(RenderArgs &A, const double *verts, const float *verts_f, const double *normals, const uint32_t *offsets,
                     const uint32_t *frags, const uint8_t *bits_flat, int res, const float *ao, const float *shadow,
                     const lvx_camera *cam_host, const lvx_render_params *params_host, double *rgb, uint8_t *srgb,
                     int32_t *hit_id, uint64_t *stats) {
    if (!pow2(res) || !cam_host || !params_host || !hit_id) return LVX_E_ARG;
    const lvx_render_params &p = *params_host;
    if (p.mode < 0 || p.mode > 1 || p.k < 1 || p.k > 64 || !(p.alpha > 0.0 && p.alpha <= 1.0)) return LVX_E_ARG;
    if (cam_host->width <= 0 || cam_host->height <= 0) return LVX_E_ARG;
    if (p.tile_x0 < 0 || p.tile_y0 < 0 || p.tile_x1 > cam_host->width || p.tile_y1 > cam_host->height) return LVX_E_ARG;
    if (p.use_clip && !normals) return LVX_E_ARG;
    A.verts = verts; A.verts_f = verts_f; A.normals = normals; A.offsets = offsets; A.frags = frags; A.bits = bits_flat;
    A.ao = ao; A.sh = shadow;
    const LevelOffsets L = make_level_offsets(res);
    for (int l = 0; l < 16; l++) A.bits_off[l] = l < L.n_levels ? (uint32_t)L.off[l] : 0;
    A.res = res; A.n_levels = L.n_levels; A.cam = *cam_host; A.p = p;
    A.rgb = rgb; A.srgb = srgb; A.hit_id = hit_id; A.stats = stats;
    A.hit_t = nullptr; A.need_bits = nullptr; A.need_list = nullptr; A.guard_volumes = 0;
    return LVX_OK;
}

extern "C" {

int lvx_render(const double *verts, const float *verts_f, const double *normals, const uint32_t *offsets, const uint32_t *frags,
               const uint8_t *bits_flat, int res, const float *ao, const float *shadow,
               const lvx_camera *cam_host, const lvx_render_params *params_host, double *rgb, uint8_t *srgb,
               int32_t *hit_id, uint64_t *stats, void *stream) {
    RenderArgs A;
    const int rc = fill_args(A, verts, verts_f, normals, offsets, frags, bits_flat, res, ao, shadow, cam_host, params_host,
                             rgb, srgb, hit_id, stats);
    if (rc != LVX_OK) return rc;
    if (!verts_f) return LVX_E_ARG;
    const int tw = A.p.tile_x1 - A.p.tile_x0, th = A.p.tile_y1 - A.p.tile_y0;
    if (tw <= 0 || th <= 0) return LVX_OK;
    if (A.p.mode == 0) {
        const dim3 cgrid((tw + 8 * RC_WARPS - 1) / (8 * RC_WARPS), (th + 3) / 4);
        k_render_opaque_coop<false><<<cgrid, RC_WARPS * 32, 0, (cudaStream_t)stream>>>(A);
    } else {
        const dim3 cgrid((tw + 8 * RC_WARPS - 1) / (8 * RC_WARPS), (th + 3) / 4);
        k_render_transparent_coop<<<cgrid, RC_WARPS * 32, 0, (cudaStream_t)stream>>>(A);
    }
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

int lvx_trace_hits(const double *verts, const float *verts_f, const double *normals, const uint32_t *offsets, const uint32_t *frags,
                   const uint8_t *bits_flat, int res, const lvx_camera *cam_host,
                   const lvx_render_params *params_host, double *hit_t, int32_t *hit_id, uint32_t *need_bits,
                   uint32_t *need_list, uint64_t *stats, void *stream) {
    RenderArgs A;
    const int rc = fill_args(A, verts, verts_f, normals, offsets, frags, bits_flat, res, nullptr, nullptr, cam_host,
                             params_host, nullptr, nullptr, hit_id, stats);
    if (rc != LVX_OK) return rc;
    if (A.p.mode != 0 || !verts_f || !hit_t || !need_bits || !need_list) return LVX_E_ARG;
    const int tw = A.p.tile_x1 - A.p.tile_x0, th = A.p.tile_y1 - A.p.tile_y0;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t V = (int64_t)res * res * res;
    LVX_CUDA(cudaMemsetAsync(need_bits, 0, (size_t)((V + 31) / 32) * 4, s));
    LVX_CUDA(cudaMemsetAsync(need_list, 0, 8, s));
    if (tw <= 0 || th <= 0) return LVX_OK;
    A.hit_t = hit_t; A.need_bits = need_bits; A.need_list = need_list;
    const dim3 cgrid((tw + 8 * RC_WARPS - 1) / (8 * RC_WARPS), (th + 3) / 4);
    k_render_opaque_coop<true><<<cgrid, RC_WARPS * 32, 0, s>>>(A);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

int lvx_resolve(const double *verts, const double *normals, const uint8_t *bits_flat, int res, const float *ao,
                const float *shadow, const lvx_camera *cam_host, const lvx_render_params *params_host,
                const double *hit_t, const int32_t *hit_id, double *rgb, uint8_t *srgb, void *stream) {
    RenderArgs A;
    const int rc = fill_args(A, verts, nullptr, normals, nullptr, nullptr, bits_flat, res, ao, shadow, cam_host, params_host,
                             rgb, srgb, const_cast<int32_t *>(hit_id), nullptr);
    if (rc != LVX_OK) return rc;
    if (!hit_t) return LVX_E_ARG;
    const int tw = A.p.tile_x1 - A.p.tile_x0, th = A.p.tile_y1 - A.p.tile_y0;
    if (tw <= 0 || th <= 0) return LVX_OK;
    A.hit_t = const_cast<double *>(hit_t);
    A.guard_volumes = 1;
    const dim3 grid((tw + 31) / 32, (th + 3) / 4);
    k_resolve<<<grid, 128, 0, (cudaStream_t)stream>>>(A);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

}  // extern "C"
