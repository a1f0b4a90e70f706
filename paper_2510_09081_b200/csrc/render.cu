// render.cu -- image-order voxel ray tracing: grid clip, hierarchical empty-space skip, face-to-face
// DDA, analytic clipped ray-capsule intersection, opaque first hit or exact ordered k-buffer
// transparency, AO/shadow lookup.  Replaces lv/raytracer.py:113-256 (_ray_capsule,
// _capsule_normal), 272-347 (marching helpers), 368-423 (_tri3d, _shade, _pixel_ray), 430-515
// (_voxel_best_hit, _opaque_kernel), 518-645 (_transparent_kernel) and 94-97 (_to_srgb).
#include "lvx_device.cuh"

namespace lvx {

struct RenderArgs {
    const double *verts, *normals;
    const uint32_t *offsets, *frags;
    const uint8_t *bits;
    const float *ao, *sh;
    int64_t bits_off[16];
    int res, n_levels;
    lvx_camera cam;
    lvx_render_params p;
    double *rgb;
    uint8_t *srgb;
    int32_t *hit_id;
    uint64_t *stats;
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

// lv/raytracer.py:294-313
__device__ __forceinline__ double voxel_exit(double ox, double oy, double oz, double dx, double dy, double dz,
                                             int x, int y, int z, int lvl) {
    const int size = 1 << lvl;
    const int bx = (x >> lvl) << lvl, by = (y >> lvl) << lvl, bz = (z >> lvl) << lvl;
    double t = 1e30;
    if (dx > 0.0) t = fmin(t, ((double)(bx + size) - ox) / dx); else if (dx < 0.0) t = fmin(t, ((double)bx - ox) / dx);
    if (dy > 0.0) t = fmin(t, ((double)(by + size) - oy) / dy); else if (dy < 0.0) t = fmin(t, ((double)by - oy) / dy);
    if (dz > 0.0) t = fmin(t, ((double)(bz + size) - oz) / dz); else if (dz < 0.0) t = fmin(t, ((double)bz - oz) / dz);
    return t;
}

// lv/raytracer.py:316-326
__device__ __forceinline__ int empty_level(const RenderArgs &A, int x, int y, int z) {
    int l = 0;
    while (l < A.n_levels - 1) {
        const int nl = l + 1;
        const int64_t rl = A.res >> nl;
        if (A.bits[A.bits_off[nl] + (x >> nl) + rl * ((y >> nl) + rl * (z >> nl))] != 0) break;
        l = nl;
    }
    return l;
}

// lv/raytracer.py:368-390 (volumes are f32, widened exactly like the reference's astype(f64))
__device__ __forceinline__ double tri3d(const float *__restrict__ vol, int res, double px, double py, double pz) {
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
                acc += wx * wy * wz * (double)vol[x + (int64_t)res * (y + (int64_t)res * z)];
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
    const double ao = A.ao ? tri3d(A.ao, A.res, px, py, pz) : 1.0;
    const double sh = A.sh ? tri3d(A.sh, A.res, px, py, pz) : 1.0;
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
                        te = voxel_exit(ox, oy, oz, dx, dy, dz, x, y, z, 0);
                    } else {
                        const int l = empty_level(A, x, y, z);
                        te = voxel_exit(ox, oy, oz, dx, dy, dz, x, y, z, l);
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
                        const int l = empty_level(A, x, y, z);
                        const double te = voxel_exit(ox, oy, oz, dx, dy, dz, x, y, z, l);
                        t = te > t ? te : t + 1e-6;
                        continue;
                    }
                    const double te = voxel_exit(ox, oy, oz, dx, dy, dz, x, y, z, 0);
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

}  // namespace lvx

using namespace lvx;

extern "C" {

int lvx_render(const double *verts, const double *normals, const uint32_t *offsets, const uint32_t *frags,
               const uint8_t *bits_flat, int res, const float *ao, const float *shadow,
               const lvx_camera *cam_host, const lvx_render_params *params_host, double *rgb, uint8_t *srgb,
               int32_t *hit_id, uint64_t *stats, void *stream) {
    if (!pow2(res) || !cam_host || !params_host || !hit_id) return LVX_E_ARG;
    const lvx_render_params &p = *params_host;
    if (p.mode < 0 || p.mode > 1 || p.k < 1 || p.k > 64 || !(p.alpha > 0.0 && p.alpha <= 1.0)) return LVX_E_ARG;
    if (cam_host->width <= 0 || cam_host->height <= 0) return LVX_E_ARG;
    if (p.tile_x0 < 0 || p.tile_y0 < 0 || p.tile_x1 > cam_host->width || p.tile_y1 > cam_host->height) return LVX_E_ARG;
    if (p.use_clip && !normals) return LVX_E_ARG;
    const int tw = p.tile_x1 - p.tile_x0, th = p.tile_y1 - p.tile_y0;
    if (tw <= 0 || th <= 0) return LVX_OK;
    RenderArgs A;
    A.verts = verts; A.normals = normals; A.offsets = offsets; A.frags = frags; A.bits = bits_flat;
    A.ao = ao; A.sh = shadow;
    const LevelOffsets L = make_level_offsets(res);
    for (int l = 0; l < 16; l++) A.bits_off[l] = l < L.n_levels ? L.off[l] : 0;
    A.res = res; A.n_levels = L.n_levels; A.cam = *cam_host; A.p = p;
    A.rgb = rgb; A.srgb = srgb; A.hit_id = hit_id; A.stats = stats;
    const dim3 grid((tw + 7) / 8, (th + 15) / 16);
    if (p.mode == 0) k_render<0><<<grid, 128, 0, (cudaStream_t)stream>>>(A);
    else k_render<1><<<grid, 128, 0, (cudaStream_t)stream>>>(A);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

}  // extern "C"
