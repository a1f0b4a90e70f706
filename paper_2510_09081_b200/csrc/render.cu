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
    // tight index (abuffer.cu; all three NULL = none): per voxel the fragments whose capsule can reach
    // into the voxel, compacted to the front of the list's range, with their slots in the full list
    const uint32_t *tfrags;
    const uint16_t *tslot, *tcnt;
    const uint8_t *march;      // per voxel: 255 = occupied/visible, else the empty level (lvx_march_levels)
    const float *ao, *sh;
    int res;
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
    int guard_volumes;       // ao/sh hold values only where requested: read 1.0 where march[] != 255
};

__device__ __forceinline__ bool clip_ok(const Capsule &c, double px, double py, double pz) {
    if (!c.clip) return true;
    if ((px - c.a.x) * c.n0.x + (py - c.a.y) * c.n0.y + (pz - c.a.z) * c.n0.z < -1e-9) return false;
    if ((px - c.b.x) * c.n1.x + (py - c.b.y) * c.n1.y + (pz - c.b.z) * c.n1.z > 1e-9) return false;
    return true;
}

// Conservative miss test (single precision).  An accepted hit is a point of the ray that lies
// inside the voxel being visited (lv/raytracer.py:446-452) and within r + 3.2e-5 of the segment
// [a, b] (every surface the f64 routine can return is that close to the capsule's axis).  The ray's
// stretch inside the voxel is contained in {C + s*D, |s| <= h}: C = the ray point half-way between
// the voxel's entry and exit parameters, h = half their difference + 1e-3 (the march parameters
// differ from the geometric entry/exit by at most the reference's 1e-6 nudges).  So if the
// distance between that stretch and the segment exceeds r + 2e-3 the pair cannot produce an
// accepted hit.  The closest-points computation is the standard clamped two-segment solve; all
// differences are a few voxels long and the f32 inputs are rounded at magnitudes <= 1024
// (<= 6.1e-5 absolute), which the 2e-3 margin covers several times.  ~55 full-rate operations
// against ~500 half-rate f64 ones for the exact routine, and unlike a ray-LINE test it also rejects
// capsules the ray only reaches before or after this voxel.
__device__ __forceinline__ bool surely_misses_f32(float Cx, float Cy, float Cz, float h, float Dx, float Dy, float Dz,
                                                  const float *__restrict__ vf, int64_t i, float R2) {
    const float ax = vf[3 * i], ay = vf[3 * i + 1], az = vf[3 * i + 2];
    const float bx = vf[3 * i + 3], by = vf[3 * i + 4], bz = vf[3 * i + 5];
    const float wx = ax - Cx, wy = ay - Cy, wz = az - Cz;
    const float ex = bx - ax, ey = by - ay, ez = bz - az;
    // (explicit fmaf: the translation unit is compiled with -fmad=false for the f64 code)
    const float dw = fmaf(Dx, wx, fmaf(Dy, wy, Dz * wz)), de = fmaf(Dx, ex, fmaf(Dy, ey, Dz * ez));
    const float ee = fmaf(ex, ex, fmaf(ey, ey, ez * ez)), ew = fmaf(ex, wx, fmaf(ey, wy, ez * wz));
    const float den = fmaf(-de, de, ee);                    // |D| = 1
    // Nearly parallel ray and segment: den = ee sin^2(angle) carries ~1e-7 ee of rounding, so below
    // sin^2 = 1e-4 the closest-pair parameter would be noise and the distance an OVER-estimate of up to
    // ~2e-3 voxel^2 -- more than the margin.  Such pairs go to the exact f64 test instead.
    if (ee > 1e-12f && !(den > 1e-4f * ee)) return false;
    float sr = 0.f;                                         // parameter on the ray stretch
    if (den > 1e-12f) sr = fminf(fmaxf(__fdividef(fmaf(dw, ee, -de * ew), den), -h), h);
    float u = 0.f;                                          // parameter on the segment
    if (ee > 1e-12f) {
        u = __fdividef(fmaf(de, sr, -ew), ee);
        if (u < 0.f) { u = 0.f; sr = fminf(fmaxf(dw, -h), h); }
        else if (u > 1.f) { u = 1.f; sr = fminf(fmaxf(dw + de, -h), h); }
    } else {
        sr = fminf(fmaxf(dw, -h), h);
    }
    const float qx = fmaf(u, ex, fmaf(-sr, Dx, wx)), qy = fmaf(u, ey, fmaf(-sr, Dy, wy)), qz = fmaf(u, ez, fmaf(-sr, Dz, wz));
    return fmaf(qx, qx, fmaf(qy, qy, qz * qz)) > R2;
}

// lv/raytracer.py:113-222: smallest t >= 0 on the clipped capsule surface, or -1.
// The candidate loops are deliberately NOT unrolled: the routine is executed by few lanes at a time and
// the cooperative kernels were stalling on instruction fetch (ncu: 26 % no_instruction stalls at
// ~7000 SASS instructions per kernel); rolled loops execute the same operations in the same order.
// `sub` < 0: all candidate surfaces.  `sub` = 0 / 1: only the first / second candidate of each pair
// (near / far cylinder root, end sphere a / b, clip plane a / b) -- two lanes then share one test and
// the smaller of their results is the routine's result (a minimum does not depend on the order).
__device__ double ray_capsule(double ox, double oy, double oz, double dx, double dy, double dz, const Capsule &c,
                              int sub = -1) {
    const int k0 = sub < 0 ? 0 : sub, k1 = sub < 0 ? 2 : sub + 1;
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
#pragma unroll 1
                for (int k = k0; k < k1; k++) {
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
#pragma unroll 1
    for (int cap = k0; cap < k1; cap++) {
        const double cx = cap ? bx : ax, cy = cap ? by : ay, cz = cap ? bz : az;
        const double ocx = ox - cx, ocy = oy - cy, ocz = oz - cz;
        const double bq = ocx * dx + ocy * dy + ocz * dz;
        const double cq = ocx * ocx + ocy * ocy + ocz * ocz - r * r;
        const double disc = bq * bq - cq;
        if (disc < 0.0) continue;
        const double sq = sqrt(disc);
#pragma unroll 1
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
#pragma unroll 1
        for (int pl = k0; pl < k1; pl++) {
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

// lv/raytracer.py:294-313: t = min over the axes of (face - o) / d.
// The three IEEE quotients are formed without the division instruction sequence.  With
// y = RN(1/d) (computed once per ray by a true division) and q0 = RN(n*y), two Markstein
// corrections q <- fma(fma(-d, q, n), y, q) give the correctly rounded n/d: after the first one q
// is a faithful approximation, and Markstein's theorem (Muller et al., Handbook of FP Arithmetic,
// Thm 4.9) makes the second one exact.  (No overflow/underflow here: |n| <= 2048 and a component
// of a unit vector is either 0 -- axis skipped -- or >= 2^-1074; components below 1e-280 are
// treated as 0-free by the guarded path.)  5 dependent f64 instructions per axis, branch-free.
struct RayInv { double ix, iy, iz; bool slow; };
__device__ __forceinline__ RayInv make_inv(double dx, double dy, double dz) {
    const double tiny = 1e-280;
    const bool slow = (dx != 0.0 && fabs(dx) <= tiny) || (dy != 0.0 && fabs(dy) <= tiny) || (dz != 0.0 && fabs(dz) <= tiny);
    return RayInv{dx != 0.0 ? 1.0 / dx : 0.0, dy != 0.0 ? 1.0 / dy : 0.0, dz != 0.0 ? 1.0 / dz : 0.0, slow};
}
__device__ __forceinline__ double exact_quot(double n, double d, double y) {
    double q = n * y;
    q = __fma_rn(__fma_rn(-d, q, n), y, q);
    q = __fma_rn(__fma_rn(-d, q, n), y, q);
    return q;
}
// the literal form (true divisions), for rays with a denormal-range direction component
__device__ __noinline__ double voxel_exit_slow(double ox, double oy, double oz, double dx, double dy, double dz,
                                               int x, int y, int z, int lvl) {
    const int size = 1 << lvl;
    const int bx = (x >> lvl) << lvl, by = (y >> lvl) << lvl, bz = (z >> lvl) << lvl;
    double t = 1e30;
    if (dx != 0.0) t = fmin(t, ((double)(dx > 0.0 ? bx + size : bx) - ox) / dx);
    if (dy != 0.0) t = fmin(t, ((double)(dy > 0.0 ? by + size : by) - oy) / dy);
    if (dz != 0.0) t = fmin(t, ((double)(dz > 0.0 ? bz + size : bz) - oz) / dz);
    return t;
}
__device__ __forceinline__ double voxel_exit(double ox, double oy, double oz, double dx, double dy, double dz,
                                             const RayInv &inv, int x, int y, int z, int lvl) {
    if (inv.slow) return voxel_exit_slow(ox, oy, oz, dx, dy, dz, x, y, z, lvl);
    // far face of the level-lvl node per axis: ((c >> lvl) + [d > 0]) << lvl
    const double nx = (double)(((x >> lvl) + (dx > 0.0 ? 1 : 0)) << lvl) - ox;
    const double ny = (double)(((y >> lvl) + (dy > 0.0 ? 1 : 0)) << lvl) - oy;
    const double nz = (double)(((z >> lvl) + (dz > 0.0 ? 1 : 0)) << lvl) - oz;
    const double big = 1e30;
    const double tx = dx != 0.0 ? exact_quot(nx, dx, inv.ix) : big;
    const double ty = dy != 0.0 ? exact_quot(ny, dy, inv.iy) : big;
    const double tz = dz != 0.0 ? exact_quot(nz, dz, inv.iz) : big;
    return fmin(fmin(fmin(big, tx), ty), tz);
}

// lv/raytracer.py:368-390 (volumes are f32, widened exactly like the reference's astype(f64)).
// The AO and the shadow volume are sampled at the same point, so the corner indices and weights
// are formed once; each sum keeps the reference's order of additions.
struct ShadeCtx {
    const double *verts, *normals;
    const float *ao, *sh;
    const uint8_t *guard;      // non-NULL: volumes hold values only where guard[idx] == 255, 1.0 elsewhere
    int res, clip;
    double r, l0, l1, l2;      // capsule radius, direction to the light
};
__device__ __forceinline__ ShadeCtx make_shade_ctx(const RenderArgs &A) {
    return ShadeCtx{A.verts, A.normals, A.ao, A.sh, A.guard_volumes ? A.march : nullptr, A.res, A.p.use_clip != 0,
                    A.p.radius, A.p.light_to_source[0], A.p.light_to_source[1], A.p.light_to_source[2]};
}

#if defined(LVX_COUNT) && LVX_COUNT == 3
__device__ uint32_t g_dbg_bits[1 << 22];      // debug: voxels whose AO/shadow some blended hit reads (res <= 512)
__device__ unsigned long long g_dbg_unique;
#endif
__device__ __forceinline__ void tri3d2(const ShadeCtx &cx, double px, double py, double pz, double &ao, double &sh) {
    const int res = cx.res;
    const double ux = px - 0.5, uy = py - 0.5, uz = pz - 0.5;
    const int ix = (int)floor(ux), iy = (int)floor(uy), iz = (int)floor(uz);
    const double fx = ux - ix, fy = uy - iy, fz = uz - iz;
    double acc_a = 0.0, acc_s = 0.0;
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
                const bool unit = cx.guard && cx.guard[idx] != 255;
#if defined(LVX_COUNT) && LVX_COUNT == 3
                { const uint32_t bit = 1u << (idx & 31);
                  if (!(atomicOr(&g_dbg_bits[idx >> 5], bit) & bit)) atomicAdd(&g_dbg_unique, 1ull); }
#endif
                const double w = wx * wy * wz;
                if (cx.ao) acc_a += w * (unit ? 1.0 : (double)cx.ao[idx]);
                if (cx.sh) acc_s += w * (unit ? 1.0 : (double)cx.sh[idx]);
            }
        }
    }
    ao = cx.ao ? acc_a : 1.0;
    sh = cx.sh ? acc_s : 1.0;
}

// lv/raytracer.py:393-411
__device__ __forceinline__ void shade(const ShadeCtx &cx, const Capsule &c, double nx, double ny, double nz,
                                      double px, double py, double pz, double &cr, double &cg, double &cb) {
    const double sx = c.b.x - c.a.x, sy = c.b.y - c.a.y, sz = c.b.z - c.a.z;
    const double sn = sqrt(sx * sx + sy * sy + sz * sz);
    if (sn == 0.0) { cr = cg = cb = 0.5; }
    else { cr = fabs(sx) / sn; cg = fabs(sy) / sn; cb = fabs(sz) / sn; }
    double ao, sh;
    tri3d2(cx, px, py, pz, ao, sh);
    double ndl = nx * cx.l0 + ny * cx.l1 + nz * cx.l2;
    if (ndl < 0.0) ndl = 0.0;
    const double k = 0.4 * ao + 0.6 * sh * ndl;
    cr = cr * k; cg = cg * k; cb = cb * k;
}

// normal + colour of the hit of segment i at (hx, hy, hz) (lv/raytracer.py:502-505, 612-620)
struct rgb3 { double r, g, b; };
__device__ __forceinline__ rgb3 shade_hit_inl(const ShadeCtx &cx, int64_t i, double hx, double hy, double hz) {
    const Capsule c = load_capsule(cx.verts, cx.normals, i, cx.r, cx.clip != 0);
    double nx, ny, nz;
    rgb3 o;
    capsule_normal(hx, hy, hz, c, nx, ny, nz);
    shade(cx, c, nx, ny, nz, hx, hy, hz, o.r, o.g, o.b);
    return o;
}
// One out-of-line copy for the transparent kernel, which shades from two places: the kernel's code
// size, not its arithmetic, is what limits it (ncu: instruction-fetch stalls lead the stall list).
__device__ __noinline__ rgb3 shade_hit(const ShadeCtx *cx, int64_t i, double hx, double hy, double hz) {
    return shade_hit_inl(*cx, i, hx, hy, hz);
}

__device__ __forceinline__ uint8_t to_srgb8(double v) {   // lv/raytracer.py:94-97
    const double c = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
    const double s = c <= 0.0031308 ? 12.92 * c : 1.055 * pow(c, 1.0 / 2.4) - 0.055;
    return (uint8_t)(int)rint(s * 255.0);
}

// ----------------------------------------------------------------------------- warp-cooperative tracing
// A per-pixel loop spends most of its instructions in the heavy f64 intersection with 2-3 of 32
// lanes active (ncu: profiles/r01c).  The kernels below keep the reference's per-ray semantics
// (lv/raytracer.py:459-515, 518-645) but share the work of a warp's 8x4 pixel tile.  Per round:
//   1. every unfinished ray marches to its next occupied voxel: one byte of the march table per
//      DDA step says "occupied" or how large the surrounding empty node is (hierarchical skip);
//   2./3. stage A: each lane walks the tight ranges of its voxels (abuffer.cu: the fragments whose
//      capsule can reach into the voxel, compacted by the ordering pass) and the lanes push them,
//      one per lane per step, into queue A (ballot + popc compaction);
//   4. stage B: 32 queued pairs at a time read the fragment's segment (f32 copy) and run the cheap
//      conservative miss test fully converged; survivors are compacted into queue B;
//   5. stage C: 32 queued pairs at a time run the full clipped f64 ray-capsule routine; accepted
//      hits are folded on the owning lane (opaque: min t, first slot wins ties -- 453; transparent:
//      per-warp hit list -> per-lane k-slot buffers).
// Pairs are taken from the back of the queues; the order of processing never matters because
// hits are folded with an order-independent rule.
constexpr int RC_WARPS = 4;
#define LVX_FULL 0xffffffffu
// Values derived from threadIdx that live for the whole kernel (lane, the warp's shared-memory
// offset, the lower-lanes mask).  Under register pressure ptxas rematerialises them at every use
// -- S2R + shifts were ~10 % of the executed instructions (ncu source view); an empty volatile asm
// makes the value opaque, so it stays in its register.
#define LVX_PIN(x) asm volatile("" : "+r"(x))
// -DLVX_COUNT: debug build that counts the work of each stage in the spare stats words
// (12: occupied voxels recorded, 13: tight pairs queued, 14: pairs surviving the f32 test, 15: accepted hits)
#ifdef LVX_COUNT
#define LVX_CNT(slot, n) do { if (lane == 0 && (n)) atomicAdd((unsigned long long *)&A.stats[slot], (unsigned long long)(n)); } while (0)
#else
#define LVX_CNT(slot, n) do { } while (0)
#endif
#ifndef LVX_SPEC
#define LVX_SPEC 5      // occupied voxels a ray walks ahead per round (opaque).  Measured on C2 with the tight
                        // index: 2 -> 2.39 ms, 3 -> 2.27, 4 -> 1.96, 5 -> 1.91, 6 -> 1.93, 8 -> 1.96 (at 5 CTAs/SM)
#endif
#ifndef LVX_SPEC_T
#define LVX_SPEC_T 4    // ... per round (transparent: rays rarely stop early, so deeper is cheap)
#endif

// Speculation.  A round costs a fixed chain of dependent loads and flushes of half-empty
// batches, so every ray records its next M occupied voxels per round (the DDA does not depend on
// hit results) and the pairs of all M voxels go through stages A-C together.  Results are then
// consumed in voxel order ("ordinal" m), exactly like the reference would: the first ordinal
// with a hit ends an opaque ray, a transparent ray blends ordinal by ordinal and stops where the
// reference stops.  Work done for ordinals behind that point is discarded and not counted.
template <int M>
struct PairQueues {
    double dir[3][32];
    float dirf[3][32];
    float pf[M][3][32];             // the ray's mid point inside voxel m (f32, for the conservative pre-test)
    float hf[M][32];                // ... and half the parameter length of its stretch there (+ margin)
    int16_t vox[M][3][32];          // res <= 1024
    uint32_t fo[M][32], n[M][32];   // fragment list of voxel m (n = 0: none)
    uint16_t tn[M][32];             // ... of which the first tn entries of the tight index are worth testing
    uint32_t qa_rs[64], qa_g[64];   // queue A: (ordinal << 21 | ray << 16 | index in the range), global index
    uint32_t qb_rs[64], qb_i[64];   // queue B: same tag, segment index
};
#define LVX_RS_RAY(rs) (((rs) >> 16) & 31u)
#define LVX_RS_ORD(rs) ((rs) >> 21)
#define LVX_RS_SLOT(rs) ((rs) & 0xFFFFu)

// Runs stages A-C for one round over the lists S.fo/S.n[0..n_ord) of every lane (n_ord <= M);
// `stage_c(valid, rs, seg, last, sub)` is called with 32 (or fewer, at the end) queue-B entries; the
// final call has last = true (and possibly no valid entry at all).  sub >= 0: lanes 2e and 2e+1 both
// hold entry e and evaluate candidate subset `sub` (see ray_capsule); the callee merges the pair.
// Written as one loop with a single call site per stage: the stages are large (stage C inlines the
// f64 intersection routine), and every extra inlined copy costs instruction-cache capacity.
// `last_ord()`: the highest ordinal this lane's ray still needs (opaque: the ordinal of the best hit found so
// far -- stage C of its early pairs has usually run by the time stage A reaches its later voxels; n_ord - 1 when
// every ordinal is needed).  Ordinals beyond it are not queued at all.
template <int M, class F, class G>
__device__ __forceinline__ void run_pairs(const RenderArgs &A, PairQueues<M> &S, int n_ord, int lane, uint32_t lt_mask,
                                          float R2f, F &&stage_c, G &&last_ord) {
    uint32_t qa = 0, qb = 0;
    // stage-A cursor of this lane: ordinal m, next global index g of its range, entries left, index in the range
    int m = -1;
    uint32_t g = 0, left = 0, idx = 0, tag = 0;
    bool a_done = false;
    for (;;) {
        // ---- stage C: full batches, or whatever is left once the producers are done
        const bool tail = a_done && qa == 0;
        if (qb >= 32 || tail) {
            const uint32_t take = qb < 32 ? qb : 32, base = qb - take;
            // a batch of at most 16 pairs is spread over two lanes per pair: each lane evaluates half
            // of the candidate surfaces of the f64 routine (ray_capsule's `sub`)
            const bool split = take <= 16;
            const uint32_t e = split ? (uint32_t)lane >> 1 : (uint32_t)lane;
            const bool valid = e < take;
            const uint32_t rs = valid ? S.qb_rs[base + e] : 0, ii = valid ? S.qb_i[base + e] : 0;
            qb = base;
            __syncwarp();
            const bool fin = tail && qb == 0;
            stage_c(valid, rs, ii, fin, split ? (lane & 1) : -1);
            if (fin) break;
            continue;
        }
        // ---- stage B: conservative f32 miss test on (up to) 32 queued pairs, survivors -> queue B
        if (qa >= 32 || (a_done && qa > 0)) {
            const uint32_t take = qa < 32 ? qa : 32, base = qa - take;
            bool pass = false;
            uint32_t rs1 = 0, ii = 0;
            if ((uint32_t)lane < take) {
                rs1 = S.qa_rs[base + lane];
                const uint32_t g = S.qa_g[base + lane];
                if (A.tfrags) { ii = A.tfrags[g]; rs1 = (rs1 & 0xFFFF0000u) | A.tslot[g]; }   // slot in the full list
                else ii = A.frags[g];                                                        // (range index == slot)
                const uint32_t rr = LVX_RS_RAY(rs1), mm = LVX_RS_ORD(rs1);
                pass = !surely_misses_f32(S.pf[mm][0][rr], S.pf[mm][1][rr], S.pf[mm][2][rr], S.hf[mm][rr], S.dirf[0][rr],
                                          S.dirf[1][rr], S.dirf[2][rr], A.verts_f, (int64_t)ii, R2f);
            }
            qa = base;
            const uint32_t mb = __ballot_sync(LVX_FULL, pass);
            if (pass) {
                const uint32_t pos = qb + __popc(mb & lt_mask);
                S.qb_rs[pos] = rs1; S.qb_i[pos] = ii;
            }
            qb += __popc(mb);
#if LVX_COUNT != 2
            LVX_CNT(14, __popc(mb));
#endif
            __syncwarp();
            continue;
        }
        // ---- stage A: every lane walks its own ranges (ordinal after ordinal); in each step all
        // lanes that still have an entry push one pair.  A lane whose range is used up moves on to
        // its next ordinal in the same step, so the loop runs max-over-lanes(sum of range lengths)
        // times, not sum-over-ordinals(max-over-lanes).
        bool fin;
        do {    // (tight loop: this is the most frequent step of the whole kernel)
            if (left == 0 && m < n_ord) {
                m++;
                if (m > last_ord()) m = n_ord;          // a hit in an earlier voxel: the later ones cannot matter
                if (m < n_ord) {
                    g = S.fo[m][lane]; left = S.tn[m][lane]; idx = 0;
                    tag = ((uint32_t)m << 21) | ((uint32_t)lane << 16);
                }
            }
            const uint32_t ma = __ballot_sync(LVX_FULL, left != 0);
            if (left) {
                const uint32_t pos = qa + __popc(ma & lt_mask);
                S.qa_rs[pos] = tag | idx; S.qa_g[pos] = g;
                g++; idx++; left--;
            }
            qa += __popc(ma);
#if LVX_COUNT != 2
            LVX_CNT(13, __popc(ma));
#endif
            __syncwarp();
            fin = __ballot_sync(LVX_FULL, m < n_ord) == 0;
        } while (!fin && qa < 32);
        if (fin) a_done = true;
    }
}

// lv/raytracer.py:414-423 + 272-291: the pixel's ray and its parameter range inside the grid
__device__ __forceinline__ bool setup_ray(const RenderArgs &A, int px, int py, double &dx, double &dy, double &dz,
                                          double &t, double &t1) {
    const int w = A.cam.width, h = A.cam.height, res = A.res;
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
    const double o[3] = {A.cam.pos[0], A.cam.pos[1], A.cam.pos[2]}, d[3] = {dx, dy, dz};
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
    t = t0 > 0.0 ? t0 : 0.0;
    return t1 >= t0;
}

// One DDA step of lv/raytracer.py:475-482 / 542-556 from parameter `tcur`.  Returns 0 when the
// ray has left the grid, 1 after skipping an empty node, 2 after recording an occupied voxel as
// ordinal `m` of this lane (tent = its entry parameter, te = its exit parameter).  In both of the
// latter cases tcur has advanced to where the ray goes on (lv/raytracer.py:506-509).
template <int M>
__device__ __forceinline__ int dda_step(const RenderArgs &A, PairQueues<M> &S, int lane, int m, double ox, double oy,
                                        double oz, double dx, double dy, double dz, const RayInv &inv, double t1,
                                        double &tcur, double &tent, double &te) {
    const int res = A.res;
    if (!(tcur < t1)) return 0;
    const double tm = tcur + 1e-6;
    const int x = (int)floor(ox + dx * tm), y = (int)floor(oy + dy * tm), z = (int)floor(oz + dz * tm);
    if (x < 0 || y < 0 || z < 0 || x >= res || y >= res || z >= res) return 0;
    const uint32_t idx = (uint32_t)x + (uint32_t)res * ((uint32_t)y + (uint32_t)res * (uint32_t)z);   // res <= 1024
    // the list bounds are fetched together with the march byte (independent loads, one round
    // trip); they are only used when the voxel turns out to be occupied
    const int lv = A.march[idx];
    const uint32_t fo = A.offsets[idx], fe = A.offsets[idx + 1];
    const uint32_t tn = A.tcnt ? A.tcnt[idx] : 0u;
    const bool occ = lv == 255;
    const double tx = voxel_exit(ox, oy, oz, dx, dy, dz, inv, x, y, z, occ ? 0 : lv);
    if (occ) {
        S.fo[m][lane] = fo;
        S.n[m][lane] = fe - fo;
        S.tn[m][lane] = A.tcnt ? (uint16_t)tn : (uint16_t)min(fe - fo, 0xFFFFu);
        S.vox[m][0][lane] = (int16_t)x; S.vox[m][1][lane] = (int16_t)y; S.vox[m][2][lane] = (int16_t)z;
        tent = tcur;
        te = tx;
        const double tc = 0.5 * (tcur + tx);     // a point of the ray inside the voxel
        S.pf[m][0][lane] = (float)(ox + dx * tc); S.pf[m][1][lane] = (float)(oy + dy * tc); S.pf[m][2][lane] = (float)(oz + dz * tc);
        S.hf[m][lane] = (float)(0.5 * (tx - tcur)) + 1e-3f;
    }
    tcur = tx > tcur ? tx : tcur + 1e-6;
    return occ ? 2 : 1;
}

// ----------------------------------------------------------------------------- ray supply
// The trace kernels are persistent: a warp draws 8x4 pixel tiles from a global counter and hands
// their pixels to lanes whose ray has finished, so that a warp does not march on with a handful of
// live rays (ncu before: 10-15 of 32 threads active in the DDA and intersection code).  A fresh
// warp takes a whole tile, lane k = pixel k of the tile; later refills fill idle lanes with the
// next pixels of the warp's current tile.
#ifndef LVX_REFILL
#define LVX_REFILL 32     // idle lanes that trigger a refill (measured on C2/C3: 4, 8 and 16 are slower than
                          // waiting for the whole tile -- mixing rays of different tiles in a warp costs
                          // more in lost voxel/segment reuse than the idle lanes do)
#endif
struct TileQueue {
    uint32_t pend_tile, pend_mask;   // warp-uniform: tile being handed out, its pixels not yet assigned
    uint32_t n_tiles, tiles_x;
    bool more;                       // the global counter has not run out yet
};
__device__ __forceinline__ TileQueue make_tile_queue(const RenderArgs &A) {
    const uint32_t tx = (uint32_t)(A.p.tile_x1 - A.p.tile_x0 + 7) / 8, ty = (uint32_t)(A.p.tile_y1 - A.p.tile_y0 + 3) / 4;
    return TileQueue{0u, 0u, tx * ty, tx, true};
}
// Called by the whole warp.  Lanes with has == false may receive a pixel: returns true and sets px, py.
__device__ __forceinline__ bool assign_pixels(const RenderArgs &A, TileQueue &Q, bool has, int lane, int &px, int &py) {
    const uint32_t lt_mask = (1u << lane) - 1u;
    bool got = false;
    for (;;) {
        const uint32_t idle = __ballot_sync(LVX_FULL, !has && !got);
        if (idle == 0) break;
        if (Q.pend_mask == 0) {
            if (!Q.more) break;
            unsigned long long tile = 0;
            if (lane == 0) tile = atomicAdd((unsigned long long *)&A.stats[LVX_ST_TILE_CURSOR], 1ull);
            tile = __shfl_sync(LVX_FULL, tile, 0);
            if (tile >= (unsigned long long)Q.n_tiles) { Q.more = false; break; }
            Q.pend_tile = (uint32_t)tile;
            Q.pend_mask = 0xffffffffu;
        }
        const uint32_t n_take = min(__popc(idle), __popc(Q.pend_mask));
        const uint32_t rank = __popc(idle & lt_mask);
        uint32_t mybit = 0;
        if (!has && !got && rank < n_take) {
            const uint32_t bit = __fns(Q.pend_mask, 0, (int)rank + 1);
            px = A.p.tile_x0 + (int)(Q.pend_tile % Q.tiles_x) * 8 + (int)(bit & 7u);
            py = A.p.tile_y0 + (int)(Q.pend_tile / Q.tiles_x) * 4 + (int)(bit >> 3);
            got = true;
            mybit = 1u << bit;
        }
        Q.pend_mask &= ~__reduce_or_sync(LVX_FULL, mybit);
    }
    return got;
}

// ----------------------------------------------------------------------------- opaque
struct WarpShared {
    PairQueues<LVX_SPEC> q;
    double hit_t[32];
    uint32_t hit_rs[32], hit_i[32];
};

#ifndef LVX_RC_MINB
#define LVX_RC_MINB 5   // 96 registers, no spills (6 CTAs/SM = 80 registers spills in the march loop: 2.39 vs 2.20 ms)
#endif
template <bool DEFER>
__global__ void __launch_bounds__(RC_WARPS * 32, LVX_RC_MINB)
k_render_opaque_coop(const RenderArgs A) {
    constexpr int M = LVX_SPEC;
    __shared__ __align__(16) unsigned char smem_raw[sizeof(WarpShared) * RC_WARPS];
    uint32_t lane_u = threadIdx.x & 31u, soff = (threadIdx.x >> 5) * (uint32_t)sizeof(WarpShared);
    LVX_PIN(lane_u); LVX_PIN(soff);
    const int lane = (int)lane_u;
    WarpShared &S = *reinterpret_cast<WarpShared *>(smem_raw + soff);
    uint32_t lt_mask = (1u << lane_u) - 1u;
    LVX_PIN(lt_mask);
    const int w = A.cam.width, res = A.res;
    const double ox = A.cam.pos[0], oy = A.cam.pos[1], oz = A.cam.pos[2];
    const bool clip = A.p.use_clip != 0;
    const double r = A.p.radius;
    const float R2f = ((float)r + 2e-3f) * ((float)r + 2e-3f);
    TileQueue Q = make_tile_queue(A);
    bool has = false, active = false;     // this lane holds a pixel / its ray is still marching
    int px = 0, py = 0;
    double dx = 0.0, dy = 0.0, dz = 1.0, t = 0.0, t1 = -1.0;
    RayInv inv{0.0, 0.0, 0.0, false};
    double best_t = -1.0;      // final hit of this lane's ray
    int64_t best_i = -1;
    uint64_t n_tests = 0;

    for (;;) {
        uint32_t am = __ballot_sync(LVX_FULL, active);
        if (__popc(am) <= 32 - LVX_REFILL) {
            // ---- 0. retire finished rays, hand new pixels to the idle lanes
            const bool done = has && !active;
            if (__ballot_sync(LVX_FULL, done)) {
                if (!DEFER) {
                    if (done) {
                        double out_r = A.p.background[0], out_g = A.p.background[1], out_b = A.p.background[2];
                        int32_t out_id = -1;
                        if (best_t >= 0.0) {
                            const rgb3 c = shade_hit_inl(make_shade_ctx(A), best_i, ox + dx * best_t, oy + dy * best_t, oz + dz * best_t);
                            out_r = c.r; out_g = c.g; out_b = c.b;
                            out_id = (int32_t)best_i;
                        }
                        const int64_t pix = (int64_t)py * w + px;
                        if (A.rgb) { A.rgb[3 * pix] = out_r; A.rgb[3 * pix + 1] = out_g; A.rgb[3 * pix + 2] = out_b; }
                        if (A.srgb) { A.srgb[3 * pix] = to_srgb8(out_r); A.srgb[3 * pix + 1] = to_srgb8(out_g); A.srgb[3 * pix + 2] = to_srgb8(out_b); }
                        A.hit_id[pix] = out_id;
                    }
                } else {
                    // Shading on demand: record the hit, and request AO/shadow for the (visible) voxels
                    // its trilinear lookup will read (lv/raytracer.py:368-390).  The request is a bit
                    // per voxel set with a fire-and-forget atomic; k_need_list compacts the bits into
                    // the list the cone tracer walks.
                    if (done) {
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
                                if (A.march[idx] == 255) atomicOr(&A.need_bits[idx >> 5], 1u << (idx & 31));
                            }
                        }
                    }
                }
                if (done) has = false;
            }
            if (assign_pixels(A, Q, has, lane, px, py)) {
                has = px < A.p.tile_x1 && py < A.p.tile_y1;     // pixels of a partial tile beyond the rect
                best_t = -1.0; best_i = -1;
                active = has && setup_ray(A, px, py, dx, dy, dz, t, t1);
                S.q.dir[0][lane] = dx; S.q.dir[1][lane] = dy; S.q.dir[2][lane] = dz;
                S.q.dirf[0][lane] = (float)dx; S.q.dirf[1][lane] = (float)dy; S.q.dirf[2][lane] = (float)dz;
                inv = make_inv(dx, dy, dz);
            }
            __syncwarp();
            am = __ballot_sync(LVX_FULL, active);
            if (am == 0) {
                if (!Q.more && Q.pend_mask == 0 && __ballot_sync(LVX_FULL, has) == 0) break;
                continue;
            }
        }
        // ---- 1. record the next Mr occupied voxels (lv/raytracer.py:475-482, 506-509); every lane
        // steps its own DDA until it has Mr of them or leaves the grid
        constexpr int Mr = M;
        bool leaving = false, go = active;
        int n_vox = 0;
        double tcur = t;
#if defined(LVX_COUNT) && LVX_COUNT == 2
        { const uint32_t al = __popc(am); LVX_CNT(13, 1); LVX_CNT(14, al); }
#endif
        while (__any_sync(LVX_FULL, go)) {
#if defined(LVX_COUNT) && LVX_COUNT == 2
            { const uint32_t gl = __popc(__ballot_sync(LVX_FULL, go)); LVX_CNT(15, 1); LVX_CNT(11, gl); }
#endif
            if (go) {
                double tent, te;
                const int st = dda_step<M>(A, S.q, lane, n_vox, ox, oy, oz, dx, dy, dz, inv, t1, tcur, tent, te);
                if (st == 0) { leaving = true; go = false; }
                else if (st == 2 && ++n_vox == Mr) go = false;
            }
        }
#pragma unroll 1
        for (int m = n_vox; m < Mr; m++) { S.q.n[m][lane] = 0; S.q.tn[m][lane] = 0; }
        __syncwarp();
        // best hit of this lane's ray in this round: lowest ordinal, then min t, then lowest slot
        double cur_t = -1.0;
        uint32_t cur_ms = 0xffffffffu, cur_i = 0;      // (ordinal << 16) | slot
        run_pairs<M>(A, S.q, Mr, lane, lt_mask, R2f, [&](bool valid, uint32_t rs, uint32_t ii, bool, int sub) {
            bool hit = false;
            double ht = -1.0;
            const uint32_t hr = LVX_RS_RAY(rs), hm_ = LVX_RS_ORD(rs);
            double ddx = 0.0, ddy = 0.0, ddz = 1.0;
            if (valid) {
                ddx = S.q.dir[0][hr]; ddy = S.q.dir[1][hr]; ddz = S.q.dir[2][hr];
                const Capsule c = load_capsule(A.verts, A.normals, (int64_t)ii, r, clip);
                ht = ray_capsule(ox, oy, oz, ddx, ddy, ddz, c, sub);
            }
            if (sub >= 0) {     // two lanes per pair: the smaller admissible t of the two halves, kept on the even lane
                const double other = __shfl_xor_sync(LVX_FULL, ht, 1);
                ht = ht < 0.0 ? other : (other < 0.0 ? ht : fmin(ht, other));
                if (lane & 1) valid = false;
            }
            if (valid) {
                if (ht >= 0.0) {   // lv/raytracer.py:446-452: the hit must lie in the voxel being visited
                    const int hx = (int)floor(ox + ddx * ht), hy = (int)floor(oy + ddy * ht), hz = (int)floor(oz + ddz * ht);
                    hit = hx == S.q.vox[hm_][0][hr] && hy == S.q.vox[hm_][1][hr] && hz == S.q.vox[hm_][2][hr];
                }
            }
            // fold hits on the owning lanes (lv/raytracer.py:453: min t, first slot wins ties)
            uint32_t hm = __ballot_sync(LVX_FULL, hit);
            if (hm == 0) return;
            if (hit) { S.hit_t[lane] = ht; S.hit_rs[lane] = rs; S.hit_i[lane] = ii; }
            __syncwarp();
            while (hm) {
                const int src = __ffs(hm) - 1;
                hm &= hm - 1;
                const uint32_t rs2 = S.hit_rs[src];
                if ((uint32_t)lane == LVX_RS_RAY(rs2)) {
                    const double tt = S.hit_t[src];
                    const uint32_t ms2 = (LVX_RS_ORD(rs2) << 16) | LVX_RS_SLOT(rs2);
                    const uint32_t o2 = ms2 >> 16, oc = cur_ms >> 16;
                    if (cur_t < 0.0 || o2 < oc || (o2 == oc && (tt < cur_t || (tt == cur_t && ms2 < cur_ms)))) {
                        cur_t = tt; cur_ms = ms2; cur_i = S.hit_i[src];
                    }
                }
            }
            __syncwarp();
        }, [&]() { return cur_t >= 0.0 ? (int)(cur_ms >> 16) : Mr - 1; });
        if (active) {
            // tests the reference would have run: every voxel up to and including the one with the hit
            const int m_end = cur_t >= 0.0 ? (int)(cur_ms >> 16) : Mr - 1;
            uint32_t cnt = 0;
#pragma unroll 1
            for (int m = 0; m <= m_end; m++) cnt += S.q.n[m][lane];
            n_tests += cnt;
            if (cur_t >= 0.0) { best_t = cur_t; best_i = cur_i; active = false; }
            else if (leaving) active = false;
            else t = tcur;
        }
        __syncwarp();
    }
    n_tests = warp_sum_u64(n_tests);
    if (lane == 0 && n_tests)
        atomicAdd((unsigned long long *)&A.stats[LVX_ST_RAY_TESTS], (unsigned long long)n_tests);
}

// ----------------------------------------------------------------------------- transparent
// Same work sharing for lv/raytracer.py:518-645.  In-voxel hits become (ordinal, key = depth16 <<
// 16 | slot, t, segment) records in a per-warp list, which the owning lanes drain into their
// private k-slot buffers (one per ordinal).  The k smallest keys above `last_key` are a set, so
// the insertion order does not matter (keys are unique: the slot is in the low bits) and the
// reference's result is reproduced exactly, including the re-scan of a voxel when more than k
// hits were accepted: the ray then starts its next round in that same voxel with `last_key` set
// (and its tests are counted again like the reference does).
//
// Deferred shading.  Control flow only needs the accumulated alpha, which depends on the NUMBER
// of blended hits (A += (1-A)*alpha), not on their colour.  So the blend step just fixes each
// hit's weight w = (1-A)*alpha and appends (ray, w, t, segment) to a per-warp FIFO; whenever 32
// entries are queued their normals, AO/shadow lookups and colours are evaluated on all 32 lanes
// at once and the owning lanes add w*colour in FIFO order -- per ray that is the reference's
// order of additions, so the f64 sums keep their bits.
#ifndef LVX_HL_CAP
#define LVX_HL_CAP 96
#endif
constexpr int HL_CAP = LVX_HL_CAP;   // >= 64: a batch of 32 hits must fit on top of 32 undrained ones
constexpr int KMAX = 64;        // lv/raytracer.py:64: k <= 64

struct WarpSharedT {
    PairQueues<LVX_SPEC_T> q;
    double t_enter[LVX_SPEC_T][32], inv_span[LVX_SPEC_T][32], t_exit[LVX_SPEC_T][32];
    double hl_t[HL_CAP];
    uint32_t hl_key[HL_CAP], hl_i[HL_CAP];
    uint8_t hl_r[HL_CAP];           // ordinal << 5 | ray
    uint32_t own[32];               // drain: per ray, the records it owns in the current chunk
    double d_w[64], d_t[64];        // deferred shading FIFO
    uint32_t d_i[64], d_ray[64];
    double d_c[3][32];              // w * colour of the batch being folded
};

#ifndef LVX_RT_MINB
#define LVX_RT_MINB 4
#endif
__global__ void __launch_bounds__(RC_WARPS * 32, LVX_RT_MINB)
k_render_transparent_coop(const RenderArgs A) {
    constexpr int M = LVX_SPEC_T;
    extern __shared__ __align__(16) unsigned char smem_raw[];      // RC_WARPS x WarpSharedT + ShadeCtx (> 48 KB: opt-in)
    ShadeCtx *ctx = reinterpret_cast<ShadeCtx *>(smem_raw + sizeof(WarpSharedT) * RC_WARPS);
    uint32_t lane_u = threadIdx.x & 31u, soff = (threadIdx.x >> 5) * (uint32_t)sizeof(WarpSharedT);
    LVX_PIN(lane_u); LVX_PIN(soff);
    const int lane = (int)lane_u;
    WarpSharedT &S = *reinterpret_cast<WarpSharedT *>(smem_raw + soff);
    if (threadIdx.x == 0) *ctx = make_shade_ctx(A);
    __syncthreads();
    const int w = A.cam.width;
    const double ox = A.cam.pos[0], oy = A.cam.pos[1], oz = A.cam.pos[2];
    const bool clip = A.p.use_clip != 0;
    const double r = A.p.radius;
    const int kslots = A.p.k;
    const bool early = A.p.early_termination != 0;
    const double alpha = A.p.alpha;
    uint32_t lt_mask = (1u << lane_u) - 1u;
    LVX_PIN(lt_mask);
    const float R2f = ((float)r + 2e-3f) * ((float)r + 2e-3f);
    TileQueue Q = make_tile_queue(A);
    bool has = false, active = false;
    int px = 0, py = 0;
    double dx = 0.0, dy = 0.0, dz = 1.0, t = 0.0, t1 = -1.0;
    RayInv inv{0.0, 0.0, 0.0, false};
    double col_r = 0.0, col_g = 0.0, col_b = 0.0, acc_a = 0.0;
    int64_t first_hit = -1;
    // k-slot buffers, one per ordinal, packed with stride k (local memory)
    uint32_t keybuf[M * KMAX], ibuf[M * KMAX];
    double tbuf[M * KMAX];
    int kept[M];
    uint32_t accepted[M];
    uint64_t n_tests = 0;
    uint32_t qd = 0;           // entries in the deferred shading FIFO
    int repeat_m = -1;         // >= 0: the ray re-scans the voxel recorded as that ordinal last round
    int64_t last_key = -1;     // ... accepting only keys above last_key (applies to ordinal 0 of the new round)

    // shades the first min(qd, 32) FIFO entries and folds w*colour into the owners' sums
    auto shade_batch = [&]() {
        const uint32_t take = qd < 32 ? qd : 32;
        if ((uint32_t)lane < take) {
            const uint32_t rr = S.d_ray[lane];
            const double tt = S.d_t[lane], wgt = S.d_w[lane];
            const double ddx = S.q.dir[0][rr], ddy = S.q.dir[1][rr], ddz = S.q.dir[2][rr];
            // lv/raytracer.py:612-620
            const rgb3 c = shade_hit(ctx, (int64_t)S.d_i[lane], ox + ddx * tt, oy + ddy * tt, oz + ddz * tt);
            S.d_c[0][lane] = wgt * c.r; S.d_c[1][lane] = wgt * c.g; S.d_c[2][lane] = wgt * c.b;
        }
        __syncwarp();
#pragma unroll 1
        for (uint32_t e = 0; e < take; e++)
            if (S.d_ray[e] == (uint32_t)lane) { col_r += S.d_c[0][e]; col_g += S.d_c[1][e]; col_b += S.d_c[2][e]; }
        // move the tail (at most 31 entries) to the front
        const bool mv = (uint32_t)lane + 32 < qd;
        double mw = 0.0, mt = 0.0;
        uint32_t mi = 0, mr = 0;
        if (mv) { mw = S.d_w[lane + 32]; mt = S.d_t[lane + 32]; mi = S.d_i[lane + 32]; mr = S.d_ray[lane + 32]; }
        __syncwarp();
        if (mv) { S.d_w[lane] = mw; S.d_t[lane] = mt; S.d_i[lane] = mi; S.d_ray[lane] = mr; }
        qd -= take;
        __syncwarp();
    };

    for (;;) {
        uint32_t am = __ballot_sync(LVX_FULL, active);
        if (__popc(am) <= 32 - LVX_REFILL) {
            // ---- 0. retire finished rays (their queued colours first), hand new pixels to idle lanes
            const bool done = has && !active;
            if (__ballot_sync(LVX_FULL, done)) {
                while (qd > 0) shade_batch();
                if (done) {
                    const double out_r = col_r + (1.0 - acc_a) * A.p.background[0];
                    const double out_g = col_g + (1.0 - acc_a) * A.p.background[1];
                    const double out_b = col_b + (1.0 - acc_a) * A.p.background[2];
                    const int64_t pix = (int64_t)py * w + px;
                    if (A.rgb) { A.rgb[3 * pix] = out_r; A.rgb[3 * pix + 1] = out_g; A.rgb[3 * pix + 2] = out_b; }
                    if (A.srgb) { A.srgb[3 * pix] = to_srgb8(out_r); A.srgb[3 * pix + 1] = to_srgb8(out_g); A.srgb[3 * pix + 2] = to_srgb8(out_b); }
                    A.hit_id[pix] = (int32_t)first_hit;
                    has = false;
                }
            }
            if (assign_pixels(A, Q, has, lane, px, py)) {
                has = px < A.p.tile_x1 && py < A.p.tile_y1;
                col_r = col_g = col_b = acc_a = 0.0;
                first_hit = -1; repeat_m = -1; last_key = -1;
                active = has && setup_ray(A, px, py, dx, dy, dz, t, t1);
                S.q.dir[0][lane] = dx; S.q.dir[1][lane] = dy; S.q.dir[2][lane] = dz;
                S.q.dirf[0][lane] = (float)dx; S.q.dirf[1][lane] = (float)dy; S.q.dirf[2][lane] = (float)dz;
                inv = make_inv(dx, dy, dz);
            }
            __syncwarp();
            am = __ballot_sync(LVX_FULL, active);
            if (am == 0) {
                if (!Q.more && Q.pend_mask == 0 && __ballot_sync(LVX_FULL, has) == 0) break;
                continue;
            }
        }
        // ---- 1. record the next M occupied voxels; a re-scan keeps its voxel as ordinal 0
        bool go = active;
        int n_vox = 0;                                         // ordinals recorded by this lane
        double tcur = t;
        const int64_t lk0 = repeat_m >= 0 ? last_key : -1;     // key floor of ordinal 0
        if (active && repeat_m >= 0) {
            const int s = repeat_m;                            // own column only: no other lane reads it yet
            S.q.fo[0][lane] = S.q.fo[s][lane]; S.q.n[0][lane] = S.q.n[s][lane]; S.q.tn[0][lane] = S.q.tn[s][lane];
#pragma unroll
            for (int a = 0; a < 3; a++) { S.q.vox[0][a][lane] = S.q.vox[s][a][lane]; S.q.pf[0][a][lane] = S.q.pf[s][a][lane]; }
            S.q.hf[0][lane] = S.q.hf[s][lane];
            const double te = S.t_exit[s][lane];               // tcur == t == that voxel's entry parameter
            const double span = te - tcur;
            S.t_enter[0][lane] = tcur; S.t_exit[0][lane] = te;
            S.inv_span[0][lane] = span > 0.0 ? 65535.0 / span : 0.0;
            tcur = te > tcur ? te : tcur + 1e-6;
            n_vox = 1;
            if (M == 1) go = false;
        }
        repeat_m = -1;
#if defined(LVX_COUNT) && LVX_COUNT == 2
        { const uint32_t al = __popc(am); LVX_CNT(13, 1); LVX_CNT(14, al); }
#endif
        while (__any_sync(LVX_FULL, go)) {
#if defined(LVX_COUNT) && LVX_COUNT == 2
            { const uint32_t gl = __popc(__ballot_sync(LVX_FULL, go)); LVX_CNT(15, 1); LVX_CNT(11, gl); }
#endif
            if (go) {
                // lv/raytracer.py:543-544: the alpha cut-off is re-checked at apply time, per ordinal
                double tent, te;
                const int st = dda_step<M>(A, S.q, lane, n_vox, ox, oy, oz, dx, dy, dz, inv, t1, tcur, tent, te);
                if (st == 0) go = false;
                else if (st == 2) {
                    const double span = te - tent;             // t_enter = the previous exit (lv/raytracer.py:557-560)
                    S.t_enter[n_vox][lane] = tent; S.t_exit[n_vox][lane] = te;
                    S.inv_span[n_vox][lane] = span > 0.0 ? 65535.0 / span : 0.0;
                    if (++n_vox == M) go = false;
                }
            }
        }
#pragma unroll 1
        for (int m = 0; m < M; m++) {
            if (m >= n_vox) { S.q.n[m][lane] = 0; S.q.tn[m][lane] = 0; }
            kept[m] = 0; accepted[m] = 0;
        }
        __syncwarp();
        uint32_t hl_n = 0;

        // owners pull their records out of the hit list (insertion sort, lv/raytracer.py:589-607)
        auto drain = [&]() {
            for (uint32_t c0 = 0; c0 < hl_n; c0 += 32) {
                // lane e looks at record c0+e; all records of one ray are matched into a bit mask
                // that the ray's own lane picks up from shared memory
                const bool have = c0 + lane < hl_n;
                const uint32_t tag_e = have ? S.hl_r[c0 + lane] : 0xffu;
                const uint32_t same = __match_any_sync(LVX_FULL, have ? (tag_e & 31u) : 32u + (uint32_t)lane);
                S.own[lane] = 0;
                __syncwarp();
                if (have) S.own[tag_e & 31u] = same;          // every writer of a slot writes the same mask
                __syncwarp();
                uint32_t mine = S.own[lane];
                __syncwarp();
                while (mine) {
                    const uint32_t e = c0 + (uint32_t)(__ffs(mine) - 1);
                    mine &= mine - 1;
                    const int m = (int)(S.hl_r[e] >> 5);
                    const uint32_t key = S.hl_key[e];
                    if (m == 0 && (int64_t)key <= lk0) continue;
                    accepted[m]++;
                    uint32_t *kb = keybuf + m * kslots, *ib = ibuf + m * kslots;
                    double *tb = tbuf + m * kslots;
                    int j;
                    if (kept[m] < kslots) { j = kept[m]; kept[m]++; }
                    else if (key < kb[kslots - 1]) j = kslots - 1;
                    else continue;
                    while (j > 0 && kb[j - 1] > key) {
                        kb[j] = kb[j - 1]; tb[j] = tb[j - 1]; ib[j] = ib[j - 1];
                        j--;
                    }
                    kb[j] = key; tb[j] = S.hl_t[e]; ib[j] = S.hl_i[e];
                }
            }
            hl_n = 0;
            __syncwarp();
        };

        run_pairs<M>(A, S.q, M, lane, lt_mask, R2f, [&](bool valid, uint32_t rs, uint32_t ii, bool fin, int sub) {
            bool hit = false;
            uint32_t hkey = 0;
            double ht = -1.0;
            const uint32_t hr = LVX_RS_RAY(rs), hm_ = LVX_RS_ORD(rs);
            double ddx = 0.0, ddy = 0.0, ddz = 1.0;
            if (valid) {
                ddx = S.q.dir[0][hr]; ddy = S.q.dir[1][hr]; ddz = S.q.dir[2][hr];
                const Capsule c = load_capsule(A.verts, A.normals, (int64_t)ii, r, clip);
                ht = ray_capsule(ox, oy, oz, ddx, ddy, ddz, c, sub);
            }
            if (sub >= 0) {     // two lanes per pair (see run_pairs): merge, keep the even lane
                const double other = __shfl_xor_sync(LVX_FULL, ht, 1);
                ht = ht < 0.0 ? other : (other < 0.0 ? ht : fmin(ht, other));
                if (lane & 1) valid = false;
            }
            if (valid) {
                if (ht >= 0.0) {
                    const int hx = (int)floor(ox + ddx * ht), hy = (int)floor(oy + ddy * ht), hz = (int)floor(oz + ddz * ht);
                    hit = hx == S.q.vox[hm_][0][hr] && hy == S.q.vox[hm_][1][hr] && hz == S.q.vox[hm_][2][hr];
                    if (hit) {   // lv/raytracer.py:583-588
                        int64_t q = (int64_t)((ht - S.t_enter[hm_][hr]) * S.inv_span[hm_][hr]);
                        if (q < 0) q = 0; else if (q > 65535) q = 65535;
                        hkey = ((uint32_t)q << 16) | LVX_RS_SLOT(rs);
                    }
                }
            }
            const uint32_t hm = __ballot_sync(LVX_FULL, hit);
            if (hit) {      // the list has room for 32 more records at this point
                const uint32_t pos = hl_n + __popc(hm & lt_mask);
                S.hl_t[pos] = ht; S.hl_key[pos] = hkey; S.hl_i[pos] = ii; S.hl_r[pos] = (uint8_t)((hm_ << 5) | hr);
            }
            hl_n += __popc(hm);
#if LVX_COUNT != 2
            LVX_CNT(15, __popc(hm));
#endif
            __syncwarp();
            if (hl_n + 32 > HL_CAP || fin) drain();
        }, [&]() { return M - 1; });
        // ---- consume the ordinals in order (lv/raytracer.py:543-544, 608-637): fix the blend
        // weights now, queue the colours
        bool going = active;       // false once this lane's ray has stopped consuming this round
#pragma unroll 1
        for (int m = 0; m < M; m++) {
            // a ray consumes ordinal m if it is still going, has not reached the alpha cut-off
            // (checked before every voxel, lv/raytracer.py:543-544) and has such a voxel
            bool use = going;
            if (use && early && acc_a >= 0.999) { use = false; going = false; active = false; }
            if (use && m >= n_vox) { use = false; going = false; active = false; }   // left the grid
            if (use) n_tests += S.q.n[m][lane];
            const int km = use ? kept[m] : 0;
            const int kmax = __reduce_max_sync(LVX_FULL, km);
            bool stopped = !use;
            const uint32_t *ib = ibuf + m * kslots;
            const double *tb = tbuf + m * kslots;
            for (int j = 0; j < kmax; j++) {
                if (!stopped && (j >= km || (early && acc_a >= 0.999))) stopped = true;
                double wgt = 0.0;
                if (!stopped) {
                    wgt = (1.0 - acc_a) * alpha;
                    acc_a += wgt;
                    if (first_hit < 0) first_hit = ib[j];
                }
                const uint32_t pm = __ballot_sync(LVX_FULL, !stopped);
                if (pm == 0) break;
                if (!stopped) {
                    const uint32_t pos = qd + __popc(pm & lt_mask);
                    S.d_w[pos] = wgt; S.d_t[pos] = tb[j]; S.d_i[pos] = ib[j]; S.d_ray[pos] = (uint32_t)lane;
                }
                qd += __popc(pm);
                __syncwarp();
                if (qd >= 32) shade_batch();
            }
            if (use) {
                // lv/raytracer.py:632-637
                if (accepted[m] <= (uint32_t)kslots || (early && acc_a >= 0.999)) {
                    const double t_in = S.t_enter[m][lane], t_out = S.t_exit[m][lane];
                    t = t_out > t_in ? t_out : t_in + 1e-6;      // on to the next voxel
                } else {
                    last_key = keybuf[m * kslots + kslots - 1];  // stay: re-scan this voxel next round
                    repeat_m = m;
                    t = S.t_enter[m][lane];
                    going = false;
                }
            }
        }
        if (active && early && acc_a >= 0.999) active = false;   // lv/raytracer.py:543-544
        __syncwarp();
    }
    n_tests = warp_sum_u64(n_tests);
    if (lane == 0 && n_tests)
        atomicAdd((unsigned long long *)&A.stats[LVX_ST_RAY_TESTS], (unsigned long long)n_tests);
#if defined(LVX_COUNT) && LVX_COUNT == 3
    if (threadIdx.x == 0) A.stats[13] = g_dbg_unique;     // (monotone: the last block to finish leaves the total)
#endif
}

// Requested voxels (one bit each) -> list, ascending inside every block's chunk: block scan of the
// per-thread popcounts, one atomic on the list counter per block.
__global__ void __launch_bounds__(256)
k_need_list(const uint32_t *__restrict__ need_bits, int64_t n_words, uint32_t *__restrict__ need_list) {
    __shared__ uint32_t s_warp[8];
    __shared__ unsigned long long s_base;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t m = i < n_words ? need_bits[i] : 0u;
    const uint32_t c = __popc(m);
    uint32_t inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(LVX_FULL, inc, o);
        if (lane >= o) inc += v;
    }
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        const uint32_t wv = lane < 8 ? s_warp[lane] : 0;
        uint32_t wi = wv;
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
            const uint32_t v = __shfl_up_sync(LVX_FULL, wi, o);
            if (lane >= o) wi += v;
        }
        if (lane < 8) s_warp[lane] = wi - wv;
        if (lane == 7 && wi) s_base = atomicAdd(reinterpret_cast<unsigned long long *>(need_list), (unsigned long long)wi);
    }
    __syncthreads();
    if (c) {
        uint64_t slot = LVX_LIST_HDR + s_base + s_warp[warp] + (inc - c);
        while (m) {
            const int bit = __ffs(m) - 1;
            m &= m - 1;
            need_list[slot++] = (uint32_t)(i * 32 + bit);
        }
    }
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
        const rgb3 c = shade_hit_inl(make_shade_ctx(A), (int64_t)A.hit_id[pix], hx, hy, hz);
        out_r = c.r; out_g = c.g; out_b = c.b;
    }
    if (A.rgb) { A.rgb[3 * pix] = out_r; A.rgb[3 * pix + 1] = out_g; A.rgb[3 * pix + 2] = out_b; }
    if (A.srgb) { A.srgb[3 * pix] = to_srgb8(out_r); A.srgb[3 * pix + 1] = to_srgb8(out_g); A.srgb[3 * pix + 2] = to_srgb8(out_b); }
}

}  // namespace lvx

using namespace lvx;

// persistent launch: one warp per 8x4 pixel tile at most, otherwise every SM filled to its occupancy
static unsigned persistent_grid(int tw, int th, int blocks_per_sm) {
    static int n_sm = 0;
    if (!n_sm) {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n_sm <= 0)
            n_sm = 148;
    }
    const int64_t tiles = (int64_t)((tw + 7) / 8) * ((th + 3) / 4);
#ifdef LVX_GRID_CAP
    if (blocks_per_sm > LVX_GRID_CAP) blocks_per_sm = LVX_GRID_CAP;
#endif
    const int64_t need = (tiles + RC_WARPS - 1) / RC_WARPS, fill = (int64_t)n_sm * (blocks_per_sm > 0 ? blocks_per_sm : 1);
    return (unsigned)(need < fill ? need : fill);
}

static int fill_args(RenderArgs &A, const double *verts, const float *verts_f, const double *normals, const uint32_t *offsets,
                     const uint32_t *frags, const uint32_t *tight_frags, const uint16_t *tight_slot, const uint16_t *tight_cnt,
                     const uint8_t *march, int res, const float *ao, const float *shadow,
                     const lvx_camera *cam_host, const lvx_render_params *params_host, double *rgb, uint8_t *srgb,
                     int32_t *hit_id, uint64_t *stats) {
    if (!pow2(res) || res > 1024 || !cam_host || !params_host || !hit_id || !march) return LVX_E_ARG;
    const lvx_render_params &p = *params_host;
    if (p.mode < 0 || p.mode > 1 || p.k < 1 || p.k > 64 || !(p.alpha > 0.0 && p.alpha <= 1.0)) return LVX_E_ARG;
    if (cam_host->width <= 0 || cam_host->height <= 0) return LVX_E_ARG;
    if (p.tile_x0 < 0 || p.tile_y0 < 0 || p.tile_x1 > cam_host->width || p.tile_y1 > cam_host->height) return LVX_E_ARG;
    if (p.use_clip && !normals) return LVX_E_ARG;
    A.verts = verts; A.verts_f = verts_f; A.normals = normals; A.offsets = offsets; A.frags = frags; A.march = march;
    if ((tight_frags != nullptr) != (tight_slot != nullptr) || (tight_frags != nullptr) != (tight_cnt != nullptr)) return LVX_E_ARG;
    A.tfrags = tight_frags; A.tslot = tight_slot; A.tcnt = tight_cnt;
    A.ao = ao; A.sh = shadow;
    A.res = res; A.cam = *cam_host; A.p = p;
    A.rgb = rgb; A.srgb = srgb; A.hit_id = hit_id; A.stats = stats;
    A.hit_t = nullptr; A.need_bits = nullptr; A.need_list = nullptr; A.guard_volumes = 0;
    return LVX_OK;
}

extern "C" {

int lvx_render(const double *verts, const float *verts_f, const double *normals, const uint32_t *offsets, const uint32_t *frags,
               const uint32_t *tight_frags, const uint16_t *tight_slot, const uint16_t *tight_cnt,
               const uint8_t *march, int res, const float *ao, const float *shadow,
               const lvx_camera *cam_host, const lvx_render_params *params_host, double *rgb, uint8_t *srgb,
               int32_t *hit_id, uint64_t *stats, void *stream) {
    RenderArgs A;
    const int rc = fill_args(A, verts, verts_f, normals, offsets, frags, tight_frags, tight_slot, tight_cnt, march, res, ao, shadow, cam_host, params_host,
                             rgb, srgb, hit_id, stats);
    if (rc != LVX_OK) return rc;
    if (!verts_f) return LVX_E_ARG;
    const int tw = A.p.tile_x1 - A.p.tile_x0, th = A.p.tile_y1 - A.p.tile_y0;
    if (tw <= 0 || th <= 0) return LVX_OK;
    if (!stats) return LVX_E_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    LVX_CUDA(cudaMemsetAsync(stats + LVX_ST_TILE_CURSOR, 0, 8, s));
    if (A.p.mode == 0) {
        static int per_sm = 0;
        if (!per_sm) LVX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_render_opaque_coop<false>, RC_WARPS * 32, 0));
        k_render_opaque_coop<false><<<persistent_grid(tw, th, per_sm), RC_WARPS * 32, 0, s>>>(A);
    } else {
        const size_t smem = sizeof(WarpSharedT) * RC_WARPS + sizeof(ShadeCtx);
        static int per_sm = 0;
        if (!per_sm) {
            LVX_CUDA(cudaFuncSetAttribute(k_render_transparent_coop, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            LVX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_render_transparent_coop, RC_WARPS * 32, smem));
        }
        k_render_transparent_coop<<<persistent_grid(tw, th, per_sm), RC_WARPS * 32, smem, s>>>(A);
    }
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

int lvx_trace_hits(const double *verts, const float *verts_f, const double *normals, const uint32_t *offsets, const uint32_t *frags,
                   const uint32_t *tight_frags, const uint16_t *tight_slot, const uint16_t *tight_cnt,
                   const uint8_t *march, int res, const lvx_camera *cam_host,
                   const lvx_render_params *params_host, double *hit_t, int32_t *hit_id, uint32_t *need_bits,
                   uint32_t *need_list, uint64_t *stats, void *stream) {
    RenderArgs A;
    const int rc = fill_args(A, verts, verts_f, normals, offsets, frags, tight_frags, tight_slot, tight_cnt, march, res, nullptr, nullptr, cam_host,
                             params_host, nullptr, nullptr, hit_id, stats);
    if (rc != LVX_OK) return rc;
    if (A.p.mode != 0 || !verts_f || !hit_t || !need_bits || !need_list) return LVX_E_ARG;
    const int tw = A.p.tile_x1 - A.p.tile_x0, th = A.p.tile_y1 - A.p.tile_y0;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t V = (int64_t)res * res * res;
    if (!stats) return LVX_E_ARG;
    LVX_CUDA(cudaMemsetAsync(need_bits, 0, (size_t)((V + 31) / 32) * 4, s));
    LVX_CUDA(cudaMemsetAsync(need_list, 0, 8, s));
    if (tw <= 0 || th <= 0) return LVX_OK;
    LVX_CUDA(cudaMemsetAsync(stats + LVX_ST_TILE_CURSOR, 0, 8, s));
    A.hit_t = hit_t; A.need_bits = need_bits; A.need_list = need_list;
    static int per_sm = 0;
    if (!per_sm) LVX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_render_opaque_coop<true>, RC_WARPS * 32, 0));
    k_render_opaque_coop<true><<<persistent_grid(tw, th, per_sm), RC_WARPS * 32, 0, s>>>(A);
    {
        const int64_t n_words = (V + 31) / 32;
        k_need_list<<<blocks_for(n_words, 256), 256, 0, s>>>(need_bits, n_words, need_list);
    }
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

int lvx_resolve(const double *verts, const double *normals, const uint8_t *march, int res, const float *ao,
                const float *shadow, const lvx_camera *cam_host, const lvx_render_params *params_host,
                const double *hit_t, const int32_t *hit_id, double *rgb, uint8_t *srgb, void *stream) {
    RenderArgs A;
    const int rc = fill_args(A, verts, nullptr, normals, nullptr, nullptr, nullptr, nullptr, nullptr, march, res, ao, shadow, cam_host, params_host,
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
