/*
 * lvx_oracle.c -- CPU ORACLE (test infrastructure, NOT the product).
 *
 * A plain-C, f64, FMA-free restatement of the reference package's per-frame pipeline
 * (reference = /root/reference/pkg/src/linevox, numpy + numba).  It exists so that the
 * CUDA path can be checked on the GPU box, where the Python reference is not available.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load it.  It is pinned against golden fixtures generated from the LIVE
 * reference (tests/golden/make_golden.py -> tests/test_oracle_golden.py).
 *
 * Build:  gcc -O2 -ffp-contract=off -fopenmp -fPIC -shared lvx_oracle.c -o liblvx_oracle.so -lm
 * (-ffp-contract=off: numba/LLVM does not contract a*b+c without fastmath; neither may we.)
 *
 * Every function cites the reference file:line it follows.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef int64_t i64;
typedef uint32_t u32;
typedef uint8_t u8;

#define OCC_SCALE 4096.0

void orc_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}
int orc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ---------------------------------------------------------------- upload ----------- */

/* voxelizer.py:438  verts = (f64(v32) - world_min) / voxel_size */
void orc_to_voxel(const float *v32, i64 nv, const double *wmin, double vs, double *out) {
#pragma omp parallel for schedule(static)
    for (i64 i = 0; i < nv; i++)
        for (int a = 0; a < 3; a++) out[3 * i + a] = ((double)v32[3 * i + a] - wmin[a]) / vs;
}

/* lineset.py:74-79  every vertex index that is not the last of its polyline */
i64 orc_segment_ids(const i64 *off, i64 n_poly, i64 *segs) {
    i64 n = 0;
    for (i64 p = 0; p < n_poly; p++)
        for (i64 i = off[p]; i < off[p + 1] - 1; i++) segs[n++] = i;
    return n;
}

static double norm3(const double *d) { return sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]); }

/* lineset.py:213-242  per-vertex unit tangents; returns -(p+1) for a fully degenerate polyline */
i64 orc_clip_normals(const float *v32, const i64 *off, i64 n_poly, double *normals) {
    i64 bad = 0;
#pragma omp parallel for schedule(dynamic, 64)
    for (i64 p = 0; p < n_poly; p++) {
        i64 s = off[p], e = off[p + 1], m = e - s;
        for (i64 i = 0; i < m; i++) {
            i64 a, b; /* d = v[b] - v[a] */
            if (i == 0) { a = s; b = s + 1; }
            else if (i == m - 1) { a = e - 2; b = e - 1; }
            else { a = s + i - 1; b = s + i + 1; }
            double d[3];
            for (int c = 0; c < 3; c++) d[c] = (double)v32[3 * b + c] - (double)v32[3 * a + c];
            double len = norm3(d);
            if (len == 0.0) {
                /* lineset.py:231-240: borrow the nearest nonzero segment direction */
                i64 k = i < m - 2 ? i : m - 2; /* seg_dirs[min(i, len-1)] */
                for (int c = 0; c < 3; c++)
                    d[c] = (double)v32[3 * (s + k + 1) + c] - (double)v32[3 * (s + k) + c];
                len = norm3(d);
                if (len == 0.0) {
                    int found = 0;
                    for (i64 j = 0; j < m - 1 && !found; j++) {
                        for (int c = 0; c < 3; c++)
                            d[c] = (double)v32[3 * (s + j + 1) + c] - (double)v32[3 * (s + j) + c];
                        len = norm3(d);
                        if (len > 0.0) found = 1;
                    }
                    if (!found) {
#pragma omp critical
                        { if (bad == 0 || -(p + 1) > bad) bad = -(p + 1); }
                        d[0] = d[1] = d[2] = 0.0; len = 1.0;
                    }
                }
            }
            for (int c = 0; c < 3; c++) normals[3 * (s + i) + c] = d[c] / len;
        }
    }
    return bad;
}

/* ---------------------------------------------------------------- traversal -------- */

typedef struct { i64 *c; i64 n, cap; } cells_t;

static void cells_push(cells_t *L, i64 x, i64 y, i64 z) {
    if (L->n == L->cap) {
        L->cap = L->cap ? L->cap * 2 : 256;
        L->c = (i64 *)realloc(L->c, sizeof(i64) * 3 * L->cap);
    }
    i64 *p = L->c + 3 * L->n++;
    p[0] = x; p[1] = y; p[2] = z;
}

/* voxelizer.py:89-106 */
static void rank3(double ax, double ay, double az, int *a0, int *a1, int *a2) {
    int m = 0, r1, r2;
    if (ay > ax && ay >= az) m = 1;
    else if (az > ax && az > ay) m = 2;
    if (m == 0) { r1 = 1; r2 = 2; }
    else if (m == 1) { r1 = 0; r2 = 2; }
    else { r1 = 0; r2 = 1; }
    double vr2 = (r2 == 1) ? ay : az;
    double vr1 = (r1 == 0) ? ax : ay;
    *a0 = m;
    if (vr2 > vr1) { *a1 = r2; *a2 = r1; } else { *a1 = r1; *a2 = r2; }
}

/* voxelizer.py:116-140 */
static void aabb_cells(const double *v0, const double *v1, double r, cells_t *L) {
    i64 lo[3], hi[3];
    for (int a = 0; a < 3; a++) {
        lo[a] = (i64)floor(fmin(v0[a], v1[a]) - r);
        hi[a] = (i64)floor(fmax(v0[a], v1[a]) + r);
    }
    for (i64 z = lo[2]; z <= hi[2]; z++)
        for (i64 y = lo[1]; y <= hi[1]; y++)
            for (i64 x = lo[0]; x <= hi[0]; x++) cells_push(L, x, y, z);
}

/* voxelizer.py:143-206  Algorithm 1, major-axis slab walk */
static void capsule_cells(const double *v0in, const double *v1in, double r, cells_t *L) {
    double d[3], v0[3], v1[3], s[3], v0e[3], v1e[3], p0[3], p1[3];
    for (int a = 0; a < 3; a++) d[a] = v1in[a] - v0in[a];
    if (d[0] == 0.0 && d[1] == 0.0 && d[2] == 0.0) { aabb_cells(v0in, v1in, r, L); return; }
    int a0, a1, a2;
    rank3(fabs(d[0]), fabs(d[1]), fabs(d[2]), &a0, &a1, &a2);
    if (d[a0] < 0.0) {
        for (int a = 0; a < 3; a++) { v0[a] = v1in[a]; v1[a] = v0in[a]; d[a] = -d[a]; }
    } else {
        for (int a = 0; a < 3; a++) { v0[a] = v0in[a]; v1[a] = v1in[a]; }
    }
    for (int a = 0; a < 3; a++) {
        s[a] = d[a] / d[a0];
        v0e[a] = v0[a] - s[a] * r;
        v1e[a] = v1[a] + s[a] * r;
    }
    double q1 = d[a1] / d[a0], q2 = d[a2] / d[a0];
    double r1 = r * sqrt(1.0 + q1 * q1);
    double r2 = r * sqrt(1.0 + q2 * q2);
    i64 lo_j = (i64)floor(fmin(v0[a1], v1[a1]) - r), hi_j = (i64)floor(fmax(v0[a1], v1[a1]) + r);
    i64 lo_k = (i64)floor(fmin(v0[a2], v1[a2]) - r), hi_k = (i64)floor(fmax(v0[a2], v1[a2]) + r);
    double t_min = v0e[a0], t_max = v1e[a0], t0 = t_min;
    for (int a = 0; a < 3; a++) p0[a] = v0e[a];
    while (t0 < t_max) {
        double t1 = fmin(t_max, floor(t0 + 1.0));
        for (int a = 0; a < 3; a++) p1[a] = v0e[a] + s[a] * (t1 - t_min);
        i64 j_min = (i64)floor(fmin(p0[a1], p1[a1]) - r1), j_max = (i64)floor(fmax(p0[a1], p1[a1]) + r1);
        i64 k_min = (i64)floor(fmin(p0[a2], p1[a2]) - r2), k_max = (i64)floor(fmax(p0[a2], p1[a2]) + r2);
        if (j_min < lo_j) j_min = lo_j;
        if (j_max > hi_j) j_max = hi_j;
        if (k_min < lo_k) k_min = lo_k;
        if (k_max > hi_k) k_max = hi_k;
        i64 ci = (i64)floor(t0), c[3];
        for (i64 j = j_min; j <= j_max; j++)
            for (i64 k = k_min; k <= k_max; k++) {
                c[a0] = ci; c[a1] = j; c[a2] = k;
                cells_push(L, c[0], c[1], c[2]);
            }
        t0 = t1;
        for (int a = 0; a < 3; a++) p0[a] = p1[a];
    }
}

/* voxelizer.py:209-251 */
static void dda_cells(const double *v0, const double *v1, cells_t *L) {
    i64 x = (i64)floor(v0[0]), y = (i64)floor(v0[1]), z = (i64)floor(v0[2]);
    i64 ex = (i64)floor(v1[0]), ey = (i64)floor(v1[1]), ez = (i64)floor(v1[2]);
    i64 steps = llabs(ex - x) + llabs(ey - y) + llabs(ez - z);
    cells_push(L, x, y, z);
    if (steps == 0) return;
    double dx = v1[0] - v0[0], dy = v1[1] - v0[1], dz = v1[2] - v0[2];
    int sx = dx > 0 ? 1 : -1, sy = dy > 0 ? 1 : -1, sz = dz > 0 ? 1 : -1;
    const double big = 1e30;
    double tmx = dx != 0.0 ? ((double)(x + (sx > 0 ? 1 : 0)) - v0[0]) / dx : big;
    double tmy = dy != 0.0 ? ((double)(y + (sy > 0 ? 1 : 0)) - v0[1]) / dy : big;
    double tmz = dz != 0.0 ? ((double)(z + (sz > 0 ? 1 : 0)) - v0[2]) / dz : big;
    double tdx = dx != 0.0 ? fabs(1.0 / dx) : big;
    double tdy = dy != 0.0 ? fabs(1.0 / dy) : big;
    double tdz = dz != 0.0 ? fabs(1.0 / dz) : big;
    for (i64 i = 1; i <= steps; i++) {
        if (tmx <= tmy && tmx <= tmz) { x += sx; tmx += tdx; }
        else if (tmy <= tmz) { y += sy; tmy += tdy; }
        else { z += sz; tmz += tdz; }
        cells_push(L, x, y, z);
    }
}

static void seg_cells(const double *verts, i64 i, double r, int method, cells_t *L) {
    L->n = 0;
    if (method == 0) dda_cells(verts + 3 * i, verts + 3 * i + 3, L);
    else if (method == 1) capsule_cells(verts + 3 * i, verts + 3 * i + 3, r, L);
    else aabb_cells(verts + 3 * i, verts + 3 * i + 3, r, L);
}

/* exported for the unit known-answer test (tests/golden/unit_vectors.npz) */
i64 orc_capsule_cells(const double *v0, const double *v1, double r, i64 *out, i64 cap) {
    cells_t L = {0, 0, 0};
    capsule_cells(v0, v1, r, &L);
    i64 n = L.n;
    for (i64 i = 0; i < n && i < cap; i++) { out[3*i] = L.c[3*i]; out[3*i+1] = L.c[3*i+1]; out[3*i+2] = L.c[3*i+2]; }
    free(L.c);
    return n;
}

/* ---------------------------------------------------------------- sdf / occupancy -- */

/* voxelizer.py:254-283 */
double orc_sdf(double px, double py, double pz, double ax, double ay, double az,
               double bx, double by, double bz, double n0x, double n0y, double n0z,
               double n1x, double n1y, double n1z, double r, int use_clip) {
    double dx = bx - ax, dy = by - ay, dz = bz - az;
    double p0x = px - ax, p0y = py - ay, p0z = pz - az;
    double dd = dx * dx + dy * dy + dz * dz, h;
    if (dd > 0.0) {
        h = (p0x * dx + p0y * dy + p0z * dz) / dd;
        if (h < 0.0) h = 0.0; else if (h > 1.0) h = 1.0;
    } else h = 0.0;
    double qx = p0x - dx * h, qy = p0y - dy * h, qz = p0z - dz * h;
    double sdf = sqrt(qx * qx + qy * qy + qz * qz) - r;
    if (use_clip) {
        double s0 = -(p0x * n0x + p0y * n0y + p0z * n0z);
        double s1 = (px - bx) * n1x + (py - by) * n1y + (pz - bz) * n1z;
        if (s0 > sdf) sdf = s0;
        if (s1 > sdf) sdf = s1;
    }
    return sdf;
}

/* voxelizer.py:286-298 */
double orc_occupancy(double px, double py, double pz, double ax, double ay, double az,
                     double bx, double by, double bz, double n0x, double n0y, double n0z,
                     double n1x, double n1y, double n1z, double r, double r_min, int use_clip) {
    double rc = r > r_min ? r : r_min;
    double q = r / rc, corr = q * q;
    double sdf = orc_sdf(px, py, pz, ax, ay, az, bx, by, bz, n0x, n0y, n0z, n1x, n1y, n1z, rc, use_clip);
    double occ = 0.5 - sdf;
    if (occ < 0.0) occ = 0.0; else if (occ > 1.0) occ = 1.0;
    return occ * corr;
}

/* ---------------------------------------------------------------- voxelize --------- */

/* voxelizer.py:301-340 + 490-495.  Accumulates exact 64-bit per-voxel sums (the merge of
 * the reference's per-chunk saturating grids equals min(sum, 0xFFFF) per field), then packs.
 * `saturated` follows the single-chunk (workers=1) meaning: increments past 0xFFFF. */
void orc_voxelize(const double *verts, const i64 *segs, i64 n_seg, const double *normals,
                  int use_clip, double r, double rt, double r_min, int res, int method,
                  u32 *base, i64 *visited_out, i64 *saturated_out) {
    i64 V = (i64)res * res * res;
    uint64_t *cnt = (uint64_t *)calloc(V, sizeof(uint64_t));
    uint64_t *occ = (uint64_t *)calloc(V, sizeof(uint64_t));
#pragma omp parallel
    {
        cells_t L = {0, 0, 0};
#pragma omp for schedule(dynamic, 256)
        for (i64 si = 0; si < n_seg; si++) {
            i64 i = segs[si];
            const double *v0 = verts + 3 * i, *v1 = v0 + 3;
            const double *n0 = normals + 3 * i, *n1 = n0 + 3;
            seg_cells(verts, i, rt, method, &L);
            for (i64 c = 0; c < L.n; c++) {
                i64 x = L.c[3 * c], y = L.c[3 * c + 1], z = L.c[3 * c + 2];
                if (x < 0 || y < 0 || z < 0 || x >= res || y >= res || z >= res) continue;
                double o = orc_occupancy(x + 0.5, y + 0.5, z + 0.5, v0[0], v0[1], v0[2], v1[0], v1[1], v1[2],
                                         n0[0], n0[1], n0[2], n1[0], n1[1], n1[2], r, r_min, use_clip);
                uint64_t q = (uint64_t)(i64)rint(o * OCC_SCALE); /* python round(): half-to-even */
                i64 idx = x + (i64)res * (y + (i64)res * z);
#pragma omp atomic
                cnt[idx] += 1;
#pragma omp atomic
                occ[idx] += q;
            }
        }
        free(L.c);
    }
    i64 visited = 0, sat = 0;
#pragma omp parallel for reduction(+ : visited, sat) schedule(static)
    for (i64 i = 0; i < V; i++) {
        uint64_t c = cnt[i], o = occ[i];
        visited += (i64)c;
        if (c > 0xFFFF) { sat += (i64)(c - 0xFFFF); c = 0xFFFF; }
        if (o > 0xFFFF) o = 0xFFFF;
        base[i] = (u32)((c << 16) | o);
    }
    free(cnt); free(occ);
    *visited_out = visited; *saturated_out = sat;
}

/* level sizes: res^3, (res/2)^3, ..., 1.  offs has n_levels+1 entries. */
static int level_offsets(int res, i64 *offs) {
    int n = 0; i64 o = 0;
    for (int r = res; r >= 1; r >>= 1) { offs[n++] = o; o += (i64)r * r * r; }
    offs[n] = o;
    return n;
}
i64 orc_pyramid_size(int res) { i64 offs[40]; int n = level_offsets(res, offs); return offs[n]; }

/* voxelizer.py:422-432, 496   level 0 = min(occ_q,4096)/4096; parent = mean of 8 children */
void orc_build_mips(const u32 *base, int res, double *flat) {
    i64 offs[40] = {0};
    int n_levels = level_offsets(res, offs);
    i64 V = (i64)res * res * res;
#pragma omp parallel for schedule(static)
    for (i64 i = 0; i < V; i++) {
        u32 q = base[i] & 0xFFFF;
        if (q > 4096) q = 4096;
        flat[i] = (double)q / OCC_SCALE;
    }
    for (int l = 1; l < n_levels; l++) {
        int rl = res >> l, rp = rl * 2;
        const double *src = flat + offs[l - 1];
        double *dst = flat + offs[l];
#pragma omp parallel for collapse(2) schedule(static)
        for (int z = 0; z < rl; z++)
            for (int y = 0; y < rl; y++)
                for (int x = 0; x < rl; x++) {
                    double s = 0.0; /* exact: all terms are multiples of 2^-(12+3(l-1)) */
                    for (int dz = 0; dz < 2; dz++)
                        for (int dy = 0; dy < 2; dy++)
                            for (int dx = 0; dx < 2; dx++)
                                s += src[(2 * x + dx) + (i64)rp * ((2 * y + dy) + (i64)rp * (2 * z + dz))];
                    dst[x + (i64)rl * (y + (i64)rl * z)] = s / 8.0;
                }
    }
}

/* ---------------------------------------------------------------- culling ---------- */

/* culling.py:112-127 */
void orc_erode(const double *field, int res, double *out) {
#pragma omp parallel for collapse(2) schedule(static)
    for (int z = 0; z < res; z++)
        for (int y = 0; y < res; y++)
            for (int x = 0; x < res; x++) {
#define CL(v) ((v) < 0.0 ? 0.0 : ((v) > 1.0 ? 1.0 : (v)))
#define AT(X, Y, Z) (((X) < 0 || (Y) < 0 || (Z) < 0 || (X) >= res || (Y) >= res || (Z) >= res) ? 0.0 \
                     : CL(field[(X) + (i64)res * ((Y) + (i64)res * (Z))]))
                double m = AT(x, y, z);
                m = fmin(m, AT(x, y, z - 1)); m = fmin(m, AT(x, y, z + 1));
                m = fmin(m, AT(x, y - 1, z)); m = fmin(m, AT(x, y + 1, z));
                m = fmin(m, AT(x - 1, y, z)); m = fmin(m, AT(x + 1, y, z));
                out[x + (i64)res * (y + (i64)res * z)] = m;
#undef AT
#undef CL
            }
}

/* culling.py:143-188 */
static int march_blocked(const double *eroded, int res, i64 x, i64 y, i64 z,
                         double cx, double cy, double cz, double theta) {
    double ox = x + 0.5, oy = y + 0.5, oz = z + 0.5;
    double dx = cx - ox, dy = cy - oy, dz = cz - oz;
    i64 ex = (i64)floor(cx), ey = (i64)floor(cy), ez = (i64)floor(cz);
    int sx = dx > 0 ? 1 : -1, sy = dy > 0 ? 1 : -1, sz = dz > 0 ? 1 : -1;
    const double big = 1e30;
    double tmx = dx != 0.0 ? ((double)(x + (sx > 0 ? 1 : 0)) - ox) / dx : big;
    double tmy = dy != 0.0 ? ((double)(y + (sy > 0 ? 1 : 0)) - oy) / dy : big;
    double tmz = dz != 0.0 ? ((double)(z + (sz > 0 ? 1 : 0)) - oz) / dz : big;
    double tdx = dx != 0.0 ? fabs(1.0 / dx) : big;
    double tdy = dy != 0.0 ? fabs(1.0 / dy) : big;
    double tdz = dz != 0.0 ? fabs(1.0 / dz) : big;
    double t;
    for (;;) {
        if (tmx <= tmy && tmx <= tmz) { x += sx; t = tmx; tmx += tdx; }
        else if (tmy <= tmz) { y += sy; t = tmy; tmy += tdy; }
        else { z += sz; t = tmz; tmz += tdz; }
        if (t >= 1.0) return 0;
        if (x < 0 || y < 0 || z < 0 || x >= res || y >= res || z >= res) return 0;
        if (x == ex && y == ey && z == ez) return 0;
        if (eroded[x + (i64)res * (y + (i64)res * z)] >= theta) return 1;
    }
}

/* culling.py:191-200 */
void orc_visibility(const double *eroded, const u8 *occupied, int res,
                    double cx, double cy, double cz, double theta, u8 *out) {
    i64 V = (i64)res * res * res;
#pragma omp parallel for schedule(dynamic, 4096)
    for (i64 idx = 0; idx < V; idx++) {
        out[idx] = 0;
        if (!occupied[idx]) continue;
        i64 x = idx % res, y = (idx / res) % res, z = idx / ((i64)res * res);
        if (!march_blocked(eroded, res, x, y, z, cx, cy, cz, theta)) out[idx] = 1;
    }
}

/* culling.py:130-140 followed by `& occ_bits` (culling.py:224) */
void orc_dilate_and(const u8 *bits, const u8 *occupied, int res, u8 *out) {
#pragma omp parallel for collapse(2) schedule(static)
    for (int z = 0; z < res; z++)
        for (int y = 0; y < res; y++)
            for (int x = 0; x < res; x++) {
                u8 m = 0;
                for (int dz = -1; dz <= 1; dz++)
                    for (int dy = -1; dy <= 1; dy++)
                        for (int dx = -1; dx <= 1; dx++) {
                            int X = x + dx, Y = y + dy, Z = z + dz;
                            if (X < 0 || Y < 0 || Z < 0 || X >= res || Y >= res || Z >= res) continue;
                            if (bits[X + (i64)res * (Y + (i64)res * Z)]) m = 1;
                        }
                i64 idx = x + (i64)res * (y + (i64)res * z);
                out[idx] = (u8)(m & (occupied[idx] != 0));
            }
}

/* culling.py:103-109; flat[0:V] must already hold the base bits (0/1) */
void orc_or_mips(u8 *flat, int res) {
    i64 offs[40] = {0};
    int n_levels = level_offsets(res, offs);
    for (i64 i = 0; i < offs[1]; i++) flat[i] = flat[i] != 0;
    for (int l = 1; l < n_levels; l++) {
        int rl = res >> l, rp = rl * 2;
        const u8 *src = flat + offs[l - 1];
        u8 *dst = flat + offs[l];
        for (int z = 0; z < rl; z++)
            for (int y = 0; y < rl; y++)
                for (int x = 0; x < rl; x++) {
                    u8 m = 0;
                    for (int dz = 0; dz < 2; dz++)
                        for (int dy = 0; dy < 2; dy++)
                            for (int dx = 0; dx < 2; dx++)
                                m |= src[(2 * x + dx) + (i64)rp * ((2 * y + dy) + (i64)rp * (2 * z + dz))];
                    dst[x + (i64)rl * (y + (i64)rl * z)] = m;
                }
    }
}

/* ---------------------------------------------------------------- A-buffer --------- */

/* abuffer.py:104-114 */
i64 orc_scan_offsets(const u32 *base, const u8 *cull_base, i64 V, i64 *offsets, i64 *counts) {
    i64 run = 0;
    for (i64 i = 0; i < V; i++) {
        i64 c = (i64)(base[i] >> 16);
        if (cull_base && !cull_base[i]) c = 0;
        counts[i] = c;
        offsets[i] = run;
        run += c;
    }
    return run;
}

/* abuffer.py:145-181 */
static int segment_visible(const u8 *cull_flat, const i64 *cull_offs, int res, int n_levels,
                           i64 lo_x, i64 lo_y, i64 lo_z, i64 hi_x, i64 hi_y, i64 hi_z) {
    i64 stack[8 * 40 + 8][4];
    int sp = 0;
    stack[0][0] = n_levels - 1; stack[0][1] = stack[0][2] = stack[0][3] = 0; sp = 1;
    while (sp > 0) {
        sp--;
        i64 l = stack[sp][0], x = stack[sp][1], y = stack[sp][2], z = stack[sp][3];
        if ((x << l) > hi_x || ((x + 1) << l) <= lo_x) continue;
        if ((y << l) > hi_y || ((y + 1) << l) <= lo_y) continue;
        if ((z << l) > hi_z || ((z + 1) << l) <= lo_z) continue;
        i64 rl = res >> l;
        if (cull_flat[cull_offs[l] + x + rl * (y + rl * z)] == 0) continue;
        if (l == 0) return 1;
        for (int dz = 0; dz < 2; dz++)
            for (int dy = 0; dy < 2; dy++)
                for (int dx = 0; dx < 2; dx++) {
                    stack[sp][0] = l - 1; stack[sp][1] = 2 * x + dx;
                    stack[sp][2] = 2 * y + dy; stack[sp][3] = 2 * z + dz; sp++;
                }
    }
    return 0;
}

static int cmp_u32(const void *a, const void *b) {
    u32 x = *(const u32 *)a, y = *(const u32 *)b;
    return x < y ? -1 : (x > y);
}

/* abuffer.py:195-255, 281-328.  Counting pass + write pass.  The reference's per-chunk
 * cursors make every voxel list ascending in segment index (abuffer.py:313-317 with
 * ascending `segs`); we scatter with an atomic cursor and sort each list, which yields the
 * same arrays because a segment visits a voxel at most once.  For method dda/aabb the same
 * holds.  Returns 0, or -1 when the second traversal's counts differ from the scanned
 * counts (abuffer.py:310-311; only checked when `check` != 0, i.e. pyramid.saturated == 0). */
int orc_second_pass(const double *verts, const i64 *segs, i64 n_seg, double rt, int res, int method,
                    int use_cull, const u8 *cull_flat, const i64 *cull_offs, int n_levels,
                    const i64 *offsets, const i64 *counts, i64 total, int check,
                    u32 *frags, i64 *incidences_out) {
    i64 V = (i64)res * res * res;
    i64 *cur = (i64 *)calloc(V, sizeof(i64));
    int mismatch = 0;
#pragma omp parallel
    {
        cells_t L = {0, 0, 0};
#pragma omp for schedule(dynamic, 256)
        for (i64 si = 0; si < n_seg; si++) {
            i64 i = segs[si];
            const double *a = verts + 3 * i, *b = a + 3;
            if (use_cull) {
                i64 lo[3], hi[3];
                for (int c = 0; c < 3; c++) {
                    lo[c] = (i64)floor(fmin(a[c], b[c]) - rt);
                    hi[c] = (i64)floor(fmax(a[c], b[c]) + rt);
                }
                if (!segment_visible(cull_flat, cull_offs, res, n_levels, lo[0], lo[1], lo[2], hi[0], hi[1], hi[2]))
                    continue;
            }
            seg_cells(verts, i, rt, method, &L);
            for (i64 c = 0; c < L.n; c++) {
                i64 x = L.c[3 * c], y = L.c[3 * c + 1], z = L.c[3 * c + 2];
                if (x < 0 || y < 0 || z < 0 || x >= res || y >= res || z >= res) continue;
                i64 idx = x + (i64)res * (y + (i64)res * z);
                if (use_cull && cull_flat[idx] == 0) continue;
                i64 k;
#pragma omp atomic capture
                k = cur[idx]++;
                if (k < counts[idx] && offsets[idx] + k < total) frags[offsets[idx] + k] = (u32)i;
            }
        }
        free(L.c);
    }
    i64 inc = 0;
#pragma omp parallel for reduction(+ : inc) reduction(| : mismatch) schedule(dynamic, 4096)
    for (i64 v = 0; v < V; v++) {
        inc += cur[v];
        if (cur[v] != counts[v]) mismatch |= 1;
        i64 n = cur[v] < counts[v] ? cur[v] : counts[v];
        if (n > 1) qsort(frags + offsets[v], (size_t)n, sizeof(u32), cmp_u32);
    }
    free(cur);
    *incidences_out = inc;
    return (check && mismatch) ? -1 : 0;
}

/* ---------------------------------------------------------------- shading ---------- */

/* shading.py:72-109 */
static double trilinear(const double *flat, const i64 *offs, int res, int l, double px, double py, double pz) {
    int rl = res >> l;
    double scale = 1.0 / (double)(1 << l);
    double ux = px * scale - 0.5, uy = py * scale - 0.5, uz = pz * scale - 0.5;
    i64 ix = (i64)floor(ux), iy = (i64)floor(uy), iz = (i64)floor(uz);
    double fx = ux - ix, fy = uy - iy, fz = uz - iz;
    const double *b = flat + offs[l];
    double acc = 0.0;
    for (int dz = 0; dz < 2; dz++) {
        i64 z = iz + dz; if (z < 0) z = 0; else if (z >= rl) z = rl - 1;
        double wz = dz ? fz : 1.0 - fz;
        for (int dy = 0; dy < 2; dy++) {
            i64 y = iy + dy; if (y < 0) y = 0; else if (y >= rl) y = rl - 1;
            double wy = dy ? fy : 1.0 - fy;
            for (int dx = 0; dx < 2; dx++) {
                i64 x = ix + dx; if (x < 0) x = 0; else if (x >= rl) x = rl - 1;
                double wx = dx ? fx : 1.0 - fx;
                acc += wx * wy * wz * b[x + (i64)rl * (y + (i64)rl * z)];
            }
        }
    }
    return acc;
}

/* shading.py:112-132 */
double orc_cone_trace(const double *flat, const i64 *offs, int res, int n_levels,
                      double ox, double oy, double oz, double dx, double dy, double dz, double tan_half) {
    if (ox < 0.0 || oy < 0.0 || oz < 0.0 || ox > res || oy > res || oz > res) return 0.0;
    double occ = 0.0, t = 1.0;
    while (occ < 0.99) {
        double px = ox + dx * t, py = oy + dy * t, pz = oz + dz * t;
        if (px < 0.0 || py < 0.0 || pz < 0.0 || px > res || py > res || pz > res) break;
        double diam = 2.0 * t * tan_half;
        double step = diam > 1.0 ? diam : 1.0;
        int l = (int)floor(log2(step));
        if (l > n_levels - 1) l = n_levels - 1;
        double s = trilinear(flat, offs, res, l, px, py, pz);
        occ = occ + (1.0 - occ) * s;
        t += step;
    }
    return occ < 1.0 ? occ : 1.0;
}

/* shading.py:135-155, 170-185 */
void orc_shading(const double *flat, int res, const u8 *visible, const double *dirs, int n_dirs,
                 double tan_ao, double lx, double ly, double lz, double tan_shadow,
                 float *ao_out, float *shadow_out) {
    i64 offs[40] = {0};
    int n_levels = level_offsets(res, offs);
    i64 V = (i64)res * res * res;
    double w = 1.0 / n_dirs;
#pragma omp parallel for schedule(dynamic, 1024)
    for (i64 idx = 0; idx < V; idx++) {
        double ao = 1.0, sh = 1.0;
        if (visible[idx]) {
            i64 x = idx % res, y = (idx / res) % res, z = idx / ((i64)res * res);
            double ox = x + 0.5, oy = y + 0.5, oz = z + 0.5, acc = 0.0;
            for (int c = 0; c < n_dirs; c++)
                acc += w * orc_cone_trace(flat, offs, res, n_levels, ox, oy, oz,
                                          dirs[3 * c], dirs[3 * c + 1], dirs[3 * c + 2], tan_ao);
            ao = 1.0 - acc;
            sh = 1.0 - orc_cone_trace(flat, offs, res, n_levels, ox, oy, oz, -lx, -ly, -lz, tan_shadow);
            if (ao < 0.0) ao = 0.0; else if (ao > 1.0) ao = 1.0;
            if (sh < 0.0) sh = 0.0; else if (sh > 1.0) sh = 1.0;
        }
        ao_out[idx] = (float)ao;
        shadow_out[idx] = (float)sh;
    }
}

/* ---------------------------------------------------------------- ray tracing ------ */

typedef struct {
    double ax, ay, az, bx, by, bz, n0x, n0y, n0z, n1x, n1y, n1z, r;
    int use_clip;
} cap_t;

static int clip_ok(const cap_t *c, double px, double py, double pz) {
    if (!c->use_clip) return 1;
    if ((px - c->ax) * c->n0x + (py - c->ay) * c->n0y + (pz - c->az) * c->n0z < -1e-9) return 0;
    if ((px - c->bx) * c->n1x + (py - c->by) * c->n1y + (pz - c->bz) * c->n1z > 1e-9) return 0;
    return 1;
}

/* raytracer.py:113-222 */
static double ray_capsule(double ox, double oy, double oz, double dx, double dy, double dz, const cap_t *c) {
    double ax = c->ax, ay = c->ay, az = c->az, bx = c->bx, by = c->by, bz = c->bz, r = c->r;
    double bax = bx - ax, bay = by - ay, baz = bz - az;
    double oax = ox - ax, oay = oy - ay, oaz = oz - az;
    double baba = bax * bax + bay * bay + baz * baz;
    const double eps = 1e-12;
    double best = -1.0;
    if (baba > eps) {
        double bard = bax * dx + bay * dy + baz * dz;
        double baoa = bax * oax + bay * oay + baz * oaz;
        double rdoa = dx * oax + dy * oay + dz * oaz;
        double oaoa = oax * oax + oay * oay + oaz * oaz;
        double a_ = baba - bard * bard;
        double b_ = baba * rdoa - baoa * bard;
        double c_ = baba * oaoa - baoa * baoa - r * r * baba;
        if (fabs(a_) > eps) {
            double disc = b_ * b_ - a_ * c_;
            if (disc >= 0.0) {
                double sq = sqrt(disc);
                for (int k = 0; k < 2; k++) {
                    double sgn = k ? 1.0 : -1.0;
                    double t = (-b_ + sgn * sq) / a_;
                    if (t >= 0.0) {
                        double y = baoa + t * bard;
                        if (-1e-9 <= y && y <= baba + 1e-9) {
                            double px = ox + dx * t, py = oy + dy * t, pz = oz + dz * t;
                            if (clip_ok(c, px, py, pz) && (best < 0.0 || t < best)) best = t;
                        }
                    }
                }
            }
        }
    }
    for (int cap = 0; cap < 2; cap++) {
        double cx = cap ? bx : ax, cy = cap ? by : ay, cz = cap ? bz : az;
        double ocx = ox - cx, ocy = oy - cy, ocz = oz - cz;
        double bq = ocx * dx + ocy * dy + ocz * dz;
        double cq = ocx * ocx + ocy * ocy + ocz * ocz - r * r;
        double disc = bq * bq - cq;
        if (disc < 0.0) continue;
        double sq = sqrt(disc);
        for (int k = 0; k < 2; k++) {
            double sgn = k ? 1.0 : -1.0;
            double t = -bq + sgn * sq;
            if (t < 0.0) continue;
            double px = ox + dx * t, py = oy + dy * t, pz = oz + dz * t;
            double y = (px - ax) * bax + (py - ay) * bay + (pz - az) * baz;
            int on_cap = cap == 0 ? (y <= 1e-9) : (y >= baba - 1e-9);
            if (baba <= eps) on_cap = cap == 0;
            if (on_cap && clip_ok(c, px, py, pz) && (best < 0.0 || t < best)) best = t;
        }
    }
    if (c->use_clip) {
        for (int pl = 0; pl < 2; pl++) {
            double nx = pl ? c->n1x : c->n0x, ny = pl ? c->n1y : c->n0y, nz = pl ? c->n1z : c->n0z;
            double qx = pl ? bx : ax, qy = pl ? by : ay, qz = pl ? bz : az;
            double dn = dx * nx + dy * ny + dz * nz;
            if (fabs(dn) < eps) continue;
            double t = ((qx - ox) * nx + (qy - oy) * ny + (qz - oz) * nz) / dn;
            if (t < 0.0) continue;
            double px = ox + dx * t, py = oy + dy * t, pz = oz + dz * t, h;
            if (baba > eps) h = ((px - ax) * bax + (py - ay) * bay + (pz - az) * baz) / baba;
            else h = 0.0;
            if (h < 0.0) h = 0.0; else if (h > 1.0) h = 1.0;
            double wx = px - (ax + bax * h), wy = py - (ay + bay * h), wz = pz - (az + baz * h);
            if (wx * wx + wy * wy + wz * wz > r * r + 1e-9) continue;
            if (clip_ok(c, px, py, pz) && (best < 0.0 || t < best)) best = t;
        }
    }
    return best;
}

/* raytracer.py:225-256 */
static void capsule_normal(double px, double py, double pz, const cap_t *c, double *n) {
    double ax = c->ax, ay = c->ay, az = c->az, bx = c->bx, by = c->by, bz = c->bz;
    double bax = bx - ax, bay = by - ay, baz = bz - az;
    double baba = bax * bax + bay * bay + baz * baz, h;
    if (baba > 1e-12) {
        h = ((px - ax) * bax + (py - ay) * bay + (pz - az) * baz) / baba;
        if (h < 0.0) h = 0.0; else if (h > 1.0) h = 1.0;
    } else h = 0.0;
    double wx = px - (ax + bax * h), wy = py - (ay + bay * h), wz = pz - (az + baz * h);
    double s_cap = sqrt(wx * wx + wy * wy + wz * wz) - c->r;
    double nx = wx, ny = wy, nz = wz;
    if (c->use_clip) {
        double s0 = -((px - ax) * c->n0x + (py - ay) * c->n0y + (pz - az) * c->n0z);
        double s1 = (px - bx) * c->n1x + (py - by) * c->n1y + (pz - bz) * c->n1z;
        if (s0 >= s_cap && s0 >= s1) { nx = -c->n0x; ny = -c->n0y; nz = -c->n0z; }
        else if (s1 >= s_cap) { nx = c->n1x; ny = c->n1y; nz = c->n1z; }
    }
    double nn = sqrt(nx * nx + ny * ny + nz * nz);
    if (nn == 0.0) { n[0] = 0.0; n[1] = 0.0; n[2] = 1.0; return; }
    n[0] = nx / nn; n[1] = ny / nn; n[2] = nz / nn;
}

/* known-answer entry points (tests/golden/unit_vectors.npz) */
double orc_ray_capsule(const double *o, const double *d, const double *a, const double *b,
                       const double *n0, const double *n1, double r, int use_clip) {
    cap_t c = {a[0], a[1], a[2], b[0], b[1], b[2], n0[0], n0[1], n0[2], n1[0], n1[1], n1[2], r, use_clip};
    return ray_capsule(o[0], o[1], o[2], d[0], d[1], d[2], &c);
}
void orc_capsule_normal(const double *p, const double *a, const double *b, const double *n0,
                        const double *n1, double r, int use_clip, double *out) {
    cap_t c = {a[0], a[1], a[2], b[0], b[1], b[2], n0[0], n0[1], n0[2], n1[0], n1[1], n1[2], r, use_clip};
    capsule_normal(p[0], p[1], p[2], &c, out);
}

static void load_cap(cap_t *c, const double *verts, const double *normals, i64 i, double r, int use_clip) {
    const double *a = verts + 3 * i, *n = normals + 3 * i;
    c->ax = a[0]; c->ay = a[1]; c->az = a[2]; c->bx = a[3]; c->by = a[4]; c->bz = a[5];
    c->n0x = n[0]; c->n0y = n[1]; c->n0z = n[2]; c->n1x = n[3]; c->n1y = n[4]; c->n1z = n[5];
    c->r = r; c->use_clip = use_clip;
}

/* raytracer.py:272-291 */
static void grid_clip(double ox, double oy, double oz, double dx, double dy, double dz, int res,
                      double *t0o, double *t1o) {
    double t0 = 0.0, t1 = 1e30;
    double o[3] = {ox, oy, oz}, d[3] = {dx, dy, dz};
    for (int a = 0; a < 3; a++) {
        if (d[a] == 0.0) {
            if (o[a] < 0.0 || o[a] > res) { *t0o = 1.0; *t1o = -1.0; return; }
        } else {
            double ta = (0.0 - o[a]) / d[a], tb = ((double)res - o[a]) / d[a];
            if (ta > tb) { double tmp = ta; ta = tb; tb = tmp; }
            if (ta > t0) t0 = ta;
            if (tb < t1) t1 = tb;
        }
    }
    *t0o = t0; *t1o = t1;
}

/* raytracer.py:294-313 */
static double voxel_exit(double ox, double oy, double oz, double dx, double dy, double dz,
                         i64 x, i64 y, i64 z, int lvl) {
    i64 size = (i64)1 << lvl;
    i64 bx = (x >> lvl) << lvl, by = (y >> lvl) << lvl, bz = (z >> lvl) << lvl;
    double t = 1e30;
    if (dx > 0.0) t = fmin(t, ((double)(bx + size) - ox) / dx); else if (dx < 0.0) t = fmin(t, ((double)bx - ox) / dx);
    if (dy > 0.0) t = fmin(t, ((double)(by + size) - oy) / dy); else if (dy < 0.0) t = fmin(t, ((double)by - oy) / dy);
    if (dz > 0.0) t = fmin(t, ((double)(bz + size) - oz) / dz); else if (dz < 0.0) t = fmin(t, ((double)bz - oz) / dz);
    return t;
}

/* raytracer.py:316-326 */
static int empty_level(const u8 *bits, const i64 *offs, int res, int n_levels, i64 x, i64 y, i64 z) {
    int l = 0;
    while (l < n_levels - 1) {
        int nl = l + 1;
        i64 rl = res >> nl;
        if (bits[offs[nl] + (x >> nl) + rl * ((y >> nl) + rl * (z >> nl))] != 0) break;
        l = nl;
    }
    return l;
}

/* raytracer.py:368-390; volumes are f32 on our side, widened exactly like
 * np.ascontiguousarray(..., dtype=float64) (raytracer.py:682-683) */
static double tri3d(const float *vol, int res, double px, double py, double pz) {
    double ux = px - 0.5, uy = py - 0.5, uz = pz - 0.5;
    i64 ix = (i64)floor(ux), iy = (i64)floor(uy), iz = (i64)floor(uz);
    double fx = ux - ix, fy = uy - iy, fz = uz - iz, acc = 0.0;
    for (int dz = 0; dz < 2; dz++) {
        i64 z = iz + dz; if (z < 0) z = 0; if (z > res - 1) z = res - 1;
        double wz = dz ? fz : 1.0 - fz;
        for (int dy = 0; dy < 2; dy++) {
            i64 y = iy + dy; if (y < 0) y = 0; if (y > res - 1) y = res - 1;
            double wy = dy ? fy : 1.0 - fy;
            for (int dx = 0; dx < 2; dx++) {
                i64 x = ix + dx; if (x < 0) x = 0; if (x > res - 1) x = res - 1;
                double wx = dx ? fx : 1.0 - fx;
                acc += wx * wy * wz * (double)vol[x + (i64)res * (y + (i64)res * z)];
            }
        }
    }
    return acc;
}

typedef struct {
    const double *verts, *normals; int use_clip; double r;
    const i64 *frag_off, *frag_cnt; const u32 *frags;
    const u8 *bits; i64 bits_offs[40]; int res, n_levels;
    const float *ao, *sh; double lx, ly, lz;
} scene_t;

/* raytracer.py:393-411 */
static void shade(const scene_t *S, i64 i, const double *n, double px, double py, double pz, double *rgb) {
    const double *a = S->verts + 3 * i;
    double sx = a[3] - a[0], sy = a[4] - a[1], sz = a[5] - a[2];
    double sn = sqrt(sx * sx + sy * sy + sz * sz), cr, cg, cb;
    if (sn == 0.0) cr = cg = cb = 0.5;
    else { cr = fabs(sx) / sn; cg = fabs(sy) / sn; cb = fabs(sz) / sn; }
    double ao = S->ao ? tri3d(S->ao, S->res, px, py, pz) : 1.0;
    double sh = S->sh ? tri3d(S->sh, S->res, px, py, pz) : 1.0;
    double ndl = n[0] * S->lx + n[1] * S->ly + n[2] * S->lz;
    if (ndl < 0.0) ndl = 0.0;
    double k = 0.4 * ao + 0.6 * sh * ndl;
    rgb[0] = cr * k; rgb[1] = cg * k; rgb[2] = cb * k;
}

/* raytracer.py:414-423 */
static void pixel_ray(int px, int py, int w, int h, const double *fwd, const double *right,
                      const double *up, double tanf, double *d) {
    double aspect = (double)w / (double)h;
    double u = (2.0 * (px + 0.5) / w - 1.0) * aspect * tanf;
    double v = (1.0 - 2.0 * (py + 0.5) / h) * tanf;
    double dx = fwd[0] + u * right[0] + v * up[0];
    double dy = fwd[1] + u * right[1] + v * up[1];
    double dz = fwd[2] + u * right[2] + v * up[2];
    double dn = sqrt(dx * dx + dy * dy + dz * dz);
    d[0] = dx / dn; d[1] = dy / dn; d[2] = dz / dn;
}

/* raytracer.py:459-515 (mode 0) and 518-645 (mode 1).  rgb f64 (h,w,3), hit_id i32, tests i64.
 * ao/sh may be NULL (= all ones, raytracer.py:685-688; light then is (0,0,-1) by the caller). */
void orc_render(const double *verts, const double *normals, int use_clip, double r,
                const i64 *frag_off, const i64 *frag_cnt, const u32 *frags,
                const u8 *bits, int res, const float *ao, const float *sh,
                const double *light_to_src, const double *pos, const double *fwd, const double *right,
                const double *up, double tanf, int mode, double alpha, int kslots, int early_term,
                const double *bg, int w, int h, double *rgb, int32_t *hit_id, i64 *test_counts) {
    scene_t S;
    S.verts = verts; S.normals = normals; S.use_clip = use_clip; S.r = r;
    S.frag_off = frag_off; S.frag_cnt = frag_cnt; S.frags = frags; S.bits = bits;
    S.res = res; S.n_levels = level_offsets(res, S.bits_offs);
    S.ao = ao; S.sh = sh; S.lx = light_to_src[0]; S.ly = light_to_src[1]; S.lz = light_to_src[2];
    double ox = pos[0], oy = pos[1], oz = pos[2];
#pragma omp parallel for schedule(dynamic, 64)
    for (i64 pix = 0; pix < (i64)w * h; pix++) {
        int px = (int)(pix % w), py = (int)(pix / w);
        double d[3];
        pixel_ray(px, py, w, h, fwd, right, up, tanf, d);
        double dx = d[0], dy = d[1], dz = d[2];
        i64 n_tests = 0;
        double t0, t1;
        grid_clip(ox, oy, oz, dx, dy, dz, res, &t0, &t1);
        cap_t c;
        if (mode == 0) {
            int found = 0;
            if (t1 >= t0) {
                double t = t0 > 0.0 ? t0 : 0.0;
                while (t < t1) {
                    double tm = t + 1e-6, te;
                    i64 x = (i64)floor(ox + dx * tm), y = (i64)floor(oy + dy * tm), z = (i64)floor(oz + dz * tm);
                    if (x < 0 || y < 0 || z < 0 || x >= res || y >= res || z >= res) break;
                    i64 idx = x + (i64)res * (y + (i64)res * z);
                    if (bits[idx] != 0) {
                        /* raytracer.py:430-456 */
                        double best = -1.0; i64 best_i = -1;
                        i64 fo = frag_off[idx], fn = frag_cnt[idx];
                        for (i64 s = 0; s < fn; s++) {
                            i64 i = (i64)frags[fo + s];
                            load_cap(&c, verts, normals, i, r, use_clip);
                            double tt = ray_capsule(ox, oy, oz, dx, dy, dz, &c);
                            n_tests++;
                            if (tt < 0.0) continue;
                            i64 hx = (i64)floor(ox + dx * tt), hy = (i64)floor(oy + dy * tt), hz = (i64)floor(oz + dz * tt);
                            if (hx != x || hy != y || hz != z) continue;
                            if (best < 0.0 || tt < best) { best = tt; best_i = i; }
                        }
                        if (best >= 0.0) {
                            double hx = ox + dx * best, hy = oy + dy * best, hz = oz + dz * best, n[3];
                            load_cap(&c, verts, normals, best_i, r, use_clip);
                            capsule_normal(hx, hy, hz, &c, n);
                            shade(&S, best_i, n, hx, hy, hz, rgb + 3 * pix);
                            hit_id[pix] = (int32_t)best_i;
                            found = 1;
                            break;
                        }
                        te = voxel_exit(ox, oy, oz, dx, dy, dz, x, y, z, 0);
                    } else {
                        int l = empty_level(bits, S.bits_offs, res, S.n_levels, x, y, z);
                        te = voxel_exit(ox, oy, oz, dx, dy, dz, x, y, z, l);
                    }
                    t = te > t ? te : t + 1e-6;
                }
            }
            if (!found) {
                rgb[3 * pix] = bg[0]; rgb[3 * pix + 1] = bg[1]; rgb[3 * pix + 2] = bg[2];
                hit_id[pix] = -1;
            }
        } else {
            double col[3] = {0.0, 0.0, 0.0}, acc_a = 0.0;
            i64 first_hit = -1;
            i64 keybuf[64], ibuf[64];
            double tbuf[64];
            if (t1 >= t0) {
                double t = t0 > 0.0 ? t0 : 0.0;
                while (t < t1) {
                    if (early_term && acc_a >= 0.999) break;
                    double tm = t + 1e-6, te;
                    i64 x = (i64)floor(ox + dx * tm), y = (i64)floor(oy + dy * tm), z = (i64)floor(oz + dz * tm);
                    if (x < 0 || y < 0 || z < 0 || x >= res || y >= res || z >= res) break;
                    i64 idx = x + (i64)res * (y + (i64)res * z);
                    if (bits[idx] == 0) {
                        int l = empty_level(bits, S.bits_offs, res, S.n_levels, x, y, z);
                        te = voxel_exit(ox, oy, oz, dx, dy, dz, x, y, z, l);
                        t = te > t ? te : t + 1e-6;
                        continue;
                    }
                    te = voxel_exit(ox, oy, oz, dx, dy, dz, x, y, z, 0);
                    double t_enter = t, span = te - t_enter;
                    double inv_span = span > 0.0 ? 65535.0 / span : 0.0;
                    i64 fo = frag_off[idx], fn = frag_cnt[idx];
                    i64 last_key = -1;
                    for (;;) {
                        int kept = 0; i64 accepted = 0;
                        for (i64 s = 0; s < fn; s++) {
                            i64 i = (i64)frags[fo + s];
                            load_cap(&c, verts, normals, i, r, use_clip);
                            double tt = ray_capsule(ox, oy, oz, dx, dy, dz, &c);
                            n_tests++;
                            if (tt < 0.0) continue;
                            i64 hx = (i64)floor(ox + dx * tt), hy = (i64)floor(oy + dy * tt), hz = (i64)floor(oz + dz * tt);
                            if (hx != x || hy != y || hz != z) continue;
                            i64 q = (i64)((tt - t_enter) * inv_span); /* int(): truncation */
                            if (q < 0) q = 0; else if (q > 65535) q = 65535;
                            i64 key = (q << 16) | s;
                            if (key <= last_key) continue;
                            accepted++;
                            int j;
                            if (kept < kslots) { j = kept; kept++; }
                            else if (key < keybuf[kslots - 1]) j = kslots - 1;
                            else continue;
                            while (j > 0 && keybuf[j - 1] > key) {
                                keybuf[j] = keybuf[j - 1]; tbuf[j] = tbuf[j - 1]; ibuf[j] = ibuf[j - 1]; j--;
                            }
                            keybuf[j] = key; tbuf[j] = tt; ibuf[j] = i;
                        }
                        for (int j = 0; j < kept; j++) {
                            if (early_term && acc_a >= 0.999) break;
                            double tt = tbuf[j]; i64 i = ibuf[j];
                            double hx = ox + dx * tt, hy = oy + dy * tt, hz = oz + dz * tt, n[3], cc[3];
                            load_cap(&c, verts, normals, i, r, use_clip);
                            capsule_normal(hx, hy, hz, &c, n);
                            shade(&S, i, n, hx, hy, hz, cc);
                            double wgt = (1.0 - acc_a) * alpha;
                            col[0] += wgt * cc[0]; col[1] += wgt * cc[1]; col[2] += wgt * cc[2];
                            acc_a += wgt;
                            if (first_hit < 0) first_hit = i;
                        }
                        if (accepted <= kslots) break;
                        if (early_term && acc_a >= 0.999) break;
                        last_key = keybuf[kslots - 1];
                    }
                    t = te > t ? te : t + 1e-6;
                }
            }
            rgb[3 * pix] = col[0] + (1.0 - acc_a) * bg[0];
            rgb[3 * pix + 1] = col[1] + (1.0 - acc_a) * bg[1];
            rgb[3 * pix + 2] = col[2] + (1.0 - acc_a) * bg[2];
            hit_id[pix] = (int32_t)first_hit;
        }
        test_counts[pix] = n_tests;
    }
}

/* debugging / known-answer entry points */
void orc_pixel_ray(int px, int py, int w, int h, const double *fwd, const double *right,
                   const double *up, double tanf, double *d) { pixel_ray(px, py, w, h, fwd, right, up, tanf, d); }
double orc_tri3d(const float *vol, int res, double px, double py, double pz) { return tri3d(vol, res, px, py, pz); }
