// shade.cu -- voxel-cone-traced ambient occlusion and directional shadow over the occupancy
// pyramid.  Replaces lv/shading.py:72-109 (_trilinear), 112-132 (_cone_trace), 135-155
// (_shading_kernel) and the clip/f32 store of compute_shading (170-185).
//
// Work layout: visible voxels are compacted first, then one thread per visible voxel marches
// the 12 AO cones and the shadow cone (see k_shade for why that is the coalesced mapping).
#include "lvx_device.cuh"

namespace lvx {

struct ShadeParams {
    double dirs[15][3];
    double shadow_dir[3];   // -light
    double inv_dirs[15][3], inv_shadow[3];   // 1/d per component (0 where d == 0), for the t_safe bound only
    double tan_ao, tan_shadow, w;
    uint32_t mip_off[16];   // element offset of level l (l >= 1) inside `mips`
    uint32_t mask_off[16];  // word offset of level l inside the non-empty masks
    int n_dirs, res, n_levels;
};

// Non-empty masks.  Bit (ix,iy,iz) of level l says "some tap of the trilinear footprint
// [ix,ix+1]x[iy,iy+1]x[iz,iz+1] of level l is non-zero" (always set on the last row/column/slice,
// where the footprint is clamped).  A cleared bit means the sample is exactly 0.0, and
// occ + (1-occ)*0.0 == occ bit for bit, so the eight loads and ~30 f64 operations of that sample
// can be skipped without changing the result.  One bit per cell, x fastest: the 32 lanes of a
// warp (x-adjacent voxels, same cone) read the same word.
__device__ __forceinline__ bool cell_nonzero(const uint32_t *__restrict__ base, const double *__restrict__ lvl,
                                             int l, uint32_t idx) {
    return l == 0 ? (base[idx] & 0xFFFFu) != 0 : lvl[idx] != 0.0;
}

__global__ void __launch_bounds__(256)
k_nzmask(const uint32_t *__restrict__ base, const double *__restrict__ lvl, int l, int rl,
         uint32_t *__restrict__ mask) {
    const uint32_t n = (uint32_t)rl * rl * rl;
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    bool any = false;
    if (i < n) {
        const int x = i % rl, y = (i / rl) % rl, z = i / (rl * rl);
        if (x == rl - 1 || y == rl - 1 || z == rl - 1) any = true;
        else {
            // (all eight taps are loaded before the first is tested: independent loads, one round trip)
#pragma unroll
            for (int k = 0; k < 8; k++)
                any |= cell_nonzero(base, lvl, l, (x + (k & 1)) + (uint32_t)rl * ((y + ((k >> 1) & 1)) + (uint32_t)rl * (z + (k >> 2))));
        }
    }
    const uint32_t m = __ballot_sync(0xffffffffu, any);
    if ((threadIdx.x & 31) == 0 && i < n) mask[i >> 5] = m;
}

// The masks of all levels with <= 16^3 cells in one launch (a single CTA; the levels are independent).
struct NzTail { uint32_t mip_off[16], mask_off[16]; int first, n_levels, res; };
__global__ void __launch_bounds__(1024)
k_nzmask_tail(const double *__restrict__ mips, const NzTail T, uint32_t *__restrict__ masks) {
    const int lane = threadIdx.x & 31;
    for (int l = T.first; l < T.n_levels; l++) {
        const int rl = T.res >> l;
        const int n = rl * rl * rl;
        const double *lvl = mips + T.mip_off[l];
        for (int i0 = threadIdx.x - lane; i0 < n; i0 += blockDim.x) {      // warp-uniform trip count
            const int i = i0 + lane;
            bool any = false;
            if (i < n) {
                const int x = i % rl, y = (i / rl) % rl, z = i / (rl * rl);
                if (x == rl - 1 || y == rl - 1 || z == rl - 1) any = true;
                else {
#pragma unroll
                    for (int k = 0; k < 8; k++)
                        any |= lvl[(x + (k & 1)) + rl * ((y + ((k >> 1) & 1)) + rl * (z + (k >> 2)))] != 0.0;
                }
            }
            const uint32_t m = __ballot_sync(0xffffffffu, any);
            if (lane == 0) masks[T.mask_off[l] + (i >> 5)] = m;
        }
    }
}

// Level-0 footprint mask from the one-bit-per-voxel "occupancy non-zero" words (lvx_pack_wide):
// one thread per 32 cells.  Same result as k_nzmask at level 0 (rl a multiple of 32).
__global__ void __launch_bounds__(256)
k_nzmask_bits(const uint32_t *__restrict__ nz, int rl, uint32_t *__restrict__ mask) {
    const int wpr = rl >> 5;                                   // words per x-row
    const uint32_t n_words = (uint32_t)wpr * rl * rl;
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_words) return;
    const int w = i % wpr, y = (i / wpr) % rl, z = i / (wpr * rl);
    uint32_t m = 0xffffffffu;                                  // last row / slice: always set
    if (y < rl - 1 && z < rl - 1) {
        m = 0;
#pragma unroll
        for (int dz = 0; dz < 2; dz++)
#pragma unroll
            for (int dy = 0; dy < 2; dy++) {
                const uint32_t r = (uint32_t)w + (uint32_t)wpr * ((uint32_t)(y + dy) + (uint32_t)rl * (uint32_t)(z + dz));
                const uint32_t a = nz[r];
                const uint32_t nx = w + 1 < wpr ? nz[r + 1] : 0u;
                m |= a | (a >> 1) | (nx << 31);
            }
        if (w == wpr - 1) m |= 0x80000000u;                    // x = rl - 1: always set
    }
    mask[i] = m;
}

// lv/shading.py:72-109; level 0 is read straight from the packed base words
template <bool CLAMP>
__device__ __forceinline__ double trilinear(const uint32_t *__restrict__ base, const double *__restrict__ lvl,
                                            int l, int rl, int ix, int iy, int iz, double fx, double fy, double fz) {
    double acc = 0.0;
#pragma unroll
    for (int dz = 0; dz < 2; dz++) {
        const int z = CLAMP ? min(max(iz + dz, 0), rl - 1) : iz + dz;
        const double wz = dz ? fz : 1.0 - fz;
#pragma unroll
        for (int dy = 0; dy < 2; dy++) {
            const int y = CLAMP ? min(max(iy + dy, 0), rl - 1) : iy + dy;
            const double wy = dy ? fy : 1.0 - fy;
#pragma unroll
            for (int dx = 0; dx < 2; dx++) {
                const int x = CLAMP ? min(max(ix + dx, 0), rl - 1) : ix + dx;
                const double wx = dx ? fx : 1.0 - fx;
                const uint32_t idx = (uint32_t)x + (uint32_t)rl * ((uint32_t)y + (uint32_t)rl * (uint32_t)z);
                double val;
                if (l == 0) val = (double)min(base[idx] & 0xFFFFu, 4096u) * (1.0 / 4096.0);
                else val = lvl[idx];
                acc += wx * wy * wz * val;
            }
        }
    }
    return acc;
}

// lv/shading.py:112-132
__device__ __forceinline__ double cone_trace(const uint32_t *__restrict__ base, const double *__restrict__ mips,
                                             const uint32_t *__restrict__ masks, const ShadeParams &P,
                                             double ox, double oy, double oz,
                                             double dx, double dy, double dz, const double *inv_d, double tan_half) {
    const double R = (double)P.res;
    if (ox < 0.0 || oy < 0.0 || oz < 0.0 || ox > R || oy > R || oz > R) return 0.0;
    // while t <= t_safe the sample point is inside [1e-3, R-1e-3]^3 for certain, so the exact
    // six-way bounds test (line 122 of the reference) cannot fire and is not evaluated.  t_safe is
    // only this gate, so it is formed with the host's reciprocals (a product instead of three
    // divisions per cone); the 1e-3-voxel margin covers the rounding of the product many times over.
    double t_safe = 1e30;
    {
        const double o[3] = {ox, oy, oz}, d[3] = {dx, dy, dz};
#pragma unroll
        for (int a = 0; a < 3; a++) {
            if (d[a] > 0.0) t_safe = fmin(t_safe, (R - 1e-3 - o[a]) * inv_d[a]);
            else if (d[a] < 0.0) t_safe = fmin(t_safe, (1e-3 - o[a]) * inv_d[a]);
        }
    }
    double occ = 0.0, t = 1.0;
    while (occ < 0.99) {
        const double px = ox + dx * t, py = oy + dy * t, pz = oz + dz * t;
        if (t > t_safe && (px < 0.0 || py < 0.0 || pz < 0.0 || px > R || py > R || pz > R)) break;
        const double diam = 2.0 * t * tan_half;
        const double step = diam > 1.0 ? diam : 1.0;
        // floor(log2(step)), step >= 1: the unbiased exponent
        int l = (int)((__double_as_longlong(step) >> 52) & 0x7ff) - 1023;
        if (l > P.n_levels - 1) l = P.n_levels - 1;
        const int rl = P.res >> l;
        const double scale = __longlong_as_double((long long)(1023 - l) << 52);   // 1.0 / (1 << l), exact
        const double ux = px * scale - 0.5, uy = py * scale - 0.5, uz = pz * scale - 0.5;
        const int ix = (int)floor(ux), iy = (int)floor(uy), iz = (int)floor(uz);
        const double *lvl = mips + P.mip_off[l];
        const bool interior = ix >= 0 && iy >= 0 && iz >= 0 && ix < rl - 1 && iy < rl - 1 && iz < rl - 1;
        if (interior) {
            const uint32_t cell = (uint32_t)ix + (uint32_t)rl * ((uint32_t)iy + (uint32_t)rl * (uint32_t)iz);
            if ((masks[P.mask_off[l] + (cell >> 5)] >> (cell & 31)) & 1u) {
                const double s = trilinear<false>(base, lvl, l, rl, ix, iy, iz, ux - ix, uy - iy, uz - iz);
                occ = occ + (1.0 - occ) * s;
            }   // else: s == 0.0 exactly and occ is unchanged
        } else {
            const double s = trilinear<true>(base, lvl, l, rl, ix, iy, iz, ux - ix, uy - iy, uz - iz);
            occ = occ + (1.0 - occ) * s;
        }
        t += step;
    }
    return occ < 1.0 ? occ : 1.0;
}

// ao = shadow = 1 everywhere (lv/shading.py:177-178)
__global__ void __launch_bounds__(256)
k_shade_fill(int64_t n4, float4 *__restrict__ ao, float4 *__restrict__ shadow) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n4) { ao[i] = make_float4(1.f, 1.f, 1.f, 1.f); shadow[i] = make_float4(1.f, 1.f, 1.f, 1.f); }
}

// One thread per visible voxel; a warp holds 32 consecutive entries of the compacted list, i.e.
// (mostly) x-adjacent voxels.  All lanes march the SAME cone direction in lock step: t, step and
// the mip level depend only on t, so the loop is convergent and the 8 trilinear taps of the 32
// lanes fall on consecutive addresses (or the same address at coarse levels) -- a few L1
// wavefronts per load instead of one per lane.  The 12 AO cones are folded in cone order in a
// register (lv/shading.py:150-152), so the f64 sum has the reference's rounding.
#ifndef LVX_SHADE_MINB
#define LVX_SHADE_MINB 6
#endif
__global__ void __launch_bounds__(128, LVX_SHADE_MINB)
k_shade(const uint32_t *__restrict__ base, const double *__restrict__ mips,
        const uint32_t *__restrict__ masks, const ShadeParams P, const uint32_t *__restrict__ vis_list,
        float *__restrict__ ao, float *__restrict__ shadow) {
    const int64_t n = (int64_t)*reinterpret_cast<const unsigned long long *>(vis_list);
    const uint32_t *__restrict__ list = vis_list + LVX_LIST_HDR;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += stride) {
        const int64_t idx = list[e];
        const int x = (int)(idx % P.res), y = (int)((idx / P.res) % P.res), z = (int)(idx / ((int64_t)P.res * P.res));
        const double ox = x + 0.5, oy = y + 0.5, oz = z + 0.5;
        double acc = 0.0;
        for (int c = 0; c < P.n_dirs; c++)
            acc += P.w * cone_trace(base, mips, masks, P, ox, oy, oz, P.dirs[c][0], P.dirs[c][1], P.dirs[c][2], P.inv_dirs[c],
                                    P.tan_ao);
        const double sh = cone_trace(base, mips, masks, P, ox, oy, oz, P.shadow_dir[0], P.shadow_dir[1], P.shadow_dir[2],
                                     P.inv_shadow, P.tan_shadow);
        double a = 1.0 - acc, s = 1.0 - sh;
        a = a < 0.0 ? 0.0 : (a > 1.0 ? 1.0 : a);     // lv/shading.py:183-184
        s = s < 0.0 ? 0.0 : (s > 1.0 ? 1.0 : s);
        ao[idx] = (float)a;                          // lv/shading.py:185
        shadow[idx] = (float)s;
    }
}

}  // namespace lvx

using namespace lvx;

extern "C" {

// scratch: the non-empty masks of all levels
int64_t lvx_shade_scratch_bytes(int64_t n_voxels) {
    int64_t words = 0;
    for (int64_t n = n_voxels; n >= 1; n /= 8) words += (n + 31) / 32;
    return 4 * words + 64;
}

int lvx_shade(const uint32_t *base, const double *mips, int res, const uint32_t *vis_list,
              const double *dirs_host, int n_dirs, double tan_ao, const double *light_host, double tan_shadow,
              float *ao, float *shadow, int fill_ones, const uint32_t *nz_bits, void *scratch, void *stream) {
    if (!pow2(res) || n_dirs < 1 || n_dirs > 15) return LVX_E_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t V = (int64_t)res * res * res;
    ShadeParams P;
    for (int c = 0; c < n_dirs; c++)
        for (int a = 0; a < 3; a++) P.dirs[c][a] = dirs_host[3 * c + a];
    for (int a = 0; a < 3; a++) P.shadow_dir[a] = -light_host[a];   // lv/shading.py:154-155
    for (int c = 0; c < 15; c++)
        for (int a = 0; a < 3; a++) P.inv_dirs[c][a] = (c < n_dirs && P.dirs[c][a] != 0.0) ? 1.0 / P.dirs[c][a] : 0.0;
    for (int a = 0; a < 3; a++) P.inv_shadow[a] = P.shadow_dir[a] != 0.0 ? 1.0 / P.shadow_dir[a] : 0.0;
    P.tan_ao = tan_ao; P.tan_shadow = tan_shadow; P.w = 1.0 / n_dirs;
    const LevelOffsets L = make_level_offsets(res);
    uint32_t mw = 0;
    for (int l = 0; l < 16; l++) {
        P.mip_off[l] = (l >= 1 && l < L.n_levels) ? (uint32_t)(L.off[l] - L.off[1]) : 0;
        P.mask_off[l] = mw;
        if (l < L.n_levels) mw += (uint32_t)((L.off[l + 1] - L.off[l] + 31) / 32);
    }
    P.n_dirs = n_dirs; P.res = res; P.n_levels = L.n_levels;
    if (!vis_list || V < 4) return LVX_E_ARG;
    uint32_t *masks = (uint32_t *)scratch;
    for (int l = 0; l < L.n_levels; l++) {
        const int rl = res >> l;
        if (l == 0 && nz_bits && rl >= 32) {
            k_nzmask_bits<<<blocks_for((int64_t)(rl >> 5) * rl * rl, 256), 256, 0, s>>>(nz_bits, rl, masks + P.mask_off[0]);
            continue;
        }
        if (l >= 1 && rl <= 16) {     // this level and everything above it: one launch
            NzTail T;
            for (int k = 0; k < 16; k++) { T.mip_off[k] = P.mip_off[k]; T.mask_off[k] = P.mask_off[k]; }
            T.first = l; T.n_levels = L.n_levels; T.res = res;
            k_nzmask_tail<<<1, 1024, 0, s>>>(mips, T, masks);
            break;
        }
        k_nzmask<<<blocks_for((int64_t)rl * rl * rl, 256), 256, 0, s>>>(base, mips + P.mip_off[l], l, rl,
                                                                       masks + P.mask_off[l]);
    }
    if (fill_ones) k_shade_fill<<<blocks_for(V / 4, 256), 256, 0, s>>>(V / 4, (float4 *)ao, (float4 *)shadow);
    // persistent grid-stride launch: 148 SMs x 16 CTAs of 128 threads
    unsigned nb = 148 * 16;
    const unsigned need = blocks_for(V, 128);
    if (nb > need) nb = need;
    k_shade<<<nb, 128, 0, s>>>(base, mips, masks, P, vis_list, ao, shadow);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

}  // extern "C"
