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
    double tan_ao, tan_shadow, w;
    int64_t mip_off[16];    // element offset of level l (l >= 1) inside `mips`
    int n_dirs, res, n_levels;
};

// lv/shading.py:72-109; level 0 is read straight from the packed base words
__device__ __forceinline__ double trilinear(const uint32_t *__restrict__ base, const double *__restrict__ mips,
                                            const ShadeParams &P, int l, double px, double py, double pz) {
    const int rl = P.res >> l;
    const double scale = 1.0 / (double)(1 << l);
    const double ux = px * scale - 0.5, uy = py * scale - 0.5, uz = pz * scale - 0.5;
    const int ix = (int)floor(ux), iy = (int)floor(uy), iz = (int)floor(uz);
    const double fx = ux - ix, fy = uy - iy, fz = uz - iz;
    const double *lvl = mips + P.mip_off[l];
    double acc = 0.0;
#pragma unroll
    for (int dz = 0; dz < 2; dz++) {
        const int z = min(max(iz + dz, 0), rl - 1);
        const double wz = dz ? fz : 1.0 - fz;
#pragma unroll
        for (int dy = 0; dy < 2; dy++) {
            const int y = min(max(iy + dy, 0), rl - 1);
            const double wy = dy ? fy : 1.0 - fy;
#pragma unroll
            for (int dx = 0; dx < 2; dx++) {
                const int x = min(max(ix + dx, 0), rl - 1);
                const double wx = dx ? fx : 1.0 - fx;
                const int64_t idx = x + (int64_t)rl * (y + (int64_t)rl * z);
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
                                             const ShadeParams &P, double ox, double oy, double oz,
                                             double dx, double dy, double dz, double tan_half) {
    const double R = (double)P.res;
    if (ox < 0.0 || oy < 0.0 || oz < 0.0 || ox > R || oy > R || oz > R) return 0.0;
    double occ = 0.0, t = 1.0;
    while (occ < 0.99) {
        const double px = ox + dx * t, py = oy + dy * t, pz = oz + dz * t;
        if (px < 0.0 || py < 0.0 || pz < 0.0 || px > R || py > R || pz > R) break;
        const double diam = 2.0 * t * tan_half;
        const double step = diam > 1.0 ? diam : 1.0;
        // floor(log2(step)), step >= 1: the unbiased exponent
        int l = (int)((__double_as_longlong(step) >> 52) & 0x7ff) - 1023;
        if (l > P.n_levels - 1) l = P.n_levels - 1;
        const double s = trilinear(base, mips, P, l, px, py, pz);
        occ = occ + (1.0 - occ) * s;
        t += step;
    }
    return occ < 1.0 ? occ : 1.0;
}

// ao = shadow = 1 everywhere (lv/shading.py:177-178) + compaction of the visible voxels
__global__ void __launch_bounds__(256)
k_shade_prepare(const uint8_t *__restrict__ visible, int64_t V, float *__restrict__ ao, float *__restrict__ shadow,
                uint32_t *__restrict__ list, unsigned long long *__restrict__ list_n) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const bool v = idx < V && visible[idx] != 0;
    if (idx < V) { ao[idx] = 1.0f; shadow[idx] = 1.0f; }
    const uint32_t m = __ballot_sync(0xffffffffu, v);
    if (!m) return;
    unsigned long long b = 0;
    if (lane == 0) b = atomicAdd(list_n, (unsigned long long)__popc(m));
    b = __shfl_sync(0xffffffffu, b, 0);
    if (v) list[b + __popc(m & ((1u << lane) - 1u))] = (uint32_t)idx;
}

// One thread per visible voxel; a warp holds 32 consecutive entries of the compacted list, i.e.
// (mostly) x-adjacent voxels.  All lanes march the SAME cone direction in lock step: t, step and
// the mip level depend only on t, so the loop is convergent and the 8 trilinear taps of the 32
// lanes fall on consecutive addresses (or the same address at coarse levels) -- a few L1
// wavefronts per load instead of one per lane.  The 12 AO cones are folded in cone order in a
// register (lv/shading.py:150-152), so the f64 sum has the reference's rounding.
__global__ void __launch_bounds__(128)
k_shade(const uint32_t *__restrict__ base, const double *__restrict__ mips, const ShadeParams P,
        const uint32_t *__restrict__ list, const unsigned long long *__restrict__ list_n,
        float *__restrict__ ao, float *__restrict__ shadow) {
    const int64_t n = (int64_t)*list_n;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += stride) {
        const int64_t idx = list[e];
        const int x = (int)(idx % P.res), y = (int)((idx / P.res) % P.res), z = (int)(idx / ((int64_t)P.res * P.res));
        const double ox = x + 0.5, oy = y + 0.5, oz = z + 0.5;
        double acc = 0.0;
        for (int c = 0; c < P.n_dirs; c++)
            acc += P.w * cone_trace(base, mips, P, ox, oy, oz, P.dirs[c][0], P.dirs[c][1], P.dirs[c][2], P.tan_ao);
        const double sh = cone_trace(base, mips, P, ox, oy, oz, P.shadow_dir[0], P.shadow_dir[1], P.shadow_dir[2],
                                     P.tan_shadow);
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

int64_t lvx_shade_scratch_bytes(int64_t n_voxels) { return 4 * n_voxels + 64; }

int lvx_shade(const uint32_t *base, const double *mips, int res, const uint8_t *visible,
              const double *dirs_host, int n_dirs, double tan_ao, const double *light_host, double tan_shadow,
              float *ao, float *shadow, void *scratch, void *stream) {
    if (!pow2(res) || n_dirs < 1 || n_dirs > 15) return LVX_E_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t V = (int64_t)res * res * res;
    ShadeParams P;
    for (int c = 0; c < n_dirs; c++)
        for (int a = 0; a < 3; a++) P.dirs[c][a] = dirs_host[3 * c + a];
    for (int a = 0; a < 3; a++) P.shadow_dir[a] = -light_host[a];   // lv/shading.py:154-155
    P.tan_ao = tan_ao; P.tan_shadow = tan_shadow; P.w = 1.0 / n_dirs;
    const LevelOffsets L = make_level_offsets(res);
    for (int l = 0; l < 16; l++) P.mip_off[l] = (l >= 1 && l < L.n_levels) ? L.off[l] - L.off[1] : 0;
    P.n_dirs = n_dirs; P.res = res; P.n_levels = L.n_levels;
    unsigned long long *list_n = (unsigned long long *)scratch;
    uint32_t *list = (uint32_t *)((char *)scratch + 64);
    LVX_CUDA(cudaMemsetAsync(list_n, 0, 8, s));
    k_shade_prepare<<<blocks_for(V, 256), 256, 0, s>>>(visible, V, ao, shadow, list, list_n);
    // persistent grid-stride launch: 148 SMs x 16 CTAs of 128 threads
    unsigned nb = 148 * 16;
    const unsigned need = blocks_for(V, 128);
    if (nb > need) nb = need;
    k_shade<<<nb, 128, 0, s>>>(base, mips, P, list, list_n, ao, shadow);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

}  // extern "C"
