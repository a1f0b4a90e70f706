// voxelize.cu -- conservative capsule voxelization into the packed (count<<16 | occ_q) grid,
// and the occupancy pyramid.  Replaces lv/voxelizer.py:301-340 (_voxelize_kernel), the
// saturating merge at 490-495 and build_mips at 422-432.
//
// Accumulation.  The reference result per voxel is
//   (min(sum 1, 0xFFFF) << 16) | min(sum q, 0xFFFF).
// Fast path: ONE 32-bit atomicAdd of (1<<16)+q per incidence.  The add returns the old word, so
// the single thread whose add carries out of the low field sees it ((old&0xFFFF)+q > 0xFFFF),
// takes the carry back out of the count field and flags the voxel in a 1-bit "occupancy
// saturated" mask; lvx_finalize_base then writes 0xFFFF into flagged low fields.  A wrap of the
// whole word (>= 65536 segments in one voxel) raises LVX_ST_NEED_WIDE and the caller re-runs
// the exact 64-bit path (lvx_voxelize_wide + lvx_pack_wide).  The grid stays 4 B/voxel, so a
// 256^3 grid (64 MiB) is L2-resident on B200 while the atomics run.
#include "lvx_device.cuh"

#ifndef LVX_BATCH
#define LVX_BATCH 4   // cells of a traversal row whose atomics are issued back to back
#endif

namespace lvx {

#ifndef LVX_VOX_MINB
#define LVX_VOX_MINB 4
#endif
template <bool WIDE>
__global__ void __launch_bounds__(128, LVX_VOX_MINB)
k_voxelize(const double *__restrict__ verts, const double *__restrict__ normals,
           const int32_t *__restrict__ segs, int64_t seg_begin, int64_t seg_end, int use_clip,
           double r, double rt, double r_min, int res, int method,
           uint32_t *__restrict__ base, uint32_t *__restrict__ occ_sat,
           unsigned long long *__restrict__ wide, uint64_t *__restrict__ stats) {
    const int64_t si = seg_begin + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint64_t visited = 0;
    if (si < seg_end) {
        const int64_t i = segs[si];
        const Capsule c = load_capsule(verts, normals, i, r, use_clip != 0);
        const double rc = r > r_min ? r : r_min;     // lv/voxelizer.py:289-290
        const double ratio = r / rc;
        const double corr = ratio * ratio;
        const int64_t res64 = res;
        // About two thirds of the cells of the conservative traversal (radius rt = rc + 0.5 boxes)
        // have their centre farther than rc + 0.5 from the segment: there sdf >= 0.5, the clip terms
        // can only raise it, occ clamps to 0 and q = 0 exactly (lv/voxelizer.py:286-298, 328).  A
        // full-rate f32 distance with a 1e-3 relative + 1e-4 absolute margin proves that case, and
        // only the remaining cells pay for the f64 distance, square root and division.
        const SegF sf = make_segf(c.a, c.b);
        const float far2 = (float)((rc + 0.5) * (rc + 0.5)) * 1.001f + 1e-4f;
        // rows of the traversal, four cells at a time: four occupancies, then the four atomics
        // back to back, then the (rare) carry repairs that depend on their results
        for_each_row(method, c.a, c.b, rt, res, [&](int x, int y, int z, int axis, int len) {
            const int64_t stride = axis == 0 ? 1 : (axis == 1 ? res64 : res64 * res64);
            const int64_t idx0 = x + res64 * (y + res64 * z);
            const double sx = axis == 0 ? 1.0 : 0.0, sy = axis == 1 ? 1.0 : 0.0, sz = axis == 2 ? 1.0 : 0.0;
            const float fx = (float)(x - sf.ox) + 0.5f, fy = (float)(y - sf.oy) + 0.5f, fz = (float)(z - sf.oz) + 0.5f;
            visited += (uint64_t)len;
            for (int u0 = 0; u0 < len; u0 += LVX_BATCH) {
                uint32_t q[LVX_BATCH], old[LVX_BATCH];
#pragma unroll
                for (int k = 0; k < LVX_BATCH; k++) {
                    const int u = u0 + k;
                    q[k] = 0u;
                    if (u < len && !(segf_dist2(sf, fx + (float)u * (float)sx, fy + (float)u * (float)sy, fz + (float)u * (float)sz) > far2))
                        q[k] = occupancy_q(x + 0.5 + u * sx, y + 0.5 + u * sy, z + 0.5 + u * sz, c, rc, corr);
                }
                if (WIDE) {
#pragma unroll
                    for (int k = 0; k < LVX_BATCH; k++)
                        if (u0 + k < len) atomicAdd(&wide[idx0 + (u0 + k) * stride], (1ull << 32) | (unsigned long long)q[k]);
                } else {
#pragma unroll
                    for (int k = 0; k < LVX_BATCH; k++)
                        old[k] = u0 + k < len ? atomicAdd(&base[idx0 + (u0 + k) * stride], 0x10000u + q[k]) : 0u;
#pragma unroll
                    for (int k = 0; k < LVX_BATCH; k++) {
                        if (u0 + k >= len) continue;
                        const uint32_t inc = 0x10000u + q[k];
                        const int64_t idx = idx0 + (u0 + k) * stride;
                        if (old[k] + inc < old[k]) stats[LVX_ST_NEED_WIDE] = 1;   // count field wrapped
                        if ((old[k] & 0xFFFFu) + q[k] > 0xFFFFu) {
                            atomicSub(&base[idx], 0x10000u);                  // undo the carry into count
                            atomicOr(&occ_sat[idx >> 5], 1u << (idx & 31));
                        }
                    }
                }
            }
        });
    }
    visited = warp_sum_u64(visited);
    if ((threadIdx.x & 31) == 0 && visited)
        atomicAdd((unsigned long long *)&stats[LVX_ST_VISITED], (unsigned long long)visited);
}

__global__ void __launch_bounds__(256)
k_finalize_base(uint32_t *__restrict__ base, const uint32_t *__restrict__ occ_sat, int64_t n_words,
                uint64_t *__restrict__ stats) {
    // one thread per 32-voxel mask word; flagged voxels are rare
    const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= n_words) return;
    uint32_t m = occ_sat[w];
    if (!m) return;
    atomicAdd((unsigned long long *)&stats[LVX_ST_OCC_SAT], (unsigned long long)__popc(m));
    while (m) {
        const int b = __ffs(m) - 1;
        m &= m - 1;
        base[w * 32 + b] |= 0xFFFFu;
    }
}

__global__ void __launch_bounds__(256)
k_widen(const uint32_t *__restrict__ base, const uint32_t *__restrict__ occ_sat, int64_t n,
        unsigned long long *__restrict__ wide) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t w = base[i];
    uint32_t lo = w & 0xFFFFu;
    if (occ_sat && ((occ_sat[i >> 5] >> (i & 31)) & 1u)) lo = 0xFFFFu;
    wide[i] = ((unsigned long long)(w >> 16) << 32) | lo;
}

// Largest count and largest occupancy sum of a rank's accumulators (multi-GPU exchange: the sums of these maxima
// over the ranks bound every field of the merged grid; below 2^16 the packed 4-byte words can be summed instead
// of the 8-byte accumulators).  Four accumulators per thread (two 128-bit loads), grid-stride.
__global__ void __launch_bounds__(256)
k_wide_field_max(const unsigned long long *__restrict__ wide, int64_t n, unsigned long long *__restrict__ out2,
                 uint32_t *__restrict__ packed) {
    // `packed` (optional): the packed words (count << 16 | occ, fields clamped) are written in the same pass -- the
    // exchange needs them exactly when the maxima allow the packed path, and one read of the accumulators serves both
    unsigned long long mc = 0, mo = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * 4;
    auto pk = [](unsigned long long w) {
        const unsigned long long c = w >> 32, o = w & 0xFFFFFFFFull;
        return (uint32_t)((min(c, 0xFFFFull) << 16) | min(o, 0xFFFFull));
    };
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; i < n; i += stride) {
        if (i + 3 < n) {
            const ulonglong2 a = *reinterpret_cast<const ulonglong2 *>(wide + i), b = *reinterpret_cast<const ulonglong2 *>(wide + i + 2);
            mc = max(max(mc, a.x >> 32), max(max(a.y >> 32, b.x >> 32), b.y >> 32));
            mo = max(max(mo, a.x & 0xFFFFFFFFull), max(max(a.y & 0xFFFFFFFFull, b.x & 0xFFFFFFFFull), b.y & 0xFFFFFFFFull));
            if (packed) *reinterpret_cast<uint4 *>(packed + i) = make_uint4(pk(a.x), pk(a.y), pk(b.x), pk(b.y));
        } else {
            for (int64_t j = i; j < n; j++) {
                mc = max(mc, wide[j] >> 32); mo = max(mo, wide[j] & 0xFFFFFFFFull);
                if (packed) packed[j] = pk(wide[j]);
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mc = max(mc, __shfl_xor_sync(0xffffffffu, mc, o));
        mo = max(mo, __shfl_xor_sync(0xffffffffu, mo, o));
    }
    if ((threadIdx.x & 31) == 0) {
        if (mc) atomicMax(&out2[0], mc);
        if (mo) atomicMax(&out2[1], mo);
    }
}

__global__ void __launch_bounds__(256)
k_pack_wide(const unsigned long long *__restrict__ wide, int64_t n, uint32_t *__restrict__ base,
            uint32_t *__restrict__ nz_bits, uint64_t *__restrict__ stats) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint64_t sat = 0;
    bool nz = false;
    if (i < n) {
        const unsigned long long w = wide[i];
        uint64_t c = w >> 32, o = w & 0xFFFFFFFFull;
        if (c > 0xFFFF) { sat = c - 0xFFFF; c = 0xFFFF; }   // lv/voxelizer.py:333-336, 493
        if (o > 0xFFFF) o = 0xFFFF;                          // lv/voxelizer.py:494
        base[i] = (uint32_t)((c << 16) | o);
        nz = o != 0;
    }
    // one bit per voxel "level-0 occupancy is non-zero" (32 x-adjacent voxels per word): the cone
    // tracer's level-0 footprint masks are built from these bits instead of re-reading `base`
    const uint32_t m = __ballot_sync(0xffffffffu, nz);
    if (nz_bits && (threadIdx.x & 31) == 0 && i < n) nz_bits[i >> 5] = m;
    sat = warp_sum_u64(sat);
    if ((threadIdx.x & 31) == 0 && sat)
        atomicAdd((unsigned long long *)&stats[LVX_ST_SATURATED], (unsigned long long)sat);
}

// Pack + level 1 of the pyramid in one read of the accumulators (res >= 64).  One thread per level-1
// cell: its 2x2x2 children are four 16-byte loads (two x-adjacent accumulators each; a warp reads 512
// contiguous bytes per row), four 8-byte stores of packed words, one f64 store of the parent.  The
// "occupancy non-zero" bits of a row's 64 voxels are two ballots interleaved by lanes 0 and 16.
__device__ __forceinline__ uint32_t spread16(uint32_t x) {     // bit k -> bit 2k
    x = (x | (x << 8)) & 0x00FF00FFu;
    x = (x | (x << 4)) & 0x0F0F0F0Fu;
    x = (x | (x << 2)) & 0x33333333u;
    x = (x | (x << 1)) & 0x55555555u;
    return x;
}
__global__ void __launch_bounds__(256)
k_pack_mip1(const ulonglong2 *__restrict__ wide2, int res, uint32_t *__restrict__ base, uint32_t *__restrict__ nz_bits,
            double *__restrict__ mip1, uint64_t *__restrict__ stats) {
    const int rl = res >> 1;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;    // rl^3 is a multiple of the block size
    const int lane = threadIdx.x & 31;
    const int x = (int)(i % rl), y = (int)((i / rl) % rl), z = (int)(i / ((int64_t)rl * rl));
    ulonglong2 w[4];
#pragma unroll
    for (int k = 0; k < 4; k++)
        w[k] = wide2[(2 * x + (int64_t)res * ((2 * y + (k & 1)) + (int64_t)res * (2 * z + (k >> 1)))) >> 1];
    uint64_t sat = 0;
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < 4; k++) {
        const int64_t v = 2 * x + (int64_t)res * ((2 * y + (k & 1)) + (int64_t)res * (2 * z + (k >> 1)));
        uint64_t c0 = w[k].x >> 32, o0 = w[k].x & 0xFFFFFFFFull, c1 = w[k].y >> 32, o1 = w[k].y & 0xFFFFFFFFull;
        if (c0 > 0xFFFF) { sat += c0 - 0xFFFF; c0 = 0xFFFF; }     // lv/voxelizer.py:333-336, 493
        if (c1 > 0xFFFF) { sat += c1 - 0xFFFF; c1 = 0xFFFF; }
        if (o0 > 0xFFFF) o0 = 0xFFFF;                              // lv/voxelizer.py:494
        if (o1 > 0xFFFF) o1 = 0xFFFF;
        *reinterpret_cast<uint2 *>(base + v) = make_uint2((uint32_t)((c0 << 16) | o0), (uint32_t)((c1 << 16) | o1));
        s += min((uint32_t)o0, 4096u) + min((uint32_t)o1, 4096u);   // lv/voxelizer.py:496
        const uint32_t be = __ballot_sync(0xffffffffu, o0 != 0), bo = __ballot_sync(0xffffffffu, o1 != 0);
        if (nz_bits && (lane & 15) == 0)
            nz_bits[v >> 5] = spread16((be >> lane) & 0xFFFFu) | (spread16((bo >> lane) & 0xFFFFu) << 1);
    }
    mip1[i] = (double)s * (1.0 / 32768.0);   // (sum / 4096) / 8, exact
    sat = warp_sum_u64(sat);
    if (lane == 0 && sat) atomicAdd((unsigned long long *)&stats[LVX_ST_SATURATED], (unsigned long long)sat);
}

// ----------------------------------------------------------------------------- mips
// Level sums are exact dyadic rationals (multiples of 2^-(12+3l) below 2^53 ulps), so any
// summation order gives the reference's bits.

__device__ __forceinline__ double occ0(uint32_t w) {
    const uint32_t q = min(w & 0xFFFFu, 4096u);      // lv/voxelizer.py:496
    return (double)q * (1.0 / 4096.0);
}

// Level 1 of the pyramid and the "occupancy non-zero" bits from a PACKED grid (the merged grid of a packed multi-GPU
// exchange): k_pack_mip1 without the pack.  One thread per level-1 cell, 8-byte loads of x-adjacent children.
__global__ void __launch_bounds__(256)
k_base_mip1(const uint32_t *__restrict__ base, int res, uint32_t *__restrict__ nz_bits, double *__restrict__ mip1) {
    const int rl = res >> 1;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;    // rl^3 is a multiple of the block size
    const int lane = threadIdx.x & 31;
    const int x = (int)(i % rl), y = (int)((i / rl) % rl), z = (int)(i / ((int64_t)rl * rl));
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < 4; k++) {
        const int64_t v = 2 * x + (int64_t)res * ((2 * y + (k & 1)) + (int64_t)res * (2 * z + (k >> 1)));
        const uint2 w = *reinterpret_cast<const uint2 *>(base + v);
        const uint32_t o0 = w.x & 0xFFFFu, o1 = w.y & 0xFFFFu;
        s += min(o0, 4096u) + min(o1, 4096u);                               // lv/voxelizer.py:496
        const uint32_t be = __ballot_sync(0xffffffffu, o0 != 0), bo = __ballot_sync(0xffffffffu, o1 != 0);
        if (nz_bits && (lane & 15) == 0)
            nz_bits[v >> 5] = spread16((be >> lane) & 0xFFFFu) | (spread16((bo >> lane) & 0xFFFFu) << 1);
    }
    mip1[i] = (double)s * (1.0 / 32768.0);   // (sum / 4096) / 8, exact
}

// level 1 from the packed base: one thread per parent, 8-byte loads of x-adjacent children
__global__ void __launch_bounds__(256)
k_mip1(const uint32_t *__restrict__ base, int res, double *__restrict__ out) {
    const int rl = res >> 1;
    const int64_t n = (int64_t)rl * rl * rl;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int x = (int)(i % rl), y = (int)((i / rl) % rl), z = (int)(i / ((int64_t)rl * rl));
    uint32_t s = 0;
#pragma unroll
    for (int dz = 0; dz < 2; dz++)
#pragma unroll
        for (int dy = 0; dy < 2; dy++) {
            const uint2 w = *reinterpret_cast<const uint2 *>(
                base + (2 * x + (int64_t)res * ((2 * y + dy) + (int64_t)res * (2 * z + dz))));
            s += min(w.x & 0xFFFFu, 4096u) + min(w.y & 0xFFFFu, 4096u);
        }
    out[i] = (double)s * (1.0 / 32768.0);   // (sum / 4096) / 8, exact
}

__global__ void __launch_bounds__(256)
k_mip_next(const double *__restrict__ src, int rsrc, double *__restrict__ out) {
    const int rl = rsrc >> 1;
    const int64_t n = (int64_t)rl * rl * rl;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int x = (int)(i % rl), y = (int)((i / rl) % rl), z = (int)(i / ((int64_t)rl * rl));
    double s = 0.0;
#pragma unroll
    for (int dz = 0; dz < 2; dz++)
#pragma unroll
        for (int dy = 0; dy < 2; dy++) {
            const double2 w = *reinterpret_cast<const double2 *>(
                src + (2 * x + (int64_t)rsrc * ((2 * y + dy) + (int64_t)rsrc * (2 * z + dz))));
            s += w.x + w.y;
        }
    out[i] = s * 0.125;
}

// The top of the pyramid (levels of <= 16^3 nodes) in ONE launch: a single CTA builds level after
// level with a block barrier in between, instead of one tiny launch per level.
struct MipTail { int64_t off[16]; int first, n_levels, res; };   // off[l] = element offset of level l inside `mips`
__global__ void __launch_bounds__(1024)
k_mip_tail(double *__restrict__ mips, const MipTail T) {
    for (int l = T.first; l < T.n_levels; l++) {
        const int rsrc = T.res >> (l - 1), rl = T.res >> l;
        const double *src = mips + T.off[l - 1];
        double *out = mips + T.off[l];
        for (int i = threadIdx.x; i < rl * rl * rl; i += blockDim.x) {
            const int x = i % rl, y = (i / rl) % rl, z = i / (rl * rl);
            double s = 0.0;
#pragma unroll
            for (int dz = 0; dz < 2; dz++)
#pragma unroll
                for (int dy = 0; dy < 2; dy++) {
                    const double2 w = *reinterpret_cast<const double2 *>(src + (2 * x + rsrc * ((2 * y + dy) + rsrc * (2 * z + dz))));
                    s += w.x + w.y;
                }
            out[i] = s * 0.125;
        }
        __syncthreads();
    }
}

}  // namespace lvx

using namespace lvx;

extern "C" {

static int voxelize_common(bool wide_path, const double *verts, const double *normals, const int32_t *segs,
                           int64_t seg_begin, int64_t seg_end, int use_clip, double r, double rt,
                           double r_min, int res, int method, uint32_t *base, uint32_t *occ_sat,
                           uint64_t *wide, uint64_t *stats, void *stream) {
    if (!pow2(res) || res > 1024 || method < 0 || method > 2 || !(r_min > 0) || seg_end < seg_begin)
        return LVX_E_ARG;
    const int64_t n = seg_end - seg_begin;
    if (n == 0) return LVX_OK;
    const unsigned nb = blocks_for(n, 128);
    cudaStream_t s = (cudaStream_t)stream;
    if (wide_path)
        k_voxelize<true><<<nb, 128, 0, s>>>(verts, normals, segs, seg_begin, seg_end, use_clip, r, rt, r_min,
                                            res, method, nullptr, nullptr, (unsigned long long *)wide, stats);
    else
        k_voxelize<false><<<nb, 128, 0, s>>>(verts, normals, segs, seg_begin, seg_end, use_clip, r, rt, r_min,
                                             res, method, base, occ_sat, nullptr, stats);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

int lvx_voxelize(const double *verts, const double *normals, const int32_t *segs, int64_t seg_begin,
                 int64_t seg_end, int use_clip, double r, double rt, double r_min, int res, int method,
                 uint32_t *base, uint32_t *occ_sat, uint64_t *stats, void *stream) {
    return voxelize_common(false, verts, normals, segs, seg_begin, seg_end, use_clip, r, rt, r_min, res,
                           method, base, occ_sat, nullptr, stats, stream);
}

int lvx_voxelize_wide(const double *verts, const double *normals, const int32_t *segs, int64_t seg_begin,
                      int64_t seg_end, int use_clip, double r, double rt, double r_min, int res, int method,
                      uint64_t *wide, uint64_t *stats, void *stream) {
    return voxelize_common(true, verts, normals, segs, seg_begin, seg_end, use_clip, r, rt, r_min, res,
                           method, nullptr, nullptr, wide, stats, stream);
}

int lvx_widen(const uint32_t *base, const uint32_t *occ_sat, int64_t n_voxels, uint64_t *wide, void *stream) {
    k_widen<<<blocks_for(n_voxels, 256), 256, 0, (cudaStream_t)stream>>>(base, occ_sat, n_voxels,
                                                                        (unsigned long long *)wide);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

int lvx_wide_field_max(const uint64_t *wide, int64_t n_voxels, uint64_t *out2, uint32_t *packed, void *stream) {
    if (!wide || !out2 || n_voxels <= 0 || (reinterpret_cast<uintptr_t>(wide) & 15) || (reinterpret_cast<uintptr_t>(packed) & 15))
        return LVX_E_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    LVX_CUDA(cudaMemsetAsync(out2, 0, 16, s));
    unsigned nb = blocks_for((n_voxels + 3) / 4, 256);
    if (nb > 148 * 8) nb = 148 * 8;
    k_wide_field_max<<<nb, 256, 0, s>>>((const unsigned long long *)wide, n_voxels, (unsigned long long *)out2, packed);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

int lvx_base_mip1(const uint32_t *base, int res, uint32_t *nz_bits, double *mips, void *stream) {
    if (!pow2(res) || res < 64 || !base || !mips) return LVX_E_ARG;
    const int rl = res >> 1;
    k_base_mip1<<<blocks_for((int64_t)rl * rl * rl, 256), 256, 0, (cudaStream_t)stream>>>(base, res, nz_bits, mips);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

int lvx_pack_wide(const uint64_t *wide, int64_t n_voxels, uint32_t *base, uint32_t *nz_bits, uint64_t *stats, void *stream) {
    if (nz_bits && (n_voxels & 31)) return LVX_E_ARG;
    k_pack_wide<<<blocks_for(n_voxels, 256), 256, 0, (cudaStream_t)stream>>>(
        (const unsigned long long *)wide, n_voxels, base, nz_bits, stats);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

int lvx_finalize_base(uint32_t *base, const uint32_t *occ_sat, int64_t n_voxels, uint64_t *stats, void *stream) {
    const int64_t n_words = (n_voxels + 31) / 32;
    k_finalize_base<<<blocks_for(n_words, 256), 256, 0, (cudaStream_t)stream>>>(base, occ_sat, n_words, stats);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

int lvx_pack_wide_mip1(const uint64_t *wide, int res, uint32_t *base, uint32_t *nz_bits, double *mips,
                       uint64_t *stats, void *stream) {
    if (!pow2(res) || res < 64 || !mips) return LVX_E_ARG;
    const int rl = res >> 1;
    k_pack_mip1<<<blocks_for((int64_t)rl * rl * rl, 256), 256, 0, (cudaStream_t)stream>>>(
        (const ulonglong2 *)wide, res, base, nz_bits, mips, stats);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

static int build_mips_from(const uint32_t *base, int res, double *mips, void *stream) {
    if (!pow2(res)) return LVX_E_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    const LevelOffsets L = make_level_offsets(res);
    const int64_t V = L.off[1];
    if (base) {
        const int rl = res >> 1;
        k_mip1<<<blocks_for((int64_t)rl * rl * rl, 256), 256, 0, s>>>(base, res, mips);
    }
    for (int l = 2; l < L.n_levels; l++) {
        const int rsrc = res >> (l - 1), rl = res >> l;
        if (rl <= 16) {     // this level and everything above it: one launch
            MipTail T;
            for (int k = 0; k < 16; k++) T.off[k] = (k >= 1 && k < L.n_levels) ? L.off[k] - V : 0;
            T.first = l; T.n_levels = L.n_levels; T.res = res;
            k_mip_tail<<<1, 1024, 0, s>>>(mips, T);
            break;
        }
        k_mip_next<<<blocks_for((int64_t)rl * rl * rl, 256), 256, 0, s>>>(mips + (L.off[l - 1] - V), rsrc,
                                                                        mips + (L.off[l] - V));
    }
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

int lvx_build_mips(const uint32_t *base, int res, double *mips, void *stream) {
    if (!base) return LVX_E_ARG;
    return build_mips_from(base, res, mips, stream);
}

int lvx_build_mips_upper(int res, double *mips, void *stream) { return build_mips_from(nullptr, res, mips, stream); }

}  // extern "C"
