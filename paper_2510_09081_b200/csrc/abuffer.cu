// abuffer.cu -- per-frame acceleration structure: per-voxel segment lists restricted to visible
// voxels.  Replaces lv/abuffer.py:104-114 (scan_offsets) and 195-255, 281-328 (_chunk_count_kernel,
// _write_kernel, _second_pass).
//
//   count (already in base>>16)  ->  single-pass decoupled-look-back scan  ->  scatter with an
//   atomic cursor  ->  per-voxel ordering pass.
// The reference's per-chunk cursors make every list ascending in segment index
// (lv/abuffer.py:313-317; pinned by its tests, test_abuffer.py:114-122).  A segment visits a voxel
// at most once, so sorting each list reproduces the reference's `fragments` array bit for bit
// (SURVEY.md §7 H2).  The reference's extra counting traversal (_chunk_count_kernel) exists only
// to rebuild deterministic cursors and to assert determinism; here the assertion is the
// cursor==end check in the ordering pass (LVX_ST_MISMATCH -> ABufferError on the host).
//
// Loose bits.  A list holds every segment whose TRAVERSAL footprint (radius rt = max(r,r_min)+0.5)
// covers the voxel, ~5x more than the capsules (radius r) that really reach into it.  A ray hit is
// only accepted when the hit point lies inside the voxel being visited (lv/raytracer.py:446-452),
// and every surface point _ray_capsule can return lies within r + 3.2e-5 of the segment, so a
// fragment whose segment is provably farther than r_tight = r + 1e-3 from the voxel's cube can never
// yield an accepted hit there.  The scatter pass has the segment in registers and proves this per
// incidence with a separating-direction lower bound (f32, ~70 flops); the flag rides through the
// ordering pass in bit 0 of the packed word, and the ordering pass -- which holds every sorted list
// in registers anyway -- writes a TIGHT INDEX next to the reference's array: the list's tight
// fragments compacted to the front of the list's own range in `tfrags` (segment ids) and `tslot`
// (their slots in the full list, which the transparency keys need), and their number in
// `tcnt[voxel]`.  The ray tracer enumerates contiguous ranges of that index instead of scanning
// bit masks.  `frags` itself stays the reference's array, bit for bit.
#include "lvx_device.cuh"

#ifndef LVX_BATCH
#define LVX_BATCH 4   // cells of a traversal row whose atomics are issued back to back
#endif

// cursor value of a culled voxel: far above any fragment capacity (see k_scatter)
#define LVX_CURSOR_CULLED 0xF0000000u

namespace lvx {

// ----------------------------------------------------------------------------- scan
// Tile shape, measured on B200 (scan stage at 256^3 / 512^3, offsets + cursors written): 512 x 8: 0.066 / 0.434 ms,
// 1024 x 8: 0.070 / 0.452, 512 x 16: 0.075 / 0.510, 256 x 16: 0.070 / 0.461, 256 x 8: 0.064 / 0.415, 128 x 8: 0.065 / 0.432,
// 128 x 12: 0.062 / 0.393, 128 x 16: 0.063 / 0.394, 128 x 20: 0.081 / 0.530, 64 x 16: - / 0.428.  Small CTAs: while warp 0
// of a tile looks back, the tile's other warps idle, and 16 tiles per SM overlap that better than 4.
#ifndef LVX_SCAN_THREADS
#define LVX_SCAN_THREADS 128
#endif
#ifndef LVX_SCAN_ITEMS
#define LVX_SCAN_ITEMS 16       // voxels per thread, a multiple of 4 (128-bit loads and stores)
#endif
constexpr int SCAN_THREADS = LVX_SCAN_THREADS;
constexpr int SCAN_ITEMS = LVX_SCAN_ITEMS;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;
static_assert(SCAN_ITEMS % 4 == 0 && SCAN_ITEMS <= 32 && SCAN_THREADS % 32 == 0 && SCAN_THREADS <= 1024, "scan shape");
constexpr uint64_t FLAG_AGG = 1ull << 62, FLAG_INC = 2ull << 62, VAL_MASK = (1ull << 62) - 1;

__global__ void __launch_bounds__(SCAN_THREADS)
k_scan(const uint32_t *__restrict__ base, const uint8_t *__restrict__ cull, int64_t V,
       uint32_t *__restrict__ offsets, uint32_t *__restrict__ cursor, unsigned long long *__restrict__ state,
       uint64_t *__restrict__ stats) {
    __shared__ uint32_t s_tile;
    __shared__ uint32_t s_warp[SCAN_THREADS / 32];
    __shared__ uint64_t s_prefix;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // tiles are numbered in the order they start running, so a tile only ever waits for tiles
    // that are already resident (forward progress without co-residency assumptions)
    if (tid == 0) s_tile = (uint32_t)atomicAdd(&state[0], 1ull);
    __syncthreads();
    const int64_t tile = s_tile;
    unsigned long long *st = state + 1;
    const int64_t i0 = tile * SCAN_TILE + (int64_t)tid * SCAN_ITEMS;

    uint32_t c[SCAN_ITEMS];
    uint32_t culled = 0;       // bit k: voxel i0 + k is culled
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; k++) c[k] = 0;
    // V is a multiple of 8 but not necessarily of SCAN_ITEMS: groups of four voxels are all in or all out
#pragma unroll
    for (int q = 0; q < SCAN_ITEMS / 4; q++) {
        if (i0 + 4 * q < V) {
            const uint4 w = *reinterpret_cast<const uint4 *>(base + i0 + 4 * q);
            c[4 * q] = w.x >> 16; c[4 * q + 1] = w.y >> 16; c[4 * q + 2] = w.z >> 16; c[4 * q + 3] = w.w >> 16;
            if (cull) {   // lv/abuffer.py:107-108
                const uint32_t m = *reinterpret_cast<const uint32_t *>(cull + i0 + 4 * q);
#pragma unroll
                for (int k = 0; k < 4; k++)
                    if (((m >> (8 * k)) & 0xFFu) == 0) { c[4 * q + k] = 0; culled |= 1u << (4 * q + k); }
            }
        }
    }
    uint32_t tsum = 0;
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; k++) tsum += c[k];
    // block-level exclusive scan of the per-thread sums (max 16384*65535 < 2^32)
    uint32_t inc = tsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t n = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += n;
    }
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < SCAN_THREADS / 32 ? s_warp[lane] : 0;
        uint32_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t n = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += n;
        }
        if (lane < SCAN_THREADS / 32) s_warp[lane] = wi - w;   // exclusive warp prefix
        const uint64_t agg = __shfl_sync(0xffffffffu, wi, SCAN_THREADS / 32 - 1);
        uint64_t excl = 0;
        if (tile == 0) {
            if (lane == 0) atomicExch(&st[0], FLAG_INC | agg);
        } else {
            if (lane == 0) atomicExch(&st[tile], FLAG_AGG | agg);
            int64_t j = tile - 1;
            for (;;) {
                const int64_t jj = j - lane;
                uint64_t v = FLAG_INC;   // virtual tile -1: inclusive prefix 0
                if (jj >= 0) v = *reinterpret_cast<volatile unsigned long long *>(&st[jj]);
                const uint32_t flag = (uint32_t)(v >> 62);
                const uint32_t bal_inc = __ballot_sync(0xffffffffu, flag == 2);
                const uint32_t bal_inv = __ballot_sync(0xffffffffu, flag == 0);
                const int first_inc = bal_inc ? __ffs(bal_inc) - 1 : 32;
                const uint32_t need = first_inc >= 31 ? 0xffffffffu : ((2u << first_inc) - 1u);
                if (bal_inv & need) continue;   // a predecessor we need has not published yet
                uint64_t contrib = lane <= first_inc ? (v & VAL_MASK) : 0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) contrib += __shfl_xor_sync(0xffffffffu, contrib, o);
                excl += contrib;
                if (first_inc < 32) break;
                j -= 32;
            }
            if (lane == 0) atomicExch(&st[tile], FLAG_INC | ((excl + agg) & VAL_MASK));
        }
        if (lane == 0) {
            s_prefix = excl;
            if ((tile + 1) * SCAN_TILE >= V) {   // last tile: total
                offsets[V] = (uint32_t)(excl + agg);
                stats[LVX_ST_FRAG_TOTAL] = excl + agg;
            }
        }
    }
    __syncthreads();
    uint32_t run = (uint32_t)s_prefix + s_warp[warp] + (inc - tsum);
#pragma unroll
    for (int q = 0; q < SCAN_ITEMS / 4; q++) {
        uint32_t o[4];
#pragma unroll
        for (int k = 0; k < 4; k++) { o[k] = run; run += c[4 * q + k]; }
        if (i0 + 4 * q < V) {
            *reinterpret_cast<uint4 *>(offsets + i0 + 4 * q) = make_uint4(o[0], o[1], o[2], o[3]);
            if (cursor) {   // the scatter pass's cursors (see k_init_cursor): list start, or the parking value of a culled voxel
#pragma unroll
                for (int k = 0; k < 4; k++)
                    if ((culled >> (4 * q + k)) & 1u) o[k] = LVX_CURSOR_CULLED;
                *reinterpret_cast<uint4 *>(cursor + i0 + 4 * q) = make_uint4(o[0], o[1], o[2], o[3]);
            }
        }
    }
}

// ----------------------------------------------------------------------------- scatter
// lv/abuffer.py:226-255 _write_kernel.  The hierarchical segment rejection (_segment_visible,
// 145-181) is an acceleration only -- culled voxels are skipped per cell (252-253) -- so the
// output does not depend on it.
// Lower bound on the distance between segment [a, b] and the unit cube centred at the origin
// (a, b given relative to the cube centre).  Three rounds of alternating projections give a
// near-optimal separating direction n; for ANY n, dist >= (min(n.a, n.b) - max_cube n.y) / |n|.
// Returns true when that bound exceeds R, i.e. the capsule of radius R certainly misses the cube.
__device__ __forceinline__ bool segment_misses_cube(float ax, float ay, float az, float bx, float by, float bz, float R) {
    const float dx = bx - ax, dy = by - ay, dz = bz - az;
    const float dd = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
    const float inv = dd > 0.f ? __fdividef(1.f, dd) : 0.f;
    float qx = 0.f, qy = 0.f, qz = 0.f, px = ax, py = ay, pz = az;
#pragma unroll
    for (int it = 0; it < 3; it++) {
        float t = fmaf(qx - ax, dx, fmaf(qy - ay, dy, (qz - az) * dz)) * inv;
        t = fminf(fmaxf(t, 0.f), 1.f);
        px = fmaf(t, dx, ax); py = fmaf(t, dy, ay); pz = fmaf(t, dz, az);
        qx = fminf(fmaxf(px, -0.5f), 0.5f); qy = fminf(fmaxf(py, -0.5f), 0.5f); qz = fminf(fmaxf(pz, -0.5f), 0.5f);
    }
    const float nx = px - qx, ny = py - qy, nz = pz - qz;
    const float nn = fmaf(nx, nx, fmaf(ny, ny, nz * nz));
    if (!(nn > 0.f)) return false;                      // the segment touches the cube
    const float na = fmaf(nx, ax, fmaf(ny, ay, nz * az)), nb = fmaf(nx, bx, fmaf(ny, by, nz * bz));
    const float gap = fminf(na, nb) - 0.5f * (fabsf(nx) + fabsf(ny) + fabsf(nz));
    return gap > 0.f && gap * gap > R * R * nn;
}

// lv/abuffer.py:226-255 _write_kernel.  The hierarchical segment rejection (_segment_visible,
// 145-181) is an acceleration only -- culled voxels are skipped per cell (252-253) -- so the
// output does not depend on it.  Words are written as (segment << 1) | loose; the ordering pass
// strips the flag again.
// Culled voxels are not looked up: k_init_cursor parks their cursor at LVX_CURSOR_CULLED, far
// above any fragment capacity, so the position their atomic returns fails the capacity test and
// nothing is stored -- one dependent memory round trip per cell (the atomic) instead of two.
#ifndef LVX_SCAT_MINB
#define LVX_SCAT_MINB 1
#endif
// lv/abuffer.py:145-181 _segment_visible: does the segment's inflated voxel box
// floor(min - rt) .. floor(max + rt) overlap a set voxel of the culling pyramid?  The reference runs a
// depth-first search from the root; here the box is looked up at the finest level where it spans at
// most two nodes per axis (<= 8 byte loads from a level that is a few KiB..MiB and stays in L1/L2).
// The answer may be "yes" where the reference's exact search says "no" -- never the other way round --
// and the per-cell culled test below then skips every cell of such a segment, so `fragments` is the
// reference's array either way (the reference itself treats this test as an acceleration, 252-253).
struct PyrOffsets { uint32_t off[12]; int n_levels; };
__device__ __forceinline__ bool segment_visible(const uint8_t *__restrict__ flat, const PyrOffsets &O, int res,
                                                const d3 &a, const d3 &b, double rt) {
    int lo[3], hi[3];
    lo[0] = (int)floor(fmin(a.x, b.x) - rt); hi[0] = (int)floor(fmax(a.x, b.x) + rt);
    lo[1] = (int)floor(fmin(a.y, b.y) - rt); hi[1] = (int)floor(fmax(a.y, b.y) + rt);
    lo[2] = (int)floor(fmin(a.z, b.z) - rt); hi[2] = (int)floor(fmax(a.z, b.z) + rt);
#pragma unroll
    for (int k = 0; k < 3; k++) {
        lo[k] = max(lo[k], 0); hi[k] = min(hi[k], res - 1);
        if (hi[k] < lo[k]) return false;                  // entirely outside the grid: no cell at all
    }
    int l = 0;
    while (l < O.n_levels - 1 && (((hi[0] >> l) - (lo[0] >> l)) > 1 || ((hi[1] >> l) - (lo[1] >> l)) > 1 ||
                                  ((hi[2] >> l) - (lo[2] >> l)) > 1)) l++;
    const uint32_t rl = (uint32_t)res >> l;
    const uint8_t *lev = flat + O.off[l];
    for (int z = lo[2] >> l; z <= hi[2] >> l; z++)
        for (int y = lo[1] >> l; y <= hi[1] >> l; y++)
            for (int x = lo[0] >> l; x <= hi[0] >> l; x++)
                if (lev[(uint32_t)x + rl * ((uint32_t)y + rl * (uint32_t)z)]) return true;
    return false;
}

__global__ void __launch_bounds__(128, LVX_SCAT_MINB)
k_scatter(const double *__restrict__ verts, const int32_t *__restrict__ segs, int64_t n_seg, double rt,
          float r_tight, int res, int method, const uint8_t *__restrict__ own_flat, const PyrOffsets O,
          uint32_t *__restrict__ cursor, uint32_t *__restrict__ frags, int64_t cap) {
    const int64_t si = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (si >= n_seg) return;
    const int64_t i = segs[si];
    const d3 a = ld3(verts + 3 * i), b = ld3(verts + 3 * i + 3);
    if (own_flat && !segment_visible(own_flat, O, res, a, b, rt)) return;
    const int64_t res64 = res;
    // f32 view of the segment for the loose test.  Cells whose centre is farther than
    // r_tight + sqrt(3)/2 from the segment are loose without the separating-direction search.
    const SegF sf = make_segf(a, b);
    const float bfx = sf.ax + sf.ex, bfy = sf.ay + sf.ey, bfz = sf.az + sf.ez;
    const float far2 = (r_tight + 0.8661f) * (r_tight + 0.8661f) * 1.001f + 1e-4f;
    // Rows of the traversal are handled four cells at a time: the four cursor atomics are issued
    // back to back (their latencies overlap) before the first dependent fragment store.
    for_each_row(method, a, b, rt, res, [&](int x, int y, int z, int axis, int len) {
        const int64_t stride = axis == 0 ? 1 : (axis == 1 ? res64 : res64 * res64);
        const int64_t idx0 = x + res64 * (y + res64 * z);
        const float sx = axis == 0 ? 1.f : 0.f, sy = axis == 1 ? 1.f : 0.f, sz = axis == 2 ? 1.f : 0.f;
        const float fx = (float)(x - sf.ox) + 0.5f, fy = (float)(y - sf.oy) + 0.5f, fz = (float)(z - sf.oz) + 0.5f;
        for (int u0 = 0; u0 < len; u0 += LVX_BATCH) {
            uint32_t word[LVX_BATCH], pos[LVX_BATCH];
            bool on[LVX_BATCH];
#pragma unroll
            for (int k = 0; k < LVX_BATCH; k++) {
                const int u = u0 + k;
                on[k] = u < len;
                word[k] = 0;
                if (on[k]) {
                    const float cx = fx + (float)u * sx, cy = fy + (float)u * sy, cz = fz + (float)u * sz;
                    bool loose = false;
                    if (r_tight >= 0.f) {
                        loose = segf_dist2(sf, cx, cy, cz) > far2 ||
                                segment_misses_cube(sf.ax - cx, sf.ay - cy, sf.az - cz, bfx - cx, bfy - cy, bfz - cz, r_tight);
                    }
                    word[k] = ((uint32_t)i << 1) | (loose ? 1u : 0u);
                }
            }
#pragma unroll
            for (int k = 0; k < LVX_BATCH; k++) pos[k] = on[k] ? atomicAdd(&cursor[idx0 + (u0 + k) * stride], 1u) : 0u;
#pragma unroll
            for (int k = 0; k < LVX_BATCH; k++)
                if (on[k] && (int64_t)pos[k] < cap) frags[pos[k]] = word[k];
        }
    });
}

// Row-pooled form of k_scatter (capsule method).  One thread still owns one segment, but only for the
// cheap part -- stepping its traversal (RowGen) -- and the warp steps its 32 traversals in lockstep.  The rows
// they produce (3-4 cells each) go into a per-warp queue in shared memory, and whenever 32 rows are queued
// every lane takes ONE row, whoever's it is: the loose test, the cursor atomics and the fragment stores of
// 32 rows are then issued by 32 lanes, instead of by the 16-17 lanes that are still inside their own
// traversal at any given moment (segments differ a lot in their number of rows).  The f32 view of the
// owner's segment is read from shared memory.  Same cells, same words: the fragment lists do not change.
constexpr int SR_WARPS = 4;
struct ScatterWarp {
    int ox[32], oy[32], oz[32];
    float ax[32], ay[32], az[32], ex[32], ey[32], ez[32], inv_ee[32];
    uint32_t seg[32];
    uint32_t q_xyz[64], q_meta[64];      // x | y << 10 | z << 20 | axis << 30 ;  len | owner << 16
};

__global__ void __launch_bounds__(SR_WARPS * 32, LVX_SCAT_MINB)
k_scatter_rows(const double *__restrict__ verts, const int32_t *__restrict__ segs, int64_t n_seg, double rt,
               float r_tight, int res, const uint8_t *__restrict__ own_flat, const PyrOffsets O,
               uint32_t *__restrict__ cursor, uint32_t *__restrict__ frags, int64_t cap) {
    __shared__ ScatterWarp s_w[SR_WARPS];
    const int lane = threadIdx.x & 31;
    ScatterWarp &W = s_w[threadIdx.x >> 5];
    const uint32_t lt_mask = (1u << lane) - 1u;
    const int64_t si = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    RowGen g;
    g.done = true; g.j = 1; g.j_max = 0;
    if (si < n_seg) {
        const int64_t i = segs[si];
        const d3 a = ld3(verts + 3 * i), b = ld3(verts + 3 * i + 3);
        if (!own_flat || segment_visible(own_flat, O, res, a, b, rt)) {
            g.init(a, b, rt, res);
            const SegF sf = make_segf(a, b);
            W.ox[lane] = sf.ox; W.oy[lane] = sf.oy; W.oz[lane] = sf.oz;
            W.ax[lane] = sf.ax; W.ay[lane] = sf.ay; W.az[lane] = sf.az;
            W.ex[lane] = sf.ex; W.ey[lane] = sf.ey; W.ez[lane] = sf.ez; W.inv_ee[lane] = sf.inv_ee;
            W.seg[lane] = (uint32_t)i;
        }
    }
    __syncwarp();
    const float far2 = (r_tight + 0.8661f) * (r_tight + 0.8661f) * 1.001f + 1e-4f;
    const uint32_t res_u = (uint32_t)res;
    uint32_t qn = 0;
    for (;;) {
        const bool more = __any_sync(0xffffffffu, !g.finished());
        if (more) {
            int x = 0, y = 0, z = 0, axis = 0, len = 0;
            const bool have = g.next(x, y, z, axis, len);
            const uint32_t m = __ballot_sync(0xffffffffu, have);
            if (have) {
                const uint32_t pos = qn + __popc(m & lt_mask);
                W.q_xyz[pos] = (uint32_t)x | ((uint32_t)y << 10) | ((uint32_t)z << 20) | ((uint32_t)axis << 30);
                W.q_meta[pos] = (uint32_t)len | ((uint32_t)lane << 16);
            }
            qn += __popc(m);
            __syncwarp();
            if (qn < 32) continue;
        } else if (qn == 0) break;
        // ---- 32 rows (or the rest), one per lane
        const uint32_t take = qn < 32 ? qn : 32;
        qn -= take;
        if ((uint32_t)lane < take) {
            const uint32_t xyz = W.q_xyz[qn + lane], meta = W.q_meta[qn + lane];
            const int x = (int)(xyz & 1023u), y = (int)((xyz >> 10) & 1023u), z = (int)((xyz >> 20) & 1023u);
            const int axis = (int)(xyz >> 30), len = (int)(meta & 0xFFFFu), o = (int)(meta >> 16);
            SegF sf;
            sf.ox = W.ox[o]; sf.oy = W.oy[o]; sf.oz = W.oz[o];
            sf.ax = W.ax[o]; sf.ay = W.ay[o]; sf.az = W.az[o];
            sf.ex = W.ex[o]; sf.ey = W.ey[o]; sf.ez = W.ez[o]; sf.inv_ee = W.inv_ee[o];
            const uint32_t seg2 = W.seg[o] << 1;
            const float bfx = sf.ax + sf.ex, bfy = sf.ay + sf.ey, bfz = sf.az + sf.ez;
            const uint32_t stride = axis == 0 ? 1u : (axis == 1 ? res_u : res_u * res_u);
            const uint32_t idx0 = (uint32_t)x + res_u * ((uint32_t)y + res_u * (uint32_t)z);
            const float sx = axis == 0 ? 1.f : 0.f, sy = axis == 1 ? 1.f : 0.f, sz = axis == 2 ? 1.f : 0.f;
            const float fx = (float)(x - sf.ox) + 0.5f, fy = (float)(y - sf.oy) + 0.5f, fz = (float)(z - sf.oz) + 0.5f;
            for (int u0 = 0; u0 < len; u0 += LVX_BATCH) {
                uint32_t word[LVX_BATCH], pos[LVX_BATCH];
                bool on[LVX_BATCH];
#pragma unroll
                for (int k = 0; k < LVX_BATCH; k++) {
                    const int u = u0 + k;
                    on[k] = u < len;
                    word[k] = 0;
                    if (on[k]) {
                        const float cx = fx + (float)u * sx, cy = fy + (float)u * sy, cz = fz + (float)u * sz;
                        bool loose = false;
                        if (r_tight >= 0.f) {
                            loose = segf_dist2(sf, cx, cy, cz) > far2 ||
                                    segment_misses_cube(sf.ax - cx, sf.ay - cy, sf.az - cz, bfx - cx, bfy - cy, bfz - cz, r_tight);
                        }
                        word[k] = seg2 | (loose ? 1u : 0u);
                    }
                }
#pragma unroll
                for (int k = 0; k < LVX_BATCH; k++) pos[k] = on[k] ? atomicAdd(&cursor[idx0 + (uint32_t)(u0 + k) * stride], 1u) : 0u;
#pragma unroll
                for (int k = 0; k < LVX_BATCH; k++)
                    if (on[k] && (int64_t)pos[k] < cap) frags[pos[k]] = word[k];
            }
        }
        __syncwarp();
    }
}

// ----------------------------------------------------------------------------- ordering

// all-ascending bitonic network on f[0..n) executed by one warp; indices >= n act as +inf
__device__ void warp_bitonic(uint32_t *f, uint32_t n, int lane) {
    int lg = 1;
    while ((1u << lg) < n) lg++;
    const uint32_t half = 1u << (lg - 1);
    for (int lk = 1; lk <= lg; lk++) {                 // merge size k = 2^lk
        const uint32_t k = 1u << lk, hk = k >> 1;
        for (uint32_t t = lane; t < half; t += 32) {   // flip: i <-> mirror inside the k-block
            const uint32_t blk = (t >> (lk - 1)) << lk, o = t & (hk - 1);
            const uint32_t i = blk + o, l = blk + k - 1 - o;
            if (l < n) {
                const uint32_t a = f[i], b = f[l];
                if (a > b) { f[i] = b; f[l] = a; }
            }
        }
        __syncwarp();
        for (int lj = lk - 2; lj >= 0; lj--) {         // disperse: i <-> i + 2^lj
            const uint32_t j = 1u << lj;
            for (uint32_t t = lane; t < half; t += 32) {
                const uint32_t i = ((t >> lj) << (lj + 1)) + (t & (j - 1)), l = i + j;
                if (l < n) {
                    const uint32_t a = f[i], b = f[l];
                    if (a > b) { f[i] = b; f[l] = a; }
                }
            }
            __syncwarp();
        }
    }
}

// Ordering pass over the compacted list of visible voxels (the only voxels that own fragments).
// One warp sorts one list at a time, two lists in flight per iteration for memory-level
// parallelism:
//   n <= 32 : one coalesced 128-byte load, a bitonic network in registers (warp shuffles, depth
//             chosen from n), one coalesced store -- skipped when the list is already ascending;
//   n  > 32 : staged through shared memory (or sorted in place when it exceeds the stage) with
//             the all-ascending bitonic network above.
// HBM traffic is <= 8 B per fragment, every access coalesced.
constexpr int ORDER_WARPS = 8;
constexpr int ORDER_CAP = 512;   // fragments staged per warp for long lists (2 KiB)

// Bitonic sort inside aligned groups of W = 2^LG lanes (li = lane index inside the group); every
// group ends up ascending.  Lanes past a list's end hold 0xffffffff.
template <int LG>
__device__ __forceinline__ uint32_t group_sort(uint32_t v, int li) {
#pragma unroll
    for (int lk = 1; lk <= LG; lk++) {
#pragma unroll
        for (int lj = lk - 1; lj >= 0; lj--) {
            const uint32_t o = __shfl_xor_sync(0xffffffffu, v, 1 << lj);
            // keep the smaller value on the lower lane of an ascending block
            const bool keep_min = (((li >> lk) ^ (li >> lj)) & 1) == 0;
            v = keep_min ? min(v, o) : max(v, o);
        }
    }
    return v;
}

struct TightIndex {
    uint32_t *frags;     // [capacity] tight segment ids, list v at offsets[v] .. offsets[v] + cnt[v]
    uint16_t *slot;      // [capacity] their slots (positions in the full, ascending list)
    uint16_t *cnt;       // [V] tight fragments per voxel
};

// Short lists, 32 / W of them side by side: lane group g sorts the g-th list of size class W
// (W/2 < n <= W, or n <= 2 for W = 2) named by the set bits of `cls`; b, n, vox are the per-lane
// list bounds and voxel of the warp's 32 current list entries.  Each group loads its list with one
// (partial) 128-byte line, sorts it in registers, stores the stripped segment ids and the tight
// index of its list.
template <int LG>
__device__ __forceinline__ void sort_class(uint32_t cls, uint32_t b, uint32_t n, uint32_t vox, uint32_t *__restrict__ frags,
                                           const TightIndex &T, int lane) {
    constexpr int W = 1 << LG, G = 32 / W;
    const int g = lane >> LG, li = lane & (W - 1);
    const uint32_t gmask = W == 32 ? 0xffffffffu : (((1u << (W & 31)) - 1u) << (g * W));   // my group's lanes
    const uint32_t below = gmask & ((1u << lane) - 1u);                                   // ... below me
    while (cls) {
        int src = -1;
#pragma unroll
        for (int k = 0; k < G; k++) {
            if (cls) {
                const int sbit = __ffs(cls) - 1;
                cls &= cls - 1;
                if (k == g) src = sbit;
            }
        }
        const uint32_t bb = __shfl_sync(0xffffffffu, b, src < 0 ? 0 : src);
        const uint32_t nsrc = __shfl_sync(0xffffffffu, n, src < 0 ? 0 : src);   // (all lanes take part)
        const uint32_t vv = __shfl_sync(0xffffffffu, vox, src < 0 ? 0 : src);
        const uint32_t nn = src < 0 ? 0u : nsrc;
        uint32_t val = 0xffffffffu;
        if ((uint32_t)li < nn) val = frags[bb + li];
        val = group_sort<LG>(val, li);
        const bool mine = (uint32_t)li < nn;
        if (mine) frags[bb + li] = val >> 1;
        const bool tight = mine && !(val & 1u);
        const uint32_t bal = __ballot_sync(0xffffffffu, tight);
        if (T.frags) {
            if (tight) {
                const uint32_t k = bb + __popc(bal & below);
                T.frags[k] = val >> 1;
                T.slot[k] = (uint16_t)li;
            }
            if (li == 0 && nn) T.cnt[vv] = (uint16_t)__popc(bal & gmask);
        }
    }
}

// tight index of the 32 sorted packed words v (valid where `in`) at list positions i0 + lane; `run` = tight
// fragments of this list emitted so far (warp-uniform)
__device__ __forceinline__ void emit_tight(const TightIndex &T, uint32_t bb, uint32_t i0, uint32_t v, bool in,
                                           uint32_t &run, int lane) {
    const bool tight = in && !(v & 1u);
    const uint32_t bal = __ballot_sync(0xffffffffu, tight);
    if (T.frags && tight) {
        const uint32_t k = bb + run + __popc(bal & ((1u << lane) - 1u));
        T.frags[k] = v >> 1;
        T.slot[k] = (uint16_t)(i0 + lane);
    }
    run += __popc(bal);
}

// long lists: strip the flag from the sorted packed words in `src` into f[0..nn) and write the tight index
__device__ __forceinline__ void strip_long(const uint32_t *src, uint32_t *f, uint32_t b, uint32_t nn, uint32_t vv,
                                           int lane, const TightIndex &T) {
    uint32_t run = 0;
    for (uint32_t i0 = 0; i0 < nn; i0 += 32) {
        const uint32_t i = i0 + lane;
        const uint32_t v = i < nn ? src[i] : 0u;
        __syncwarp();
        if (i < nn) f[i] = v >> 1;
        emit_tight(T, b, i0, v, i < nn, run, lane);
    }
    if (T.frags && lane == 0) T.cnt[vv] = (uint16_t)run;
}

// Lists of up to 32 * R fragments (R = 2^LR registers per lane), one list at a time: element i lives
// in register i / 32 of lane i % 32.  Stages of the bitonic network whose partner distance is >= 32
// are compare-exchanges between a lane's own registers; the others are one shuffle per register.
template <int LR>
__device__ __forceinline__ void sort_regs(uint32_t todo, uint32_t b, uint32_t n, uint32_t vox, uint32_t *__restrict__ frags,
                                          const TightIndex &T, int lane) {
    constexpr int R = 1 << LR, LGN = 5 + LR;
    while (todo) {
        const int s0 = __ffs(todo) - 1;
        todo &= todo - 1;
        const uint32_t bb = __shfl_sync(0xffffffffu, b, s0), nn = __shfl_sync(0xffffffffu, n, s0);
        const uint32_t vv = __shfl_sync(0xffffffffu, vox, s0);
        uint32_t v[R];
#pragma unroll
        for (int r = 0; r < R; r++) v[r] = (uint32_t)lane + 32u * r < nn ? frags[bb + 32 * r + lane] : 0xffffffffu;
#pragma unroll
        for (int lk = 1; lk <= LGN; lk++) {
#pragma unroll
            for (int lj = lk - 1; lj >= 0; lj--) {
#pragma unroll
                for (int r = 0; r < R; r++) {
                    // bit `bit` of the element index i = lane + 32 r
                    auto ibit = [&](int bit) { return bit < 5 ? ((lane >> bit) & 1) : ((r >> (bit - 5)) & 1); };
                    const bool asc = lk == LGN ? true : ibit(lk) == 0;     // direction of the 2^lk block
                    if (lj >= 5) {
                        const int pr = r ^ (1 << (lj - 5));                // partner register, same lane
                        if (pr > r) {
                            const uint32_t lo = min(v[r], v[pr]), hi = max(v[r], v[pr]);
                            v[r] = asc ? lo : hi; v[pr] = asc ? hi : lo;
                        }
                    } else {
                        const uint32_t o = __shfl_xor_sync(0xffffffffu, v[r], 1 << lj);
                        const bool keep_min = asc == (ibit(lj) == 0);
                        v[r] = keep_min ? min(v[r], o) : max(v[r], o);
                    }
                }
            }
        }
        uint32_t run = 0;
#pragma unroll
        for (int r = 0; r < R; r++) {
            const bool in = (uint32_t)lane + 32u * r < nn;
            if (in) frags[bb + 32 * r + lane] = v[r] >> 1;
            emit_tight(T, bb, 32u * r, v[r], in, run, lane);
        }
        if (T.frags && lane == 0) T.cnt[vv] = (uint16_t)run;
    }
}

#ifndef LVX_ORDER_MINB
#define LVX_ORDER_MINB 8   // 32 registers: the rare 4-elements-per-lane path spills a little, every other path gains occupancy
#endif
__global__ void __launch_bounds__(ORDER_WARPS * 32, LVX_ORDER_MINB)
k_order(const uint32_t *__restrict__ offsets, const uint32_t *__restrict__ cursor,
        const uint32_t *__restrict__ vis_list, uint32_t *__restrict__ frags, int64_t cap,
        const TightIndex T, uint64_t *__restrict__ stats) {
    __shared__ uint32_t stage[ORDER_WARPS][ORDER_CAP];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t n_lists = (int64_t)*reinterpret_cast<const unsigned long long *>(vis_list);
    const int64_t warp_id = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    uint32_t n_long = 0;
    // each warp takes a contiguous chunk of 32 list entries per step: lane k reads entry k's bounds
    for (int64_t e0 = warp_id * 32; e0 < n_lists; e0 += n_warps * 32) {
        uint32_t b = 0, n = 0, vox = 0;
        if (e0 + lane < n_lists) {
            const uint32_t v = vis_list[LVX_LIST_HDR + e0 + lane];
            vox = v;
            b = offsets[v];
            const uint32_t e = offsets[v + 1];
            n = e - b;
            if (cursor[v] != e) stats[LVX_ST_MISMATCH] = 1;   // lv/abuffer.py:310-311
            if ((int64_t)e > cap) {                           // never touch memory past the buffer; the frame is
                n = 0;                                        // redone with a larger one, but the tracer of THIS
                if (T.cnt) T.cnt[v] = 0;                      // frame still runs: no stale tight count for it
            }
        }
        // The lists of this step are loaded one size class after the other, each load at the head of a dependent
        // load-sort-store chain (38 % of the pass's stall samples sat there): ask for all of them now, so that
        // the later classes find their lines in L2.
        if (n) {
            asm volatile("prefetch.global.L2 [%0];" ::"l"(frags + b));
            if (n > 1) asm volatile("prefetch.global.L2 [%0];" ::"l"(frags + b + n - 1));
        }
        n_long += __popc(__ballot_sync(0xffffffffu, n > 32));
        // short lists by size class, several lists per warp step
        sort_class<1>(__ballot_sync(0xffffffffu, n >= 1 && n <= 2), b, n, vox, frags, T, lane);
        sort_class<2>(__ballot_sync(0xffffffffu, n > 2 && n <= 4), b, n, vox, frags, T, lane);
        sort_class<3>(__ballot_sync(0xffffffffu, n > 4 && n <= 8), b, n, vox, frags, T, lane);
        sort_class<4>(__ballot_sync(0xffffffffu, n > 8 && n <= 16), b, n, vox, frags, T, lane);
        sort_class<5>(__ballot_sync(0xffffffffu, n > 16 && n <= 32), b, n, vox, frags, T, lane);
        // lists of 33..128 fragments one at a time, in registers (see sort_regs)
        sort_regs<1>(__ballot_sync(0xffffffffu, n > 32 && n <= 64), b, n, vox, frags, T, lane);
        sort_regs<2>(__ballot_sync(0xffffffffu, n > 64 && n <= 128), b, n, vox, frags, T, lane);
        // longer lists one at a time: staged through shared memory, or in place beyond the stage
        uint32_t work = __ballot_sync(0xffffffffu, n > 128);
        while (work) {
            const int s0 = __ffs(work) - 1;
            work &= work - 1;
            const uint32_t bb = __shfl_sync(0xffffffffu, b, s0), nn = __shfl_sync(0xffffffffu, n, s0);
            const uint32_t vv = __shfl_sync(0xffffffffu, vox, s0);
            uint32_t *f = frags + bb;
            if (nn <= ORDER_CAP) {
                uint32_t *buf = stage[warp];
                for (uint32_t i = lane; i < nn; i += 32) buf[i] = f[i];
                __syncwarp();
                warp_bitonic(buf, nn, lane);
                strip_long(buf, f, bb, nn, vv, lane, T);
                __syncwarp();
            } else {
                warp_bitonic(f, nn, lane);
                strip_long(f, f, bb, nn, vv, lane, T);
            }
        }
    }
    if (lane == 0 && n_long)
        atomicAdd((unsigned long long *)&stats[LVX_ST_LONG_LISTS], (unsigned long long)n_long);
}

// cursor[v] = offsets[v] for visible voxels, LVX_CURSOR_CULLED for culled ones (cull0 == NULL: all visible)
__global__ void __launch_bounds__(256)
k_init_cursor(const uint32_t *__restrict__ offsets, const uint8_t *__restrict__ cull0, uint32_t *__restrict__ cursor, int64_t n) {
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;   // n is a multiple of 8 (lvx_scan)
    if (i >= n) return;
    uint4 o = *reinterpret_cast<const uint4 *>(offsets + i);
    if (cull0) {
        const uchar4 c = *reinterpret_cast<const uchar4 *>(cull0 + i);
        if (!c.x) o.x = LVX_CURSOR_CULLED;
        if (!c.y) o.y = LVX_CURSOR_CULLED;
        if (!c.z) o.z = LVX_CURSOR_CULLED;
        if (!c.w) o.w = LVX_CURSOR_CULLED;
    }
    *reinterpret_cast<uint4 *>(cursor + i) = o;
}

}  // namespace lvx

using namespace lvx;

extern "C" {

int64_t lvx_scan_scratch_bytes(int64_t n_voxels) {
    const int64_t tiles = (n_voxels + SCAN_TILE - 1) / SCAN_TILE;
    return (tiles + 1) * 8;
}

int lvx_scan(const uint32_t *base, const uint8_t *cull_base, int64_t n_voxels, uint32_t *offsets,
             void *scratch, uint64_t *stats, uint32_t *cursor, void *stream) {
    if (n_voxels < 8 || (n_voxels & 7)) return LVX_E_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t tiles = (n_voxels + SCAN_TILE - 1) / SCAN_TILE;
    LVX_CUDA(cudaMemsetAsync(scratch, 0, (size_t)lvx_scan_scratch_bytes(n_voxels), s));
    k_scan<<<(unsigned)tiles, SCAN_THREADS, 0, s>>>(base, cull_base, n_voxels, offsets, cursor,
                                                   (unsigned long long *)scratch, stats);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

int64_t lvx_max_fragments(void) { return (int64_t)LVX_CURSOR_CULLED - 1; }

int lvx_scatter(const double *verts, const int32_t *segs, int64_t n_seg, double rt, double r_tight, int res, int method,
                const uint8_t *cull_flat, const uint32_t *vis_list, const uint32_t *offsets, uint32_t *cursor,
                uint32_t *frags, int64_t frag_capacity, uint32_t *tight_frags, uint16_t *tight_slot, uint16_t *tight_cnt,
                int cursor_ready, uint64_t *stats, void *stream) {
    if (!vis_list) return LVX_E_ARG;
    if (!pow2(res) || method < 0 || method > 2) return LVX_E_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t V = (int64_t)res * res * res;
    if (V & 3) return LVX_E_ARG;
    if (frag_capacity >= (int64_t)LVX_CURSOR_CULLED) return LVX_E_ARG;
    if (!cursor_ready) k_init_cursor<<<blocks_for(V / 4, 256), 256, 0, s>>>(offsets, cull_flat, cursor, V);
    const bool want_tight = tight_frags != nullptr;
    if (want_tight != (tight_slot != nullptr) || want_tight != (tight_cnt != nullptr)) return LVX_E_ARG;
    if (!want_tight) r_tight = -1.0;
    // (tight_cnt needs no clearing: it is only read for voxels whose list the ordering pass wrote)
    PyrOffsets O;
    {
        const LevelOffsets L = make_level_offsets(res);
        if (L.n_levels > 12) return LVX_E_ARG;
        for (int l = 0; l < 12; l++) O.off[l] = l < L.n_levels ? (uint32_t)L.off[l] : 0u;
        O.n_levels = L.n_levels;
    }
    static const bool old_scatter = getenv("LVX_SCATTER_OLD") != nullptr;
    if (n_seg > 0 && method == 1 && !old_scatter)       // capsule traversal: rows pooled per warp
        k_scatter_rows<<<blocks_for(n_seg, SR_WARPS * 32), SR_WARPS * 32, 0, s>>>(verts, segs, n_seg, rt, (float)r_tight, res,
                                                                                 cull_flat, O, cursor, frags, frag_capacity);
    else if (n_seg > 0)
        k_scatter<<<blocks_for(n_seg, 128), 128, 0, s>>>(verts, segs, n_seg, rt, (float)r_tight, res, method,
                                                        cull_flat, O, cursor, frags, frag_capacity);
    {
        unsigned nb = 148 * 8;   // persistent: 148 SMs x 8 CTAs of 8 warps
        const unsigned need = blocks_for((V + 31) / 32, ORDER_WARPS);
        if (nb > need) nb = need;
        const TightIndex T{tight_frags, tight_slot, tight_cnt};
        k_order<<<nb, ORDER_WARPS * 32, 0, s>>>(offsets, cursor, vis_list, frags, frag_capacity, T, stats);
    }
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

}  // extern "C"
