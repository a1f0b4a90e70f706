// cull.cu -- voxel camera-visibility culling.  Replaces lv/culling.py:112-127 (erode),
// 143-200 (_march_blocked, _visibility_kernel), 130-140 (dilate_bits), 103-109 (or_mips).
//
// Only `eroded >= THETA_BLOCK (0.999)` is ever consumed (lv/culling.py:186), and level-0
// occupancy is min(occ_q,4096)/4096, so erode+threshold collapses to the integer predicate
// "occ_q >= 4092 for the voxel and its 6 neighbours" (4092/4096 = 0.99902 >= 0.999 > 4091/4096).
// It is stored as a 1-bit mask (res^3/8 bytes: 2 MiB at 256^3, L1/L2 resident for the march).
#include "lvx_device.cuh"

namespace lvx {

#define LVX_SOLID_Q 4092u
#define LVX_BRICK 8        // coarse "may contain a blocker" bricks for the visibility march
#define LVX_SUPER 32       // and a coarser level above them
#define LVX_SOLID_CAP 16384 // solid voxels listed individually for the per-super-brick shadow test
#define LVX_SB_ROW 128     // words per super-brick row: [number of shadowing solid voxels][up to 127 of them]
#define LVX_SB_CAP (LVX_SB_ROW - 1)

__host__ __device__ inline int64_t brick_words(int res, int B) {
    const int64_t rb = (res + B - 1) / B;
    return (rb * rb * rb + 31) / 32;
}

__device__ __forceinline__ bool q_solid(const uint32_t *__restrict__ base, int res, int x, int y, int z) {
    if (x < 0 || y < 0 || z < 0 || x >= res || y >= res || z >= res) return false;   // outside counts as 0
    return (base[x + (int64_t)res * (y + (int64_t)res * z)] & 0xFFFFu) >= LVX_SOLID_Q;
}

// One block = SOLID_ITEMS x 256 consecutive voxels; a thread owns voxels tid, tid+256, ... of the
// block's chunk, so every item is a coalesced row, a warp's ballot is one word of the bit mask, and
// the four loads of a thread are in flight together.  The occupied-voxel list gets ONE counter
// atomic per block (1024 voxels).
constexpr int SOLID_ITEMS = 4;
__global__ void __launch_bounds__(256)
k_solid(const uint32_t *__restrict__ base, int res, int64_t V, uint32_t *__restrict__ solid,
        uint32_t *__restrict__ solid_list, uint32_t *__restrict__ occ_list, uint64_t *__restrict__ stats) {
    __shared__ uint32_t s_warp[8];
    __shared__ unsigned long long s_base;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t chunk = (int64_t)blockIdx.x * (SOLID_ITEMS * 256);
    uint32_t w[SOLID_ITEMS];
#pragma unroll
    for (int k = 0; k < SOLID_ITEMS; k++) {
        const int64_t idx = chunk + k * 256 + threadIdx.x;
        w[k] = idx < V ? base[idx] : 0u;
    }
    uint32_t n_occ = 0;
#pragma unroll
    for (int k = 0; k < SOLID_ITEMS; k++) {
        const int64_t idx = chunk + k * 256 + threadIdx.x;
        bool s = false;
        n_occ += (w[k] >> 16) != 0;
        if (idx < V && (w[k] & 0xFFFFu) >= LVX_SOLID_Q) {
            const int x = (int)(idx % res), y = (int)((idx / res) % res), z = (int)(idx / ((int64_t)res * res));
            s = q_solid(base, res, x - 1, y, z) && q_solid(base, res, x + 1, y, z) &&
                q_solid(base, res, x, y - 1, z) && q_solid(base, res, x, y + 1, z) &&
                q_solid(base, res, x, y, z - 1) && q_solid(base, res, x, y, z + 1);
        }
        const uint32_t m = __ballot_sync(0xffffffffu, s);
        if (lane == 0 && idx < V) {
            solid[idx >> 5] = m;
            if (m) atomicAdd((unsigned long long *)&stats[LVX_ST_SOLID], (unsigned long long)__popc(m));
        }
        // (solid voxels are rare in thin-line frames: a list of the first LVX_SOLID_CAP of them, word 0 = their
        // number.  One counter atomic per warp; once the counter is past the cap -- nobody reads the list then,
        // only "more than the cap" -- the appends stop, so a frame full of solid voxels does not queue up on it)
        if (m) {
            uint32_t slot0 = 0;
            if (lane == 0) {
                slot0 = *reinterpret_cast<volatile uint32_t *>(&solid_list[0]);
                if (slot0 <= LVX_SOLID_CAP) slot0 = atomicAdd(&solid_list[0], (uint32_t)__popc(m));
            }
            slot0 = __shfl_sync(0xffffffffu, slot0, 0);
            if (s) {
                const uint32_t slot = slot0 + __popc(m & ((1u << lane) - 1u));
                if (slot < LVX_SOLID_CAP) solid_list[LVX_LIST_HDR + slot] = (uint32_t)idx;
            }
        }
    }
    // compacted list of occupied voxels (the march kernels then run on dense warps): block scan of
    // the per-thread counts, one atomic on the list counter per block
    uint32_t inc = n_occ;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += v;
    }
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        const uint32_t c = lane < 8 ? s_warp[lane] : 0;
        uint32_t wi = c;
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += v;
        }
        if (lane < 8) s_warp[lane] = wi - c;
        if (lane == 7 && wi)
            s_base = atomicAdd((unsigned long long *)&stats[LVX_ST_OCCUPIED], (unsigned long long)wi);
    }
    __syncthreads();
    if (n_occ) {
        uint64_t slot = s_base + s_warp[warp] + (inc - n_occ);
#pragma unroll
        for (int k = 0; k < SOLID_ITEMS; k++)
            if ((w[k] >> 16) != 0) occ_list[slot++] = (uint32_t)(chunk + k * 256 + threadIdx.x);
    }
}

// Brick flags from the finished solid bits.  An 8^3 brick is flagged when it overlaps a solid voxel dilated by
// one voxel, i.e. when a solid bit is set in the brick grown by a voxel on every side; a 32^3 super-brick
// overlaps such a dilated voxel exactly when one of its 8^3 bricks does.  One warp per brick: 10 x 10 rows of
// 10 bits.  (Round 1 had every solid voxel set its bricks' flags with atomics from k_solid: in a frame full
// of solid voxels that was most of that kernel's time.)  Nothing is solid -> the flags stay as cleared.
__global__ void __launch_bounds__(128)
k_brick_flags(const uint32_t *__restrict__ solid, int res, const uint64_t *__restrict__ stats, uint32_t *__restrict__ flags) {
    if (stats[LVX_ST_SOLID] == 0) return;
    // one warp per brick, the (up to) 10 x 10 rows spread over its lanes; the flag words were cleared by the caller
    const int rb = (res + LVX_BRICK - 1) / LVX_BRICK;
    const int b = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
    if (b >= rb * rb * rb) return;
    const int bx = b % rb, by = (b / rb) % rb, bz = b / (rb * rb);
    const int x0 = max(bx * LVX_BRICK - 1, 0), x1 = min(bx * LVX_BRICK + LVX_BRICK, res - 1);
    const int y0 = max(by * LVX_BRICK - 1, 0), y1 = min(by * LVX_BRICK + LVX_BRICK, res - 1);
    const int z0 = max(bz * LVX_BRICK - 1, 0), z1 = min(bz * LVX_BRICK + LVX_BRICK, res - 1);
    const int ny = y1 - y0 + 1, n_rows = ny * (z1 - z0 + 1);
    bool any = false;
    for (int r = lane; r < n_rows; r += 32) {
        const int y = y0 + r % ny, z = z0 + r / ny;
        const int64_t i0 = x0 + (int64_t)res * (y + (int64_t)res * z), i1 = i0 + (x1 - x0);   // bits i0 .. i1 of the row
        const int64_t w0 = i0 >> 5, w1 = i1 >> 5;
        const uint32_t lo = 0xffffffffu << (i0 & 31), hi = 0xffffffffu >> (31 - (i1 & 31));
        if (w0 == w1) any |= (solid[w0] & lo & hi) != 0;
        else any |= (solid[w0] & lo) != 0 || (solid[w1] & hi) != 0;                  // (at most 10 bits: two words)
    }
    if (__any_sync(0xffffffffu, any) && lane == 0) atomicOr(&flags[b >> 5], 1u << (b & 31));
}

__global__ void __launch_bounds__(128)
k_super_flags(const uint32_t *__restrict__ flags, int res, const uint64_t *__restrict__ stats, uint32_t *__restrict__ sflags) {
    if (stats[LVX_ST_SOLID] == 0) return;
    const int rb = (res + LVX_BRICK - 1) / LVX_BRICK, rs = (res + LVX_SUPER - 1) / LVX_SUPER;
    constexpr int K = LVX_SUPER / LVX_BRICK;
    const int sb = blockIdx.x * blockDim.x + threadIdx.x;
    bool any = false;
    if (sb < rs * rs * rs) {
        const int sx = sb % rs, sy = (sb / rs) % rs, sz = sb / (rs * rs);
        for (int z = sz * K; z < min(sz * K + K, rb) && !any; z++)
            for (int y = sy * K; y < min(sy * K + K, rb) && !any; y++)
                for (int x = sx * K; x < min(sx * K + K, rb); x++) {
                    const int bi = x + rb * (y + rb * z);
                    if ((flags[bi >> 5] >> (bi & 31)) & 1u) { any = true; break; }
                }
    }
    const uint32_t m = __ballot_sync(0xffffffffu, any);
    if ((threadIdx.x & 31) == 0 && sb < ((rs * rs * rs + 31) & ~31)) sflags[sb >> 5] = m;
}

// lv/culling.py:143-188, literally: Amanatides-Woo from the voxel centre to the camera point.
// `t_stop`: a parameter beyond which the caller has PROVED that the walk cannot meet a solid voxel (see
// coarse_last_flagged); there the reference's loop can only run on to one of its `return False` exits.
__device__ __forceinline__ bool march_blocked(const uint32_t *__restrict__ solid, int res, int x, int y, int z,
                                              double cx, double cy, double cz, double t_stop = 2.0) {
    const double ox = x + 0.5, oy = y + 0.5, oz = z + 0.5;
    const double dx = cx - ox, dy = cy - oy, dz = cz - oz;
    const int ex = (int)floor(cx), ey = (int)floor(cy), ez = (int)floor(cz);
    const int sx = dx > 0 ? 1 : -1, sy = dy > 0 ? 1 : -1, sz = dz > 0 ? 1 : -1;
    const double big = 1e30;
    double tmx = dx != 0.0 ? ((double)(x + (sx > 0 ? 1 : 0)) - ox) / dx : big;
    double tmy = dy != 0.0 ? ((double)(y + (sy > 0 ? 1 : 0)) - oy) / dy : big;
    double tmz = dz != 0.0 ? ((double)(z + (sz > 0 ? 1 : 0)) - oz) / dz : big;
    const double tdx = dx != 0.0 ? fabs(1.0 / dx) : big;
    const double tdy = dy != 0.0 ? fabs(1.0 / dy) : big;
    const double tdz = dz != 0.0 ? fabs(1.0 / dz) : big;
    // The reference's loop leaves with "not blocked" on four conditions (reached the camera: t >= 1; left the
    // grid; entered the camera's own voxel; here also t > t_stop) before it looks at the voxel, and their order
    // among themselves does not matter.  t >= 1 or t > t_stop  <=>  t > min(t_stop, pred(1)); only the coordinate
    // that was stepped can leave the grid (the walk starts inside it); the camera's voxel is one flat index.
    const double t_lim = fmin(t_stop, 0x1.fffffffffffffp-1);
    const uint32_t ures = (uint32_t)res;
    const bool cam_in = (uint32_t)ex < ures && (uint32_t)ey < ures && (uint32_t)ez < ures;
    const uint32_t cam_idx = cam_in ? (uint32_t)ex + ures * ((uint32_t)ey + ures * (uint32_t)ez) : 0xffffffffu;   // (V <= 2^30)
    uint32_t idx = (uint32_t)x + ures * ((uint32_t)y + ures * (uint32_t)z);
    const uint32_t stx = (uint32_t)sx, sty = (uint32_t)(sy * res), stz = (uint32_t)(sz * res * res);
    for (;;) {
        double t;
        uint32_t c;                                                                  // the coordinate just stepped
        if (tmx <= tmy && tmx <= tmz) { x += sx; c = (uint32_t)x; idx += stx; t = tmx; tmx += tdx; }
        else if (tmy <= tmz) { y += sy; c = (uint32_t)y; idx += sty; t = tmy; tmy += tdy; }
        else { z += sz; c = (uint32_t)z; idx += stz; t = tmz; tmz += tdz; }
        if (t > t_lim || c >= ures || idx == cam_idx) return false;
        if ((solid[idx >> 5] >> (idx & 31)) & 1u) return true;
    }
}

// Conservative coarse walk: Amanatides-Woo over bricks of `brick` voxels along the segment
// o -> c (clipped to the grid); true if a flagged brick is visited.  A brick is flagged when it
// overlaps a solid voxel dilated by a whole voxel, so if the fine march would reach a solid voxel,
// at least 2 voxels of the segment lie strictly inside a flagged region, a point of it a whole voxel
// away from unflagged space, and a walk whose errors are far below one voxel must visit a flagged brick.
// Single precision is enough: the walk only has to be right up to errors much smaller than the
// one-voxel dilation of the flags (coordinates <= 1024 voxels -> errors < 1e-3 voxel).
__device__ __forceinline__ bool coarse_may_hit(const uint32_t *__restrict__ bits, int rb, int brick,
                                               float ox, float oy, float oz, float cx, float cy, float cz) {
    const float inv = 1.0f / (float)brick;
    const float o[3] = {ox * inv, oy * inv, oz * inv};
    const float d[3] = {(cx - ox) * inv, (cy - oy) * inv, (cz - oz) * inv};
    float t0 = 0.0f, t1 = 1.0f;
#pragma unroll
    for (int a = 0; a < 3; a++) {
        if (d[a] == 0.0f) { if (o[a] < 0.0f || o[a] > (float)rb) return false; }
        else {
            const float id = __fdividef(1.0f, d[a]);
            float ta = (0.0f - o[a]) * id, tb = ((float)rb - o[a]) * id;
            if (ta > tb) { const float tmp = ta; ta = tb; tb = tmp; }
            t0 = fmaxf(t0, ta); t1 = fminf(t1, tb);
        }
    }
    if (t0 > t1 + 1e-4f) return false;
    int c[3], st[3];
    float tm[3], td[3];
#pragma unroll
    for (int a = 0; a < 3; a++) {
        const float p = o[a] + d[a] * t0;
        c[a] = min(max((int)floorf(p), 0), rb - 1);
        st[a] = d[a] > 0 ? 1 : -1;
        const float id = d[a] != 0.0f ? __fdividef(1.0f, d[a]) : 0.0f;
        tm[a] = d[a] != 0.0f ? ((float)(c[a] + (d[a] > 0 ? 1 : 0)) - o[a]) * id : 1e30f;
        td[a] = d[a] != 0.0f ? fabsf(id) : 1e30f;
    }
    for (;;) {
        const int bi = c[0] + rb * (c[1] + rb * c[2]);
        if ((bits[bi >> 5] >> (bi & 31)) & 1u) return true;
        float t;
        if (tm[0] <= tm[1] && tm[0] <= tm[2]) { c[0] += st[0]; t = tm[0]; tm[0] += td[0]; }
        else if (tm[1] <= tm[2]) { c[1] += st[1]; t = tm[1]; tm[1] += td[1]; }
        else { c[2] += st[2]; t = tm[2]; tm[2] += td[2]; }
        if (t > t1 + 1e-4f) return false;
        if (c[0] < 0 || c[1] < 0 || c[2] < 0 || c[0] >= rb || c[1] >= rb || c[2] >= rb) return false;
    }
}

// The same brick walk run to the end of the segment: returns the parameter at which the walk leaves the
// LAST flagged brick (< 0: none is flagged).  Beyond that parameter (plus the caller's margin of two
// voxels) every voxel within one voxel of the segment lies in unflagged bricks, i.e. is not solid.
__device__ __forceinline__ float coarse_last_flagged(const uint32_t *__restrict__ bits, int rb, int brick,
                                                     float ox, float oy, float oz, float cx, float cy, float cz) {
    const float inv = 1.0f / (float)brick;
    const float o[3] = {ox * inv, oy * inv, oz * inv};
    const float d[3] = {(cx - ox) * inv, (cy - oy) * inv, (cz - oz) * inv};
    float t0 = 0.0f, t1 = 1.0f;
#pragma unroll
    for (int a = 0; a < 3; a++) {
        if (d[a] == 0.0f) { if (o[a] < 0.0f || o[a] > (float)rb) return -1.0f; }
        else {
            const float id = __fdividef(1.0f, d[a]);
            float ta = (0.0f - o[a]) * id, tb = ((float)rb - o[a]) * id;
            if (ta > tb) { const float tmp = ta; ta = tb; tb = tmp; }
            t0 = fmaxf(t0, ta); t1 = fminf(t1, tb);
        }
    }
    if (t0 > t1 + 1e-4f) return -1.0f;
    int c[3], st[3];
    float tm[3], td[3];
#pragma unroll
    for (int a = 0; a < 3; a++) {
        const float p = o[a] + d[a] * t0;
        c[a] = min(max((int)floorf(p), 0), rb - 1);
        st[a] = d[a] > 0 ? 1 : -1;
        const float id = d[a] != 0.0f ? __fdividef(1.0f, d[a]) : 0.0f;
        tm[a] = d[a] != 0.0f ? ((float)(c[a] + (d[a] > 0 ? 1 : 0)) - o[a]) * id : 1e30f;
        td[a] = d[a] != 0.0f ? fabsf(id) : 1e30f;
    }
    float last = -1.0f;
    for (;;) {
        const int bi = c[0] + rb * (c[1] + rb * c[2]);
        const bool flagged = (bits[bi >> 5] >> (bi & 31)) & 1u;
        float t;
        if (tm[0] <= tm[1] && tm[0] <= tm[2]) { c[0] += st[0]; t = tm[0]; tm[0] += td[0]; }
        else if (tm[1] <= tm[2]) { c[1] += st[1]; t = tm[1]; tm[1] += td[1]; }
        else { c[2] += st[2]; t = tm[2]; tm[2] += td[2]; }
        if (flagged) last = fminf(t, 1.0f);
        if (t > t1 + 1e-4f) return last;
        if (c[0] < 0 || c[1] < 0 || c[2] < 0 || c[0] >= rb || c[1] >= rb || c[2] >= rb) return last;
    }
}

// hull(B, c) = union over u in [0, 1] of the boxes c + u (B - c), B = [blo, bhi]; such a box meets the
// cube F (solid voxel v dilated by 1.5 voxels) iff six per-axis inequalities hold, each linear in u, so
// the test is an intersection of six u-intervals.  True when a voxel of B may be shadowed by v.
__device__ __forceinline__ bool shadow_reaches(const float c[3], const float blo[3], const float bhi[3], uint32_t v, int res) {
    const int s3[3] = {(int)(v % res), (int)((v / res) % res), (int)(v / ((uint32_t)res * res))};
    float u0 = 0.f, u1 = 1.f;
#pragma unroll
    for (int a = 0; a < 3; a++) {
        const float flo = (float)s3[a] - 1.5f, fhi = (float)s3[a] + 2.5f;
        // c + u (blo - c) <= fhi
        {
            const float g0 = c[a], g1 = blo[a];
            if (g0 > fhi && g1 > fhi) u1 = -1.f;
            else if (g0 <= fhi && g1 > fhi) u1 = fminf(u1, __fdividef(fhi - g0, g1 - g0) + 1e-3f);
            else if (g0 > fhi && g1 <= fhi) u0 = fmaxf(u0, __fdividef(fhi - g0, g1 - g0) - 1e-3f);
        }
        // c + u (bhi - c) >= flo
        {
            const float g0 = c[a], g1 = bhi[a];
            if (g0 < flo && g1 < flo) u1 = -1.f;
            else if (g0 >= flo && g1 < flo) u1 = fminf(u1, __fdividef(flo - g0, g1 - g0) + 1e-3f);
            else if (g0 < flo && g1 >= flo) u0 = fmaxf(u0, __fdividef(flo - g0, g1 - g0) - 1e-3f);
        }
    }
    return u0 <= u1;
}

// Shadow test per 32^3 super-brick.  A voxel can only be blocked if the segment from its centre
// to the camera meets a solid voxel, so every voxel of a super-brick B is visible when the convex
// hull of B and the camera point misses every solid voxel (dilated by 1.5 voxels: far more than
// the literal march can stray from the geometric segment).  hull(B, c) = union over u in [0, 1] of
// the boxes c + u (B - c); such a box meets the cube F iff the six per-axis inequalities hold, each
// linear in u, so the test is an intersection of six u-intervals.  Work: super-bricks x solid
// voxels (512 x 58 on C2) -- and the per-voxel brick walks then run only inside flagged super-bricks.
__global__ void __launch_bounds__(64)
k_superbrick_shadow(const uint32_t *__restrict__ solid_list, int res, float cx, float cy, float cz,
                    uint8_t *__restrict__ sb_flag, uint32_t *__restrict__ sb_rows) {
    // one block of 64 threads per super-brick, the solid voxels dealt out to the threads
    __shared__ uint32_t s_n;
    const int rs = (res + LVX_SUPER - 1) / LVX_SUPER;
    const int sb = blockIdx.x;
    uint32_t *row = sb_rows + (size_t)sb * LVX_SB_ROW;
    const uint32_t n_all = solid_list[0];
    if (n_all > LVX_SOLID_CAP) {      // too many to list: no shortcut
        if (threadIdx.x == 0) { sb_flag[sb] = 1; row[0] = 0xFFFFFFFFu; }
        return;
    }
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    const float c[3] = {cx, cy, cz};
    const int b3[3] = {sb % rs, (sb / rs) % rs, sb / (rs * rs)};
    float blo[3], bhi[3];
#pragma unroll
    for (int a = 0; a < 3; a++) { blo[a] = (float)(b3[a] * LVX_SUPER); bhi[a] = fminf((float)((b3[a] + 1) * LVX_SUPER), (float)res); }
    for (uint32_t k = threadIdx.x; k < n_all; k += blockDim.x) {
        const uint32_t v = solid_list[LVX_LIST_HDR + k];
        const bool reaches = shadow_reaches(c, blo, bhi, v, res);
        if (reaches) {      // this solid voxel's shadow reaches into the super-brick: keep it for the per-voxel test
            const uint32_t slot = atomicAdd(&s_n, 1u);
            if (slot < LVX_SB_CAP) row[1 + slot] = v;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) { sb_flag[sb] = (uint8_t)(s_n != 0); row[0] = s_n; }
}

// Per-voxel test against the solid voxels kept for the voxel's super-brick.  Returns 0 = visible,
// 1 = blocked, 2 = undecided (the literal march decides).
//  * The literal march (march_blocked) can only be stopped by a solid voxel S that it visits, and every
//    voxel it visits touches the segment centre -> camera: an f32 slab test against S dilated by 1.5
//    voxels (the margin of the super-brick test) discards the solid voxels that cannot matter.
//  * For the others the segment o + t (c - o) is clipped in f64 against S shrunk and S grown by 1e-6.
//    If it meets the shrunk cube before t = 1 - 1e-9 it stays inside S for a parameter interval of
//    >= 1e-9, a thousand times the rounding the march's accumulated crossing parameters can carry
//    (<= ~600 additions of ulp-accurate terms), so the march is in S after the step that enters it --
//    and it cannot have ended earlier: it leaves the grid or reaches the camera's voxel only after S
//    (S is in the grid, and the segment ends inside the camera's voxel).  If it misses the grown cube
//    (or only meets it beyond t = 1 + 1e-9) the march cannot visit S.  In between: undecided.
//    S = the voxel itself and S = the camera's voxel never block (lv/culling.py:176-186).
__device__ __forceinline__ int listed_solid_blocks(const uint32_t *list, uint32_t n, int res,
                                                   int x, int y, int z, double cx, double cy, double cz) {
    const float of[3] = {x + 0.5f, y + 0.5f, z + 0.5f};
    const float df[3] = {(float)cx - of[0], (float)cy - of[1], (float)cz - of[2]};
    float inv[3];
#pragma unroll
    for (int a = 0; a < 3; a++) inv[a] = df[a] != 0.f ? __fdividef(1.f, df[a]) : 0.f;
    const int self3[3] = {x, y, z};
    const int cam3[3] = {(int)floor(cx), (int)floor(cy), (int)floor(cz)};
    const double o[3] = {x + 0.5, y + 0.5, z + 0.5};
    const double d[3] = {cx - o[0], cy - o[1], cz - o[2]};
    int result = 0;
    for (uint32_t k = 0; k < n; k++) {
        const uint32_t v = list[k];
        const int s3[3] = {(int)(v % res), (int)((v / res) % res), (int)(v / ((uint32_t)res * res))};
        float t0 = 0.f, t1 = 1.f;
#pragma unroll
        for (int a = 0; a < 3; a++) {
            const float lo = (float)s3[a] - 1.5f - of[a], hi = (float)s3[a] + 2.5f - of[a];
            if (df[a] == 0.f) { if (lo > 0.f || hi < 0.f) t1 = -1.f; }
            else {
                const float ta = lo * inv[a], tb = hi * inv[a];
                t0 = fmaxf(t0, fminf(ta, tb)); t1 = fminf(t1, fmaxf(ta, tb));
            }
        }
        if (!(t0 <= t1 + 1e-3f)) continue;                     // the march cannot come near S
        if (s3[0] == self3[0] && s3[1] == self3[1] && s3[2] == self3[2]) continue;
        if (s3[0] == cam3[0] && s3[1] == cam3[1] && s3[2] == cam3[2]) continue;
        // f64: entry/exit parameters for the shrunk (sure) and the grown (maybe) cube
        double si = 0.0, so = 1.0 - 1e-9, gi = 0.0, go = 1.0 + 1e-9;
#pragma unroll
        for (int a = 0; a < 3; a++) {
            const double lo = (double)s3[a] - o[a], hi = lo + 1.0;
            if (d[a] == 0.0) {
                if (!(lo + 1e-6 < 0.0 && 0.0 < hi - 1e-6)) so = -1.0;
                if (!(lo - 1e-6 < 0.0 && 0.0 < hi + 1e-6)) go = -1.0;
            } else {
                const double id = 1.0 / d[a];
                const double sa = (lo + 1e-6) * id, sb = (hi - 1e-6) * id;
                const double ga = (lo - 1e-6) * id, gb = (hi + 1e-6) * id;
                si = fmax(si, fmin(sa, sb)); so = fmin(so, fmax(sa, sb));
                gi = fmax(gi, fmin(ga, gb)); go = fmin(go, fmax(ga, gb));
            }
        }
        if (si <= so) return 1;
        if (gi <= go) result = 2;
    }
    return result;
}

// lv/culling.py:191-200.  When the frame has no solid voxel at all nothing can block, so every
// occupied voxel is visible and the march is skipped (decided on the device, no host sync).
// Phase A over the compacted occupied voxels: coarse walks only.  Voxels that may be blocked are
// appended to `march_list`; everything else is visible.
__global__ void __launch_bounds__(128)
k_visibility(const uint32_t *__restrict__ bricks, const uint8_t *__restrict__ sb_flag,
             const uint32_t *__restrict__ sb_rows, const uint32_t *__restrict__ solid_list,
             const uint32_t *__restrict__ occ_list, int res,
             double cx, double cy, double cz, const uint64_t *__restrict__ stats,
             uint8_t *__restrict__ vis, uint32_t *__restrict__ march_list) {
    __shared__ uint32_t s_cand[4][LVX_SB_ROW];   // per warp: the solid voxels that can matter to its 32 voxels
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t n = (int64_t)stats[LVX_ST_OCCUPIED];
    const bool any_solid = stats[LVX_ST_SOLID] != 0;
    if (!any_solid) return;        // nothing can block: k_dilate treats every occupied voxel as visible
    const uint32_t n_all = solid_list[0];
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t n_iter = (n + stride - 1) / stride;
    const int rs = (res + LVX_SUPER - 1) / LVX_SUPER;
    const float cf[3] = {(float)cx, (float)cy, (float)cz};
    for (int64_t it = 0; it < n_iter; it++) {
        const int64_t e = it * stride + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
        bool may_hit = false, blocked = false, flagged = false;
        uint32_t idx = 0;
        int x = 0, y = 0, z = 0, sb = 0;
        if (e < n) {
            idx = occ_list[e];
            x = (int)(idx % res); y = (int)((idx / res) % res); z = (int)(idx / ((uint32_t)res * res));
            sb = (x / LVX_SUPER) + rs * ((y / LVX_SUPER) + rs * (z / LVX_SUPER));
            flagged = any_solid && sb_flag[sb];       // only a solid voxel can block
        }
        const uint32_t fm = __ballot_sync(0xffffffffu, flagged);
        if (fm) {
            // The warp's voxels are consecutive entries of the occupied list: neighbours in a row, mostly.
            // The listed solid voxels (those shadowing the super-brick if all lanes share one, else all of
            // them) are first tested, one per lane, against the hull of the warp's bounding box and the
            // camera; the few that remain are what every lane then decides against in closed form.
            const int sb0 = __shfl_sync(0xffffffffu, sb, __ffs(fm) - 1);
            const bool same = __all_sync(0xffffffffu, !flagged || sb == sb0);
            const uint32_t *row = sb_rows + (size_t)sb0 * LVX_SB_ROW;
            const uint32_t n_row = row[0];
            const bool use_row = same && n_row <= LVX_SB_CAP;
            const uint32_t *src = use_row ? row + 1 : solid_list + LVX_LIST_HDR;
            const uint32_t cnt = use_row ? n_row : n_all;
            // no short list for this warp (too many solid voxels shadow the super-brick, or the lanes
            // straddle super-bricks in a frame with many solid voxels): coarse walks below
            bool walk = n_all > LVX_SOLID_CAP || (!use_row && n_all > 1024u);
            bool full = false;
            uint32_t nc = 0;
            if (!walk) {
                const int big = 1 << 30;
                const float blo[3] = {(float)__reduce_min_sync(0xffffffffu, flagged ? x : big),
                                      (float)__reduce_min_sync(0xffffffffu, flagged ? y : big),
                                      (float)__reduce_min_sync(0xffffffffu, flagged ? z : big)};
                const float bhi[3] = {(float)(__reduce_max_sync(0xffffffffu, flagged ? x : -big) + 1),
                                      (float)(__reduce_max_sync(0xffffffffu, flagged ? y : -big) + 1),
                                      (float)(__reduce_max_sync(0xffffffffu, flagged ? z : -big) + 1)};
                for (uint32_t k0 = 0; k0 < cnt && !full; k0 += 32) {
                    const uint32_t k = k0 + lane;
                    uint32_t v = 0;
                    bool reaches = false;
                    if (k < cnt) { v = src[k]; reaches = shadow_reaches(cf, blo, bhi, v, res); }
                    const uint32_t hm = __ballot_sync(0xffffffffu, reaches);
                    if (nc + __popc(hm) > LVX_SB_ROW) full = true;      // too many remain: every lane takes the whole list
                    else {
                        if (reaches) s_cand[warp][nc + __popc(hm & ((1u << lane) - 1u))] = v;
                        nc += __popc(hm);
                    }
                }
                __syncwarp();
            }
            if (flagged) {
                if (!walk) {
                    const int r = full ? listed_solid_blocks(src, cnt, res, x, y, z, cx, cy, cz)
                                       : listed_solid_blocks(s_cand[warp], nc, res, x, y, z, cx, cy, cz);
                    blocked = r == 1;
                    may_hit = r == 2;
                } else {
                    // walk the segment centre->camera through the 32^3-voxel super-bricks, then the 8^3 bricks
                    const float ox = x + 0.5f, oy = y + 0.5f, oz = z + 0.5f;
                    may_hit = coarse_may_hit(bricks + brick_words(res, LVX_BRICK), rs, LVX_SUPER, ox, oy, oz, cf[0], cf[1], cf[2]);
                    if (may_hit)
                        may_hit = coarse_may_hit(bricks, (res + LVX_BRICK - 1) / LVX_BRICK, LVX_BRICK, ox, oy, oz,
                                                 cf[0], cf[1], cf[2]);
                }
            }
            __syncwarp();      // s_cand is rewritten in the next iteration
        }
        if (e < n && !may_hit && !blocked) vis[idx] = 1;
        list_append_block(march_list, may_hit, idx);
    }
}

// Phase B: the literal fine march (lv/culling.py:143-188) decides for the remaining candidates, in two
// launches.  In a frame with many solid voxels most candidates sit inside the solid mass and their walk ends
// in a blocker within a few steps, while the visible ones walk on for hundreds of steps: taken together a
// warp runs the long walks with a third of its lanes.  k_march_probe walks only the first ~6 voxels (a
// "true" of the truncated walk is a "true" of the full one; a "false" decides nothing) and compacts the
// undecided candidates into a second list; k_march then runs the long walks on full warps.
__global__ void __launch_bounds__(128)
k_march_probe(const uint32_t *__restrict__ solid, const uint32_t *__restrict__ march_list, int res, double cx, double cy,
              double cz, uint32_t *__restrict__ long_list) {
    const int64_t n = (int64_t)*reinterpret_cast<const unsigned long long *>(march_list);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t n_iter = (n + stride - 1) / stride;
    for (int64_t it = 0; it < n_iter; it++) {
        const int64_t e = it * stride + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
        bool undecided = false;
        uint32_t idx = 0;
        if (e < n) {
            idx = march_list[LVX_LIST_HDR + e];
            const int x = (int)(idx % res), y = (int)((idx / res) % res), z = (int)(idx / ((uint32_t)res * res));
            const float dmax = fmaxf(fmaxf(fabsf((float)cx - (x + 0.5f)), fabsf((float)cy - (y + 0.5f))), fabsf((float)cz - (z + 0.5f)));
            undecided = !(dmax > 0.f && march_blocked(solid, res, x, y, z, cx, cy, cz, 6.0 / (double)dmax));
            // (blocked: vis[idx] stays 0)
        }
        list_append_block(long_list, undecided, idx);
    }
}

__global__ void __launch_bounds__(128)
k_march(const uint32_t *__restrict__ solid, const uint32_t *__restrict__ bricks, const uint32_t *__restrict__ long_list,
        int res, double cx, double cy, double cz, uint8_t *__restrict__ vis) {
    const int64_t n = (int64_t)*reinterpret_cast<const unsigned long long *>(long_list);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += stride) {
        const uint32_t idx = long_list[LVX_LIST_HDR + e];
        const int x = (int)(idx % res), y = (int)((idx / res) % res), z = (int)(idx / ((uint32_t)res * res));
        // Most of these candidates are visible, and their literal walk would run on to the camera or the grid's
        // boundary long after the last place a solid voxel can be.  A brick walk over the whole segment
        // (f32, conservative: flags cover the solid voxels dilated by a voxel) gives the parameter where
        // the segment leaves the last flagged 8^3 brick; two voxels later the literal walk may stop.
        const float ox = x + 0.5f, oy = y + 0.5f, oz = z + 0.5f;
        const float tl = coarse_last_flagged(bricks, (res + LVX_BRICK - 1) / LVX_BRICK, LVX_BRICK, ox, oy, oz,
                                             (float)cx, (float)cy, (float)cz);
        bool blocked = false;
        if (tl >= 0.0f) {
            const float dmax = fmaxf(fmaxf(fabsf((float)cx - ox), fabsf((float)cy - oy)), fabsf((float)cz - oz));
            const double t_stop = dmax > 0.f ? (double)tl * 1.0001 + 2.0 / (double)dmax + 1e-4 : 2.0;
            blocked = march_blocked(solid, res, x, y, z, cx, cy, cz, t_stop);
        }
        vis[idx] = blocked ? 0 : 1;
    }
}

// Appends the set bits of the per-thread masks (bit k = voxel first + k of this thread, ITEMS voxels per
// thread, threads in voxel order) to `list` in ascending voxel order inside the block's chunk: block
// scan of the per-thread counts, ONE atomic on the list counter per block.  Called by all 256 threads.
template <int ITEMS>
__device__ __forceinline__ void list_append_items(uint32_t *list, uint32_t mask, uint32_t first,
                                                  unsigned long long *counter2) {
    __shared__ uint32_t s_warp[8];
    __shared__ unsigned long long s_base;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t c = __popc(mask);
    uint32_t inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += v;
    }
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        const uint32_t w = lane < 8 ? s_warp[lane] : 0;
        uint32_t wi = w;
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += v;
        }
        if (lane < 8) s_warp[lane] = wi - w;
        if (lane == 7 && wi) {
            s_base = atomicAdd(reinterpret_cast<unsigned long long *>(list), (unsigned long long)wi);
            if (counter2) atomicAdd(counter2, (unsigned long long)wi);
        }
    }
    __syncthreads();
    if (c) {
        uint64_t slot = LVX_LIST_HDR + s_base + s_warp[warp] + (inc - c);
#pragma unroll
        for (int k = 0; k < ITEMS; k++)
            if ((mask >> k) & 1u) list[slot++] = first + k;
    }
}

// lv/culling.py:130-140 dilate_bits, then `& occ_bits` (224).  Four x-adjacent voxels per thread
// (128-bit load of the packed words, 32-bit load/store of the byte masks); the 26-neighbour search
// only runs for occupied voxels that are not visible themselves while anything is solid at all.
__global__ void __launch_bounds__(256)
k_dilate(const uint32_t *__restrict__ base, const uint8_t *__restrict__ vis, int res, int64_t V,
         uint8_t *__restrict__ out, uint32_t *__restrict__ vis_list, uint64_t *__restrict__ stats) {
    const int64_t idx0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;     // V is a multiple of 4 (res >= 2)
    uint32_t mask = 0;
    if (idx0 < V) {
        const uint4 w = *reinterpret_cast<const uint4 *>(base + idx0);
        const uchar4 vv = *reinterpret_cast<const uchar4 *>(vis + idx0);
        const uint32_t occ[4] = {w.x >> 16, w.y >> 16, w.z >> 16, w.w >> 16};
        const uint8_t vs[4] = {vv.x, vv.y, vv.z, vv.w};
        const bool any_solid = stats[LVX_ST_SOLID] != 0;
#pragma unroll
        for (int k = 0; k < 4; k++) {
            if (!occ[k]) continue;
            bool v = vs[k] != 0 || !any_solid;     // (k_visibility does not run when nothing is solid)
            if (!v) {
                const int64_t idx = idx0 + k;
                const int x = (int)(idx % res), y = (int)((idx / res) % res), z = (int)(idx / ((int64_t)res * res));
                for (int dz = -1; dz <= 1 && !v; dz++) {
                    const int Z = z + dz;
                    if (Z < 0 || Z >= res) continue;
                    for (int dy = -1; dy <= 1 && !v; dy++) {
                        const int Y = y + dy;
                        if (Y < 0 || Y >= res) continue;
                        for (int dx = -1; dx <= 1; dx++) {
                            const int X = x + dx;
                            if (X < 0 || X >= res) continue;
                            if (vis[X + (int64_t)res * (Y + (int64_t)res * Z)]) { v = true; break; }
                        }
                    }
                }
            }
            if (v) mask |= 1u << k;
        }
        *reinterpret_cast<uchar4 *>(out + idx0) = make_uchar4(mask & 1u, (mask >> 1) & 1u, (mask >> 2) & 1u, (mask >> 3) & 1u);
    }
    list_append_items<4>(vis_list, mask, (uint32_t)idx0, (unsigned long long *)&stats[LVX_ST_VISIBLE]);
}

__global__ void __launch_bounds__(256)
k_occupied(const uint32_t *__restrict__ base, int64_t V, uint8_t *__restrict__ out, uint32_t *__restrict__ vis_list,
           uint64_t *__restrict__ stats) {
    const int64_t idx0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
    uint32_t mask = 0;
    if (idx0 < V) {
        const uint4 w = *reinterpret_cast<const uint4 *>(base + idx0);
        mask = ((w.x >> 16) ? 1u : 0u) | ((w.y >> 16) ? 2u : 0u) | ((w.z >> 16) ? 4u : 0u) | ((w.w >> 16) ? 8u : 0u);
        *reinterpret_cast<uchar4 *>(out + idx0) = make_uchar4(mask & 1u, (mask >> 1) & 1u, (mask >> 2) & 1u, (mask >> 3) & 1u);
    }
    const uint32_t wm = __reduce_add_sync(0xffffffffu, __popc(mask));
    if ((threadIdx.x & 31) == 0 && wm)
        atomicAdd((unsigned long long *)&stats[LVX_ST_OCCUPIED], (unsigned long long)wm);
    list_append_items<4>(vis_list, mask, (uint32_t)idx0, (unsigned long long *)&stats[LVX_ST_VISIBLE]);
}

// Screen-tile ownership (multi-GPU screen tiles): owner = visible AND the voxel's cube,
// grown by `margin`, meets the tile's sub-frustum -- the pyramid whose apex is the camera and whose four
// side planes pass through the tile's pixel EDGES (every pixel-centre ray of the tile lies inside).  A
// cube [c - h, c + h] meets the half-space {q : q.n >= 0} (q relative to the apex) iff
// (c - apex).n + h |n|_1 >= 0; passing all four tests is the usual conservative box/frustum test (it may
// keep a few cubes outside, never drops one that a ray can visit).  The A-buffer build of a rank is
// restricted to its owners; the MARCH bits stay the full culling pyramid, so every ray steps exactly as
// it does on one GPU and only ever visits voxels its rank owns.
struct TilePlanes { double apex[3]; double n[4][3]; double h; };
__global__ void __launch_bounds__(256)
k_owner(const uint8_t *__restrict__ cull0, int res, int64_t V, const TilePlanes P, uint8_t *__restrict__ out,
        uint32_t *__restrict__ list, uint64_t *__restrict__ stats) {
    const int64_t idx0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
    uint32_t mask = 0;
    if (idx0 < V) {
        const uchar4 c = *reinterpret_cast<const uchar4 *>(cull0 + idx0);
        const uint8_t vs[4] = {c.x, c.y, c.z, c.w};
        const int x0 = (int)(idx0 % res), y = (int)((idx0 / res) % res), z = (int)(idx0 / ((int64_t)res * res));
#pragma unroll
        for (int k = 0; k < 4; k++) {
            if (!vs[k]) continue;
            const double qx = (x0 + k) + 0.5 - P.apex[0], qy = y + 0.5 - P.apex[1], qz = z + 0.5 - P.apex[2];
            bool in = true;
#pragma unroll
            for (int p = 0; p < 4; p++) {
                const double d = qx * P.n[p][0] + qy * P.n[p][1] + qz * P.n[p][2]
                                 + P.h * (fabs(P.n[p][0]) + fabs(P.n[p][1]) + fabs(P.n[p][2]));
                in = in && d >= 0.0;
            }
            if (in) mask |= 1u << k;
        }
        *reinterpret_cast<uchar4 *>(out + idx0) = make_uchar4(mask & 1u, (mask >> 1) & 1u, (mask >> 2) & 1u, (mask >> 3) & 1u);
    }
    list_append_items<4>(list, mask, (uint32_t)idx0, (unsigned long long *)&stats[LVX_ST_OWNED]);
}

// lv/culling.py:103-109: parent = OR of its 8 children
__global__ void __launch_bounds__(256)
k_ormip(const uint8_t *__restrict__ src, int rsrc, uint8_t *__restrict__ out) {
    const int rl = rsrc >> 1;
    const int64_t n = (int64_t)rl * rl * rl;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int x = (int)(i % rl), y = (int)((i / rl) % rl), z = (int)(i / ((int64_t)rl * rl));
    uint32_t m = 0;
#pragma unroll
    for (int dz = 0; dz < 2; dz++)
#pragma unroll
        for (int dy = 0; dy < 2; dy++) {
            const uchar2 w = *reinterpret_cast<const uchar2 *>(
                src + (2 * x + (int64_t)rsrc * ((2 * y + dy) + (int64_t)rsrc * (2 * z + dz))));
            m |= w.x | w.y;
        }
    out[i] = m ? 1 : 0;
}

// March table for the ray tracer: one byte per level-0 voxel = 255 if the voxel's bit is set, else
// the value lv/raytracer.py:316-326 _empty_level would return there (largest l such that the
// ancestors at levels 1..l are all clear).  One load per DDA step instead of a walk up the pyramid.
// One thread per 4 x-adjacent voxels (they share every ancestor from level 2 up).
struct MarchOffsets { uint32_t off[16]; };

// the four march bytes of voxels x0 .. x0 + 3 (bits b), which share every ancestor from level 2 up
__device__ __forceinline__ uchar4 march_four(const uint8_t *__restrict__ flat, const MarchOffsets &O, int res, int n_levels,
                                             uint32_t x0, uint32_t y, uint32_t z, uchar4 b) {
    uchar4 out = make_uchar4(255, 255, 255, 255);
    if (b.x && b.y && b.z && b.w) return out;
    int up = 0;          // result for a voxel whose level-1 parent is clear
    uint8_t p1a = 1, p1b = 1;
    if (n_levels > 1) {
        const uint32_t r1 = (uint32_t)res >> 1;
        const uint32_t i1 = O.off[1] + (x0 >> 1) + r1 * ((y >> 1) + r1 * (z >> 1));
        p1a = flat[i1]; p1b = flat[i1 + 1];
        if (!(p1a && p1b)) {
            // In an OR pyramid a set node has set ancestors only, so "ancestors 1..l all clear" holds
            // for l up to the highest clear ancestor: all levels are loaded at once (independent
            // loads, one round trip) and the clear ones counted, instead of a dependent walk upwards.
            uint32_t clear = 0;
#pragma unroll
            for (int nl = 2; nl < 11; nl++) {     // res <= 1024: at most 11 levels
                if (nl < n_levels) {
                    const uint32_t rl = (uint32_t)res >> nl;
                    if (flat[O.off[nl] + (x0 >> nl) + rl * ((y >> nl) + rl * (z >> nl))] == 0)
                        clear |= 1u << nl;
                }
            }
            up = __ffs(~(clear | 3u)) - 2;        // the level below the first set ancestor (>= 1)
        }
    }
    const uint8_t la = p1a ? 0 : (uint8_t)up, lb = p1b ? 0 : (uint8_t)up;
    if (!b.x) out.x = la;
    if (!b.y) out.y = la;
    if (!b.z) out.z = lb;
    if (!b.w) out.w = lb;
    return out;
}

// One thread per 16 x-adjacent voxels (res >= 16), which share every ancestor from level 4 up.  Most of a volume
// lies under clear 16^3 nodes: there the 16 bytes are one value -- the highest level whose ancestors are all
// clear -- and one 128-bit store; the other runs go through march_four four voxels at a time.
__global__ void __launch_bounds__(256)
k_march_levels16(const uint8_t *__restrict__ flat, const MarchOffsets O, int res, int n_levels, int64_t n16,
                 uint8_t *__restrict__ skip) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n16) return;
    const uint32_t r16 = (uint32_t)res >> 4;
    const uint32_t x0 = (uint32_t)(g % r16) << 4, y = (uint32_t)((g / r16) % res), z = (uint32_t)(g / ((int64_t)r16 * res));
    const uint4 w = *reinterpret_cast<const uint4 *>(flat + (x0 + (int64_t)res * (y + (int64_t)res * z)));
    const uint32_t r4l = (uint32_t)res >> 4;
    if (flat[O.off[4] + (x0 >> 4) + r4l * ((y >> 4) + r4l * (z >> 4))] == 0) {
        uint32_t clear = 0;
#pragma unroll
        for (int nl = 5; nl < 11; nl++) {
            if (nl < n_levels) {
                const uint32_t rl = (uint32_t)res >> nl;
                if (flat[O.off[nl] + (x0 >> nl) + rl * ((y >> nl) + rl * (z >> nl))] == 0) clear |= 1u << nl;
            }
        }
        const uint32_t up = (uint32_t)(__ffs(~(clear | 31u)) - 2);       // levels 1..4 are clear under a clear level-4 node
        const uint32_t v = up * 0x01010101u;
        *reinterpret_cast<uint4 *>(skip + 16 * g) = make_uint4(v, v, v, v);
        return;
    }
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
    uint32_t o[4];
#pragma unroll
    for (int q = 0; q < 4; q++) {
        const uchar4 b = make_uchar4(ws[q] & 0xFF, (ws[q] >> 8) & 0xFF, (ws[q] >> 16) & 0xFF, ws[q] >> 24);
        const uchar4 r = march_four(flat, O, res, n_levels, x0 + 4 * q, y, z, b);
        o[q] = (uint32_t)r.x | (uint32_t)r.y << 8 | (uint32_t)r.z << 16 | (uint32_t)r.w << 24;
    }
    *reinterpret_cast<uint4 *>(skip + 16 * g) = make_uint4(o[0], o[1], o[2], o[3]);
}

__global__ void __launch_bounds__(256)
k_march_levels(const uint8_t *__restrict__ flat, const MarchOffsets O, int res, int n_levels, int64_t n4,
               uint8_t *__restrict__ skip) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n4) return;
    const int r4 = res >> 2;
    const int x0 = (int)(g % r4) << 2, y = (int)((g / r4) % res), z = (int)(g / ((int64_t)r4 * res));
    const uchar4 b = *reinterpret_cast<const uchar4 *>(flat + (x0 + (int64_t)res * (y + (int64_t)res * z)));
    *reinterpret_cast<uchar4 *>(skip + 4 * g) = march_four(flat, O, res, n_levels, (uint32_t)x0, (uint32_t)y, (uint32_t)z, b);
}

// The top of the OR pyramid (levels of <= 16^3 nodes) in one launch: a single CTA, level after level.
struct OrTail { int64_t off[16]; int first, n_levels, res; };
__global__ void __launch_bounds__(1024)
k_ormip_tail(uint8_t *__restrict__ flat, const OrTail T) {
    for (int l = T.first; l < T.n_levels; l++) {
        const int rsrc = T.res >> (l - 1), rl = T.res >> l;
        const uint8_t *src = flat + T.off[l - 1];
        uint8_t *out = flat + T.off[l];
        for (int i = threadIdx.x; i < rl * rl * rl; i += blockDim.x) {
            const int x = i % rl, y = (i / rl) % rl, z = i / (rl * rl);
            uint32_t m = 0;
#pragma unroll
            for (int dz = 0; dz < 2; dz++)
#pragma unroll
                for (int dy = 0; dy < 2; dy++) {
                    const uchar2 w = *reinterpret_cast<const uchar2 *>(src + (2 * x + rsrc * ((2 * y + dy) + rsrc * (2 * z + dz))));
                    m |= w.x | w.y;
                }
            out[i] = m ? 1 : 0;
        }
        __syncthreads();
    }
}

static int or_mips(uint8_t *flat, int res, cudaStream_t s) {
    const LevelOffsets L = make_level_offsets(res);
    for (int l = 1; l < L.n_levels; l++) {
        const int rsrc = res >> (l - 1), rl = res >> l;
        if (rl <= 16) {     // this level and everything above it: one launch
            OrTail T;
            for (int k = 0; k < 16; k++) T.off[k] = k < L.n_levels ? L.off[k] : 0;
            T.first = l; T.n_levels = L.n_levels; T.res = res;
            k_ormip_tail<<<1, 1024, 0, s>>>(flat, T);
            break;
        }
        k_ormip<<<blocks_for((int64_t)rl * rl * rl, 256), 256, 0, s>>>(flat + L.off[l - 1], rsrc, flat + L.off[l]);
    }
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

}  // namespace lvx

using namespace lvx;

extern "C" {

int64_t lvx_cull_scratch_words(int res) {
    if (!pow2(res)) return LVX_E_ARG;
    const int64_t V = (int64_t)res * res * res;
    const int64_t rs = (res + LVX_SUPER - 1) / LVX_SUPER;
    return (V + 31) / 32 + brick_words(res, LVX_BRICK) + brick_words(res, LVX_SUPER)
           + (LVX_LIST_HDR + LVX_SOLID_CAP) + (rs * rs * rs + 3) / 4 + 1    // + solid list, super-brick flags, alignment
           + (V + LVX_LIST_HDR)                                             // + occupied-voxel list (later: long-march list)
           + rs * rs * rs * LVX_SB_ROW;                                     // + solid voxels shadowing each super-brick
}

int lvx_cull(const uint32_t *base, int res, const double *cam_voxel_host, uint32_t *solid_bits,
             uint8_t *vis_tmp, uint8_t *cull_flat, uint32_t *vis_list, uint64_t *stats, void *stream) {
    if (!pow2(res)) return LVX_E_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t V = (int64_t)res * res * res;
    // solid_bits scratch layout: [V/32 words of solid bits][8^3-brick flags][32^3-brick flags][solid list]
    // [super-brick shadow flags][V: occupied list][super-brick rows]
    uint32_t *bricks = solid_bits + (V + 31) / 32;
    uint32_t *solid_list = bricks + brick_words(res, LVX_BRICK) + brick_words(res, LVX_SUPER);
    LVX_CUDA(cudaMemsetAsync(bricks, 0, (size_t)(brick_words(res, LVX_BRICK) + brick_words(res, LVX_SUPER) + LVX_LIST_HDR) * 4, s));
    const int rs = (res + LVX_SUPER - 1) / LVX_SUPER;
    uint8_t *sb_flag = reinterpret_cast<uint8_t *>(solid_list + LVX_LIST_HDR + LVX_SOLID_CAP);
    uint32_t *occ_list = solid_list + LVX_LIST_HDR + LVX_SOLID_CAP + (rs * rs * rs + 3) / 4;
    if ((occ_list - solid_bits) & 1) occ_list++;      // its first two words become a 64-bit list counter
    uint32_t *sb_rows = occ_list + V + LVX_LIST_HDR;
    LVX_CUDA(cudaMemsetAsync(vis_tmp, 0, (size_t)V, s));
    k_solid<<<blocks_for(V, SOLID_ITEMS * 256), 256, 0, s>>>(base, res, V, solid_bits, solid_list, occ_list, stats);
    {
        const int rb = (res + LVX_BRICK - 1) / LVX_BRICK;
        k_brick_flags<<<blocks_for((int64_t)rb * rb * rb * 32, 128), 128, 0, s>>>(solid_bits, res, stats, bricks);
        k_super_flags<<<blocks_for(((int64_t)rs * rs * rs + 31) & ~31LL, 128), 128, 0, s>>>(bricks, res, stats, bricks + brick_words(res, LVX_BRICK));
    }
    k_superbrick_shadow<<<(unsigned)(rs * rs * rs), 64, 0, s>>>(solid_list, res, (float)cam_voxel_host[0],
                                                                          (float)cam_voxel_host[1], (float)cam_voxel_host[2], sb_flag, sb_rows);
    unsigned nb = 148 * 16;
    if (nb > blocks_for(V, 128)) nb = blocks_for(V, 128);
    // vis_list doubles as the "needs the fine march" list until k_dilate refills it
    LVX_CUDA(cudaMemsetAsync(vis_list, 0, 8, s));
    k_visibility<<<nb, 128, 0, s>>>(bricks, sb_flag, sb_rows, solid_list, occ_list, res, cam_voxel_host[0], cam_voxel_host[1],
                                    cam_voxel_host[2], stats, vis_tmp, vis_list);
    // the occupied list has been consumed: its memory becomes the list of candidates whose walk is long
    LVX_CUDA(cudaMemsetAsync(occ_list, 0, 8, s));
    k_march_probe<<<nb, 128, 0, s>>>(solid_bits, vis_list, res, cam_voxel_host[0], cam_voxel_host[1], cam_voxel_host[2], occ_list);
    k_march<<<nb, 128, 0, s>>>(solid_bits, bricks, occ_list, res, cam_voxel_host[0], cam_voxel_host[1],
                               cam_voxel_host[2], vis_tmp);
    LVX_CUDA(cudaMemsetAsync(vis_list, 0, 8, s));
    k_dilate<<<blocks_for(V / 4, 256), 256, 0, s>>>(base, vis_tmp, res, V, cull_flat, vis_list, stats);
    LVX_LAUNCH_CHECK();
    return or_mips(cull_flat, res, s);
}

int lvx_occupied_pyramid(const uint32_t *base, int res, uint8_t *cull_flat, uint32_t *vis_list, uint64_t *stats,
                         void *stream) {
    if (!pow2(res)) return LVX_E_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t V = (int64_t)res * res * res;
    LVX_CUDA(cudaMemsetAsync(vis_list, 0, 8, s));
    k_occupied<<<blocks_for(V / 4, 256), 256, 0, s>>>(base, V, cull_flat, vis_list, stats);
    LVX_LAUNCH_CHECK();
    return or_mips(cull_flat, res, s);
}

int lvx_tile_owners(const uint8_t *cull_flat, int res, const lvx_camera *cam, int tile_x0, int tile_y0, int tile_x1,
                    int tile_y1, double margin, uint8_t *owner_flat, uint32_t *owner_list, uint64_t *stats, void *stream) {
    if (!pow2(res) || !cull_flat || !cam || !owner_flat || !owner_list) return LVX_E_ARG;
    if (cam->width <= 0 || cam->height <= 0 || tile_x0 < 0 || tile_y0 < 0 || tile_x1 > cam->width || tile_y1 > cam->height ||
        tile_x0 > tile_x1 || tile_y0 > tile_y1 || !(margin >= 0.0)) return LVX_E_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t V = (int64_t)res * res * res;
    if (V & 3) return LVX_E_ARG;
    // lv/raytracer.py:414-423 _pixel_ray: u = (2 (px + .5) / w - 1) aspect tan, v = (1 - 2 (py + .5) / h) tan.
    // Pixel EDGES: px + .5 -> tile_x0 and tile_x1 (a half pixel wider than the outermost centres).
    const double aspect = (double)cam->width / (double)cam->height, tf = cam->tan_half_fov;
    const double u_lo = (2.0 * tile_x0 / cam->width - 1.0) * aspect * tf, u_hi = (2.0 * tile_x1 / cam->width - 1.0) * aspect * tf;
    const double v_hi = (1.0 - 2.0 * tile_y0 / cam->height) * tf, v_lo = (1.0 - 2.0 * tile_y1 / cam->height) * tf;
    TilePlanes P;
    for (int a = 0; a < 3; a++) {
        P.apex[a] = cam->pos[a];
        P.n[0][a] = cam->right[a] - u_lo * cam->fwd[a];     // q.right >= u_lo q.fwd
        P.n[1][a] = u_hi * cam->fwd[a] - cam->right[a];     // q.right <= u_hi q.fwd
        P.n[2][a] = cam->up[a] - v_lo * cam->fwd[a];
        P.n[3][a] = v_hi * cam->fwd[a] - cam->up[a];
    }
    P.h = 0.5 + margin;
    LVX_CUDA(cudaMemsetAsync(owner_list, 0, 8, s));
    k_owner<<<blocks_for(V / 4, 256), 256, 0, s>>>(cull_flat, res, V, P, owner_flat, owner_list, stats);
    LVX_LAUNCH_CHECK();
    return or_mips(owner_flat, res, s);
}

int lvx_march_levels(const uint8_t *bits_flat, int res, uint8_t *march, void *stream) {
    if (!pow2(res) || res < 4 || !bits_flat || !march) return LVX_E_ARG;
    const LevelOffsets L = make_level_offsets(res);
    MarchOffsets O;
    for (int l = 0; l < 16; l++) O.off[l] = l < L.n_levels ? (uint32_t)L.off[l] : 0;
    const int64_t n4 = L.off[1] / 4;
    if (res >= 32) k_march_levels16<<<blocks_for(n4 / 4, 256), 256, 0, (cudaStream_t)stream>>>(bits_flat, O, res, L.n_levels, n4 / 4, march);
    else k_march_levels<<<blocks_for(n4, 256), 256, 0, (cudaStream_t)stream>>>(bits_flat, O, res, L.n_levels, n4, march);
    LVX_LAUNCH_CHECK();
    return LVX_OK;
}

int64_t lvx_list_words(int64_t n_voxels) { return n_voxels + LVX_LIST_HDR; }

}  // extern "C"
