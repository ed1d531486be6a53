// spo_table.cu -- device table construction in the wrap-padded AoSoA layout.
//
//   spo_pack_table      reference SoA (coeffs.py:117-138) -> device layout,
//                       optionally split into tiles (coeffs.py:197-210)
//   spo_fill_uniform    FillSpec.random (coeffs.py:91-94) bit-identically:
//                       numpy's Philox4x64-10 bit generator (counter 0, key from
//                       SeedSequence(entropy=seed, spawn_key=(n,))), float32
//                       draw = (u32 >> 8) * 2^-24, then *2 - 1 in fp32
//   spo_fill_normal_f64 builder-defined Box-Muller N(0,1) on the same streams
//   spo_pack_kpower     B-spline device layout -> k-power form (z-cubics in
//                       the power basis; spo_b200.h SPO_TABLE_KPOWER)
//
// Every kernel walks the destination in its own layout (row-major over
// (m, i', j', k', l)) so stores are fully coalesced; each element finds its
// reference element (i'-1 mod nx, ...) and spline m*tile_size + l.
#include "spo_common.cuh"

namespace spo {

struct PackGeom {
    int nx, ny, nz, nxp, nyp, nzp, nb, tile_size, n_splines;
    long long total;  // elements in the destination
};

__device__ __forceinline__ bool dst_coords(const PackGeom &g, long long e, int *n, long long *ref_flat) {
    const int l = (int)(e % g.nb);
    long long r = e / g.nb;
    const int kp = (int)(r % g.nzp);
    r /= g.nzp;
    const int jp = (int)(r % g.nyp);
    r /= g.nyp;
    const int ip = (int)(r % g.nxp);
    const int m = (int)(r / g.nxp);
    const int spl = m * g.tile_size + l;
    if (l >= g.tile_size || spl >= g.n_splines) return false;
    const int ii = (ip + g.nx - 1) % g.nx, jj = (jp + g.ny - 1) % g.ny, kk = (kp + g.nz - 1) % g.nz;
    *n = spl;
    *ref_flat = ((long long)ii * g.ny + jj) * g.nz + kk;
    return true;
}

template <typename T>
__global__ void pack_kernel(const T *__restrict__ src, int src_npad, PackGeom g, T *__restrict__ dst) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < g.total;
         e += (long long)gridDim.x * blockDim.x) {
        int n;
        long long f;
        dst[e] = dst_coords(g, e, &n, &f) ? src[f * src_npad + n] : T(0);
    }
}

// ---- numpy Philox4x64-10 (numpy/random/src/philox/philox.h) -------------
struct U4 {
    unsigned long long v[4];
};

__device__ __forceinline__ U4 philox4x64_10(U4 c, unsigned long long k0, unsigned long long k1) {
    const unsigned long long M0 = 0xD2E7470EE14C6C93ULL, M1 = 0xCA5A826395121157ULL;
    const unsigned long long W0 = 0x9E3779B97F4A7C15ULL, W1 = 0xBB67AE8584CAA73BULL;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) {
            k0 += W0;
            k1 += W1;
        }
        const unsigned long long hi0 = __umul64hi(M0, c.v[0]), lo0 = M0 * c.v[0];
        const unsigned long long hi1 = __umul64hi(M1, c.v[2]), lo1 = M1 * c.v[2];
        U4 o;
        o.v[0] = hi1 ^ c.v[1] ^ k0;
        o.v[1] = lo1;
        o.v[2] = hi0 ^ c.v[3] ^ k1;
        o.v[3] = lo0;
        c = o;
    }
    return c;
}

// 64-bit word w of a stream whose counter starts at 0 (incremented before
// each 4-word block): block w/4 uses counter w/4 + 1.
__device__ __forceinline__ unsigned long long philox_word(unsigned long long w, unsigned long long k0,
                                                          unsigned long long k1) {
    U4 c;
    const unsigned long long b = (w >> 2) + 1ULL;
    c.v[0] = b;
    c.v[1] = (b == 0ULL) ? 1ULL : 0ULL;  // carry (never reached in practice)
    c.v[2] = 0ULL;
    c.v[3] = 0ULL;
    const U4 o = philox4x64_10(c, k0, k1);
    return o.v[w & 3];
}

__global__ void fill_uniform_kernel(const unsigned long long *__restrict__ keys, PackGeom g,
                                    float *__restrict__ dst) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < g.total;
         e += (long long)gridDim.x * blockDim.x) {
        int n;
        long long f;
        float v = 0.0f;
        if (dst_coords(g, e, &n, &f)) {
            // next_uint32: low half of word f/2 first, then its high half
            const unsigned long long w = philox_word((unsigned long long)f >> 1, keys[2 * n], keys[2 * n + 1]);
            const unsigned int u = (f & 1) ? (unsigned int)(w >> 32) : (unsigned int)(w & 0xffffffffULL);
            const float r = (float)(u >> 8) * (1.0f / 16777216.0f);
            v = __fsub_rn(__fmul_rn(r, 2.0f), 1.0f);
        }
        dst[e] = v;
    }
}

__global__ void fill_normal_kernel(const unsigned long long *__restrict__ keys, PackGeom g,
                                   double *__restrict__ dst) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < g.total;
         e += (long long)gridDim.x * blockDim.x) {
        int n;
        long long f;
        double v = 0.0;
        if (dst_coords(g, e, &n, &f)) {
            const unsigned long long k0 = keys[2 * n], k1 = keys[2 * n + 1];
            const unsigned long long w0 = philox_word(2ULL * f, k0, k1);
            const unsigned long long w1 = philox_word(2ULL * f + 1ULL, k0, k1);
            const double u0 = (double)(w0 >> 11) * (1.0 / 9007199254740992.0);
            const double u1 = (double)(w1 >> 11) * (1.0 / 9007199254740992.0);
            v = sqrt(-2.0 * log1p(-u0)) * cospi(2.0 * u1);
        }
        dst[e] = v;
    }
}

// driver.py:174-179 _position_stream: Philox(counter=[0, walker, iteration,
// kernel_id], key=[seed, 0]).random((ns, 3)) * lengths.  Element e = 3 s + axis
// is 64-bit word e of the stream: block e/4 uses counter[0] = e/4 + 1 (numpy
// increments before generating), lane e % 4; next_double = (w >> 11) * 2^-53.
__global__ void positions_kernel(unsigned long long seed, long long walker0, long long n_walkers,
                                 unsigned long long iteration, unsigned long long kernel_id, long long ns,
                                 double lx, double ly, double lz, double *__restrict__ out) {
    const long long total = n_walkers * ns * 3;
    for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < total;
         g += (long long)gridDim.x * blockDim.x) {
        const long long w = g / (ns * 3);
        const unsigned long long e = (unsigned long long)(g - w * ns * 3);
        U4 c;
        c.v[0] = (e >> 2) + 1ULL;
        c.v[1] = (unsigned long long)(walker0 + w);
        c.v[2] = iteration;
        c.v[3] = kernel_id;
        const U4 o = philox4x64_10(c, seed, 0ULL);
        const double u = (double)(o.v[e & 3] >> 11) * (1.0 / 9007199254740992.0);
        const int axis = (int)(e % 3);
        out[g] = __dmul_rn(u, axis == 0 ? lx : (axis == 1 ? ly : lz));
    }
}

static int make_pack_geom(int dtype, int32_t n_splines, const int32_t *n3, int32_t tile_size,
                          int32_t nb, int32_t n_tiles, PackGeom *g) {
    TableGeom t;
    int rc = make_geom(n3, nb, n_tiles, dtype, &t);
    if (rc) return rc;
    if (n_splines < 1) return fail(SPO_ERR_CONFIG, "n_splines=%d must be >= 1", n_splines);
    if (tile_size < 1 || tile_size > nb)
        return fail(SPO_ERR_CONFIG, "tile_size=%d must be in [1, nb=%d]", tile_size, nb);
    if ((long long)tile_size * n_tiles < n_splines)
        return fail(SPO_ERR_CONFIG, "%d tiles of %d splines cannot hold %d splines", n_tiles,
                    tile_size, n_splines);
    g->nx = t.nx;
    g->ny = t.ny;
    g->nz = t.nz;
    g->nxp = t.nxp;
    g->nyp = t.nyp;
    g->nzp = t.nzp;
    g->nb = nb;
    g->tile_size = tile_size;
    g->n_splines = n_splines;
    g->total = t.tile_stride * n_tiles;
    return SPO_OK;
}

// k-power form: dst element (m, i', j', 4 k0 + r, l) from the four B-spline
// rows k0..k0+3 of (m, i', j') in src.  Computed in fp64 (exact sums of fp32
// inputs up to the divisions), rounded once.  With s(t) = sum_k a_k(t) c_k and
// grid.py:127-130's a_k: 6 s = (c0 + 4c1 + c2) + 3t (c2 - c0)
//   + 3t^2 (c0 - 2c1 + c2) + t^3 (-c0 + 3c1 - 3c2 + c3).
template <typename T>
__global__ void kpower_kernel(const T *__restrict__ src, long long total, int nb, int nz, T *__restrict__ dst) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const int l = (int)(e % nb);
        const long long row = e / nb;               // (m, i', j') * 4nz + 4 k0 + r
        const int kr = (int)(row % (4LL * nz));
        const long long ij = row / (4LL * nz);      // (m, i', j') flat
        const int k0 = kr >> 2, r = kr & 3;
        const T *c = src + (ij * (nz + 3) + k0) * (long long)nb + l;
        const double c0 = (double)c[0], c1 = (double)c[nb], c2 = (double)c[2LL * nb], c3 = (double)c[3LL * nb];
        double q;
        // explicit round-to-nearest steps (no FMA contraction): the order of
        // the expressions in spo_b200.h, reproducible on the host
        switch (r) {
            case 0: q = __ddiv_rn(__dadd_rn(__dadd_rn(c0, __dmul_rn(4.0, c1)), c2), 6.0); break;
            case 1: q = __ddiv_rn(__dsub_rn(c2, c0), 2.0); break;
            case 2: q = __ddiv_rn(__dadd_rn(__dsub_rn(c0, __dmul_rn(2.0, c1)), c2), 2.0); break;
            default: q = __ddiv_rn(__dadd_rn(__dsub_rn(c3, c0), __dmul_rn(3.0, __dsub_rn(c1, c2))), 6.0); break;
        }
        dst[e] = (T)q;
    }
}

static unsigned grid_for(long long total) {
    long long b = (total + 255) / 256;
    return (unsigned)(b < 148LL * 64 ? (b < 1 ? 1 : b) : 148LL * 64);
}

}  // namespace spo

using namespace spo;

extern "C" int spo_pack_table(int dtype, const void *src, int32_t src_npad, int32_t n_splines,
                              const int32_t *n3, int32_t tile_size, int32_t nb, int32_t n_tiles,
                              void *dst, void *stream) {
    if (dtype != SPO_F32 && dtype != SPO_F64) return fail(SPO_ERR_CONTRACT, "unknown dtype %d", dtype);
    PackGeom g;
    int rc = make_pack_geom(dtype, n_splines, n3, tile_size, nb, n_tiles, &g);
    if (rc) return rc;
    if (!src || !dst) return fail(SPO_ERR_CONTRACT, "NULL table pointer");
    if (src_npad < n_splines) return fail(SPO_ERR_CONTRACT, "src_npad=%d < n_splines=%d", src_npad, n_splines);
    rc = bind_device(dst);
    if (rc) return rc;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (dtype == SPO_F64)
        pack_kernel<double><<<grid_for(g.total), 256, 0, st>>>((const double *)src, src_npad, g, (double *)dst);
    else
        pack_kernel<float><<<grid_for(g.total), 256, 0, st>>>((const float *)src, src_npad, g, (float *)dst);
    return check_launch("spo_pack_table");
}

extern "C" int spo_pack_kpower(int dtype, const void *src, const int32_t *n3, int32_t nb, int32_t n_tiles,
                               void *dst, void *stream) {
    if (dtype != SPO_F32 && dtype != SPO_F64) return fail(SPO_ERR_CONTRACT, "unknown dtype %d", dtype);
    TableGeom t;
    int rc = make_geom(n3, nb, n_tiles, dtype, &t, true);
    if (rc) return rc;
    if (!src || !dst) return fail(SPO_ERR_CONTRACT, "NULL table pointer");
    if (!aligned16(src) || !aligned16(dst)) return fail(SPO_ERR_CONTRACT, "tables must be 16-byte aligned");
    rc = bind_device(dst);
    if (rc) return rc;
    if ((rc = check_on_device(src, "src table"))) return rc;
    const long long total = t.tile_stride * n_tiles;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (dtype == SPO_F64)
        kpower_kernel<double><<<grid_for(total), 256, 0, st>>>((const double *)src, total, nb, t.nz, (double *)dst);
    else
        kpower_kernel<float><<<grid_for(total), 256, 0, st>>>((const float *)src, total, nb, t.nz, (float *)dst);
    return check_launch("spo_pack_kpower");
}

extern "C" int spo_fill_uniform(const uint64_t *keys, int32_t n_splines, const int32_t *n3,
                                int32_t tile_size, int32_t nb, int32_t n_tiles, float *dst,
                                void *stream) {
    PackGeom g;
    int rc = make_pack_geom(SPO_F32, n_splines, n3, tile_size, nb, n_tiles, &g);
    if (rc) return rc;
    if (!keys || !dst) return fail(SPO_ERR_CONTRACT, "NULL pointer");
    rc = bind_device(dst);
    if (rc) return rc;
    fill_uniform_kernel<<<grid_for(g.total), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
        reinterpret_cast<const unsigned long long *>(keys), g, dst);
    return check_launch("spo_fill_uniform");
}

extern "C" int spo_fill_normal_f64(const uint64_t *keys, int32_t n_splines, const int32_t *n3,
                                   int32_t tile_size, int32_t nb, int32_t n_tiles, double *dst,
                                   void *stream) {
    PackGeom g;
    int rc = make_pack_geom(SPO_F64, n_splines, n3, tile_size, nb, n_tiles, &g);
    if (rc) return rc;
    if (!keys || !dst) return fail(SPO_ERR_CONTRACT, "NULL pointer");
    rc = bind_device(dst);
    if (rc) return rc;
    fill_normal_kernel<<<grid_for(g.total), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
        reinterpret_cast<const unsigned long long *>(keys), g, dst);
    return check_launch("spo_fill_normal_f64");
}

extern "C" int spo_fill_positions(uint64_t seed, int64_t walker0, int64_t n_walkers, uint64_t iteration,
                                  uint64_t kernel_id, int64_t ns, const double *lengths3, double *out,
                                  void *stream) {
    if (n_walkers < 0 || ns < 0) return fail(SPO_ERR_CONTRACT, "negative walker or sample count");
    if (n_walkers == 0 || ns == 0) return ok();
    if (!out || !lengths3) return fail(SPO_ERR_CONTRACT, "NULL pointer");
    const int rc = bind_device(out);
    if (rc) return rc;
    const long long total = n_walkers * ns * 3;
    positions_kernel<<<grid_for(total), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
        seed, walker0, n_walkers, iteration, kernel_id, ns, lengths3[0], lengths3[1], lengths3[2], out);
    return check_launch("spo_fill_positions");
}
