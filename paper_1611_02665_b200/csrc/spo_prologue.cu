// spo_prologue.cu -- standalone per-position prologue (kernels.py:132-140 _prep).
// The eval kernels fuse the same device functions; this entry point exposes
// them for map_to_grid / basis_weights and the bit-exact index tests.
#include "spo_common.cuh"
#include "spo_prologue.cuh"

namespace spo {

template <typename T>
__global__ void prologue_kernel(GridArgs g, const double *__restrict__ pos, long long n,
                                int *__restrict__ idx, double *__restrict__ t, T *__restrict__ w) {
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n;
         p += (long long)gridDim.x * blockDim.x) {
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
            double tt;
            const int i = map_axis(pos[3 * p + ax], g.dinv[ax], g.cnt[ax], &tt);
            if (idx) idx[3 * p + ax] = i;
            if (t) t[3 * p + ax] = tt;
            if (w) {
                T ww[12];
                axis_weights<T>(tt, g.dinv[ax], g.delta[ax], ww);
#pragma unroll
                for (int e = 0; e < 12; ++e) w[(3 * p + ax) * 12 + e] = ww[e];
            }
        }
    }
}

template <typename T>
__global__ void weights_kernel(const double *__restrict__ t, long long n, double dinv, double delta,
                               T *__restrict__ w) {
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n;
         p += (long long)gridDim.x * blockDim.x) {
        T ww[12];
        axis_weights<T>(t[p], dinv, delta, ww);
#pragma unroll
        for (int e = 0; e < 12; ++e) w[p * 12 + e] = ww[e];
    }
}

}  // namespace spo

using namespace spo;

extern "C" int spo_basis_weights(int dtype, const double *t, int64_t n, double dinv, double delta,
                                 void *w, void *stream) {
    if (dtype != SPO_F32 && dtype != SPO_F64) return fail(SPO_ERR_CONTRACT, "unknown dtype %d", dtype);
    if (n < 0) return fail(SPO_ERR_CONTRACT, "n < 0");
    if (n == 0) return ok();
    if (!t || !w) return fail(SPO_ERR_CONTRACT, "NULL pointer");
    if (!(dinv > 0.0) || !(delta > 0.0)) return fail(SPO_ERR_DOMAIN, "spacing must be positive");
    int rc = bind_device(w);
    if (rc) return rc;
    long long blocks = (n + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (dtype == SPO_F64)
        weights_kernel<double><<<(unsigned)blocks, 256, 0, st>>>(t, n, dinv, delta, (double *)w);
    else
        weights_kernel<float><<<(unsigned)blocks, 256, 0, st>>>(t, n, dinv, delta, (float *)w);
    return check_launch("spo_basis_weights");
}

extern "C" int spo_prologue(int dtype, const int32_t *n3, const double *dinv3, const double *delta3,
                            const double *pos, int64_t n_pos, int32_t *idx, double *t, void *w,
                            void *stream) {
    if (dtype != SPO_F32 && dtype != SPO_F64) return fail(SPO_ERR_CONTRACT, "unknown dtype %d", dtype);
    if (!n3 || !dinv3 || !delta3) return fail(SPO_ERR_CONTRACT, "NULL grid argument");
    if (n_pos < 0) return fail(SPO_ERR_CONTRACT, "n_pos < 0");
    if (n_pos == 0) return ok();
    if (!pos) return fail(SPO_ERR_CONTRACT, "NULL positions");
    GridArgs g;
    for (int ax = 0; ax < 3; ++ax) {
        if (n3[ax] < 1 || !(dinv3[ax] > 0.0) || !(delta3[ax] > 0.0))
            return fail(SPO_ERR_CONFIG, "invalid grid on axis %d", ax);
        g.dinv[ax] = dinv3[ax];
        g.cnt[ax] = (double)n3[ax];
        g.delta[ax] = delta3[ax];
        g.n[ax] = n3[ax];
    }
    int rc = bind_device(pos);
    if (rc) return rc;
    long long blocks = (n_pos + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (dtype == SPO_F64)
        prologue_kernel<double><<<(unsigned)blocks, 256, 0, st>>>(g, pos, n_pos, idx, t, (double *)w);
    else
        prologue_kernel<float><<<(unsigned)blocks, 256, 0, st>>>(g, pos, n_pos, idx, t, (float *)w);
    return check_launch("spo_prologue");
}
