/*
 * spo_b200.h -- C ABI of the B200-native tricubic B-spline SPO evaluator
 * (libspo_b200.so, built for sm_100a).
 *
 * This is the drop-in boundary for the reference's compiled hot path.  The
 * reference (bspb, /root/reference/pkg/src/bspb) crosses from Python into
 * numba-compiled code at exactly these calls:
 *
 *   spo_eval        replaces kernels.py:357-381  _batch_{v,vgl,vgh}_soa(data,
 *                   dxi, dyi, dzi, pos, v[, g, l | g, h]) -- the per-batch
 *                   entry the dispatcher kernels.py:445-473 (eval_batch) calls,
 *                   including the tiled loop kernels.py:452-457.  Unlike the
 *                   reference (which keeps only the last sample, kernels.py:
 *                   353-354) every position gets its own output block.
 *   spo_prologue    replaces kernels.py:132-140 (_prep) = grid.py:109-121
 *                   (_map_axis) + grid.py:124-139 (_fill_axis_weights); used by
 *                   map_to_grid / basis_weights (grid.py:155-213) and the
 *                   bit-exact index tests.
 *   spo_basis_weights  replaces grid.py:180-203 (basis_weights[_batch]).
 *   spo_pack_kpower  beyond the reference: the k-power form of a device
 *                   table (z-cubics in the power basis, SPO_TABLE_KPOWER),
 *                   the FAST kernels' cheaper table form.
 *   spo_pack_table  replaces the host table layout of coeffs.py:117-138 /
 *                   141-158 (+ tile_table 197-210): uploads a reference SoA
 *                   table into the device's wrap-padded AoSoA layout.
 *   spo_fill_uniform  replaces coeffs.py:80-94 + 165-185 (FillSpec.random +
 *                   build_table): numpy Philox4x64 streams, bit-identical,
 *                   generated straight into the device layout.
 *   spo_fill_positions  replaces driver.py:174-193 (generate_positions): the
 *                   walker Philox position streams, bit-identical, on device.
 *   spo_fill_normal_f64  builder-defined N(0,1) fill for the fp64 config
 *                   (no reference equivalent).
 *   spo_eval_lanes  replaces the shared-output tile loop of the nested driver
 *                   (driver.py:349-434) across GPUs: spo_eval storing only
 *                   lanes [0, lane_limit) into (possibly peer) memory.
 *   spo_eval_ratios beyond the reference: the consumer's contraction of every
 *                   stream with a coefficient row, fused into the kernel.
 *   spo_eval_path   which kernel spo_eval runs (no launch).
 *   spo_last_error  error text for the last failing call on this thread; the
 *                   Python host maps codes to the reference's exception types
 *                   (errors.py:4-17).
 *
 * Conventions: plain pointers and sizes only; every device pointer is a CUDA
 * device address owned by the caller; `stream` is a cudaStream_t (NULL = the
 * legacy default stream).  Calls are asynchronous and stream-ordered; none
 * allocates device memory or synchronises.  Reentrant: no global mutable state
 * except the thread-local error string.
 *
 * Device table layout (dtype T = float or double):
 *   table[m][i'][j'][k'][l],  m < n_tiles, i' < nx+3, j' < ny+3, k' < nz+3,
 *   l < nb (row length; multiple of 32 floats / 16 doubles = 128 bytes),
 *   table[m][i'][j'][k'][l] = ref[(i'-1) mod nx][(j'-1) mod ny][(k'-1) mod nz]
 *                                [m*tile_size + l]   (0 for padding lanes)
 *   so the stencil of (i0,j0,k0) is rows i0..i0+3 x j0..j0+3 x k0..k0+3 with no
 *   modulo, reproducing kernels.py:153-157.
 *
 * Output layout of spo_eval: element (position p, stream s, lane L) at
 *   out[o(p)*out_pos_stride + s*out_stream_stride + L],  L = m*nb + l,
 *   o(p) = out_index ? out_index[p] : p.   Streams in reference order
 *   (kernels.py:46-51): V: v | VGL: v gx gy gz l | VGH: v gx gy gz hxx hxy
 *   hxz hyy hyz hzz.  Strides and `out` must be 16-byte aligned.
 */
#ifndef SPO_B200_H
#define SPO_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPO_ABI_VERSION 6

/* kernel kinds: KernelKind (kernels.py:26-51) */
#define SPO_KIND_V 0
#define SPO_KIND_VGL 1
#define SPO_KIND_VGH 2

/* coefficient / output dtypes */
#define SPO_F32 0
#define SPO_F64 1

/* arithmetic modes (fp32 only) */
#define SPO_MODE_FAST 0   /* separable FMA accumulation (k, then j, then i)        */
#define SPO_MODE_STRICT 1 /* reference order, fp32 mul then add, no FMA: bitwise
                             equal to kernels.py:143-247                         */
/*
 * Table-form flag, OR-ed into `mode` (FAST only): `table` is in the k-power
 * form built by spo_pack_kpower -- per (m, i', j') the rows 4*k0 + r, r < 4,
 * hold the power-basis coefficients of the z-cubic of cell k0,
 *   q0 = (c0 + 4 c1 + c2)/6, q1 = (c2 - c0)/2, q2 = (c0 - 2 c1 + c2)/2,
 *   q3 = (c3 - c0)/6 + (c1 - c2)/2      (c_r = B-spline row k0 + r),
 * so sum_k a_k(t) c_k = q0 + t q1 + t^2 q2 + t^3 q3 for the basis of
 * grid.py:127-130.  The z-sums then cost 7 FMAs per row group instead of 12
 * (VGH: 248 instead of 328 FMAs per orbital); the table is 4 nz / (nz + 3)
 * times larger.  Results are within the FAST tolerance of the oracle, not
 * bitwise equal to the B-spline form (every path is bitwise equal to every
 * other path on the same form).
 */
#define SPO_TABLE_KPOWER 0x100

/* return codes */
#define SPO_OK 0
#define SPO_ERR_CONTRACT 1 /* -> ContractError: shapes, strides, alignment      */
#define SPO_ERR_DOMAIN 2   /* -> DomainError                                     */
#define SPO_ERR_CONFIG 3   /* -> ConfigError: tiling / unsupported combination   */
#define SPO_ERR_CUDA 4     /* CUDA launch/runtime failure                        */

int spo_abi_version(void);
const char *spo_last_error(void);

/*
 * Evaluate `kind` at n_pos positions (pos: device, [n_pos][3] float64).
 *   n3      host int32[3]   grid counts nx, ny, nz (GridSpec.counts)
 *   dinv3   host double[3]  1/dx, 1/dy, 1/dz exactly as GridSpec.inverse_spacings
 *   delta3  host double[3]  dx, dy, dz (fp64 weights use the oracle form /delta)
 *   status  device int32 or NULL: OR-ed with 1 when a position is non-finite
 *           (that position's outputs are NaN), so callers can raise DomainError
 *           without a synchronising pre-check.
 *   workspace, workspace_bytes
 *           device scratch owned by the caller, at least
 *           spo_eval_workspace_bytes(kind, dtype, mode, n_pos) bytes, 16-byte
 *           aligned, not shared with a concurrent call.  With it, FAST calls
 *           (fp32 and fp64) run the TMA-pipelined kernels: the line-window
 *           kernel for dense batches (VGL/VGH: >= 1 position per grid cell,
 *           V: >= 2; planes shared along grid lines), else the per-position
 *           kernel; with NULL
 *           they run the generic kernel.  Bitwise identical results either way
 *           (spo_eval_path tells which one runs).
 */
int spo_eval(int kind, int dtype, int mode, const void *table, const int32_t *n3, int32_t nb,
             int32_t n_tiles, const double *dinv3, const double *delta3, const double *pos,
             int64_t n_pos, void *out, int64_t out_pos_stride, int64_t out_stream_stride,
             const int64_t *out_index, int32_t *status, void *workspace, int64_t workspace_bytes,
             void *stream);

/*
 * spo_eval writing only output lanes [0, lane_limit) (1 <= lane_limit <= the
 * table's lanes) into `out`, which may live on ANOTHER GPU: the launch device
 * is the table's, and `out` may be peer memory it can reach (same process:
 * peer access is enabled here; another process: an IPC mapping).  This is
 * the fused evaluate + gather of the orbital-sharded mode:
 * rank r passes root_out + lo_r with lane_limit = its n_r splines and the
 * root's strides, so its kernel's output stores travel over NVLink straight
 * into the root's [P][S][N] buffer -- no gather buffer, no collective, no
 * permute.  Lanes must equal spline indices (untiled table, or tiles with no
 * padding lanes); out + lane stores need the usual 16-byte alignment.
 */
int spo_eval_lanes(int kind, int dtype, int mode, const void *table, const int32_t *n3, int32_t nb,
                   int32_t n_tiles, const double *dinv3, const double *delta3, const double *pos,
                   int64_t n_pos, void *out, int64_t out_pos_stride, int64_t out_stream_stride,
                   int64_t lane_limit, const int64_t *out_index, int32_t *status, void *workspace,
                   int64_t workspace_bytes, void *stream);

/*
 * Which kernel spo_eval runs for this request (no launch, no device needed):
 *   SPO_PATH_GENERIC  one-pass kernel (strict mode, no workspace, small batches)
 *   SPO_PATH_TMA      per-position TMA pipeline (spo_eval_tma.cu)
 *   SPO_PATH_LINE     line kernel: 4x4-row planes shared along grid lines
 *                     (j0, k0), for dense batches: VGL/VGH from 4 positions
 *                     per grid cell, V from 2.8 (fp64: 4) (k-power form: 1
 *                     and 2) (spo_eval_line.cu)
 *   SPO_PATH_WINDOW   its window variants (B-spline table form): (2+3) x
 *                     (2+3)-row planes shared by the positions of 2 x 2
 *                     (j0, k0) cells, for VGL/VGH from 0.3 positions per cell,
 *                     V from 0.4; for V from 1.1 (fp64: 1.3) per cell, (2+3) x 4-row
 *                     planes of two lines along j read once per group of
 *                     positions
 *   SPO_LINE=0/1/2 in the environment forces TMA / line / window.
 * -1 on bad arguments.  All paths give bitwise identical results.
 */
#define SPO_PATH_GENERIC 0
#define SPO_PATH_TMA 1
#define SPO_PATH_LINE 2
#define SPO_PATH_WINDOW 3
int spo_eval_path(int kind, int dtype, int mode, const int32_t *n3, int32_t nb, int32_t n_tiles, int64_t n_pos,
                  int64_t workspace_bytes);

/* Workspace spo_eval wants for this request (0 = none used, -1 = bad args). */
int64_t spo_eval_workspace_bytes(int kind, int dtype, int mode, int64_t n_pos);

/*
 * Fused consumer epilogue (beyond the reference): the
 * determinant-ratio style contraction of every output stream with a
 * per-position coefficient row, without writing the [P][S][lanes] outputs:
 *   ratios[p][s] = sum_n stream_s(p, n) * coef[p * coef_stride + lane(n)]
 * accumulated in fp64 (per-chunk partials reduced in a fixed order:
 * deterministic).  coef (device, table dtype) is in output-lane layout with
 * zeros in padding lanes; ratios (device) is [n_pos][S] float64.  Needs
 * spo_eval_ratios_workspace_bytes() of workspace; rows must be multiples of
 * 512 bytes (tiles of 128 fp32 / 64 fp64 lanes, or untiled N padded so).
 */
int64_t spo_eval_ratios_workspace_bytes(int kind, int dtype, int32_t nb, int32_t n_tiles, int64_t n_pos);
int spo_eval_ratios(int kind, int dtype, const void *table, const int32_t *n3, int32_t nb, int32_t n_tiles,
                    const double *dinv3, const double *delta3, const double *pos, int64_t n_pos,
                    const void *coef, int64_t coef_stride, double *ratios, int32_t *status,
                    void *workspace, int64_t workspace_bytes, void *stream);

/*
 * Per-position prologue: idx [n_pos][3] int32 (i0, j0, k0), t [n_pos][3]
 * float64, w [n_pos][3][3][4] of dtype (axis, {a, da, d2a}, 4): fp32 = grid.py
 * form (bit-exact), fp64 = oracle.py:20-42 form.  Any output may be NULL.
 */
int spo_prologue(int dtype, const int32_t *n3, const double *dinv3, const double *delta3,
                 const double *pos, int64_t n_pos, int32_t *idx, double *t, void *w,
                 void *stream);

/*
 * Basis weights for n offsets t (device float64, each in [0,1)) at one
 * spacing: w [n][3][4] of dtype; fp32 = grid.py:124-139 with dinv (bit-exact),
 * fp64 = oracle.py:20-42 with delta.  Replaces grid.py:180-203.
 */
int spo_basis_weights(int dtype, const double *t, int64_t n, double dinv, double delta, void *w,
                      void *stream);

/*
 * Pack a device copy of a reference SoA table src[nx][ny][nz][src_npad]
 * (dtype) holding n_splines splines into the wrap-padded device layout with
 * n_tiles tiles of tile_size splines, rows of nb >= tile_size lanes.
 */
int spo_pack_table(int dtype, const void *src, int32_t src_npad, int32_t n_splines,
                   const int32_t *n3, int32_t tile_size, int32_t nb, int32_t n_tiles, void *dst,
                   void *stream);

/*
 * Build the k-power form (see SPO_TABLE_KPOWER) of a device table `src` in
 * the B-spline layout above: dst[m][i'][j'][4*k0 + r][l], i' < nx+3, j' < ny+3,
 * k0 < nz, r < 4, computed in fp64 and rounded once to the table dtype.  Same
 * tiling (nb, n_tiles) as src; dst holds n_tiles*(nx+3)*(ny+3)*4nz*nb elements.
 */
int spo_pack_kpower(int dtype, const void *src, const int32_t *n3, int32_t nb, int32_t n_tiles, void *dst,
                    void *stream);

/*
 * Fill the device layout with FillSpec.random(seed) values: spline n uses the
 * numpy Philox4x64-10 stream with key keys[2n], keys[2n+1] (device uint64,
 * = SeedSequence(entropy=seed, spawn_key=(n,)).generate_state(2, uint64)),
 * counter 0, Generator.random(float32) * 2 - 1 over the C-order (nx,ny,nz) grid.
 */
int spo_fill_uniform(const uint64_t *keys, int32_t n_splines, const int32_t *n3,
                     int32_t tile_size, int32_t nb, int32_t n_tiles, float *dst, void *stream);

/*
 * Builder-defined fp64 N(0,1) fill (config 5): element e of spline n is
 * sqrt(-2 ln(1-u0)) * cos(2 pi u1), u0/u1 = the 53-bit doubles of 64-bit words
 * 2e, 2e+1 of the same Philox stream as spo_fill_uniform.
 */
int spo_fill_normal_f64(const uint64_t *keys, int32_t n_splines, const int32_t *n3,
                        int32_t tile_size, int32_t nb, int32_t n_tiles, double *dst,
                        void *stream);

/*
 * Walker position streams generated on the device, bit-identical to the
 * reference's driver.py:174-179 _position_stream(seed, walker, iteration,
 * kernel_id, ns, grid) for walkers walker0 .. walker0+n_walkers-1:
 * out [n_walkers*ns][3] float64 (device), lengths3 = GridSpec.lengths (host).
 */
int spo_fill_positions(uint64_t seed, int64_t walker0, int64_t n_walkers, uint64_t iteration,
                       uint64_t kernel_id, int64_t ns, const double *lengths3, double *out,
                       void *stream);

#ifdef __cplusplus
}
#endif
#endif /* SPO_B200_H */
