// spo_eval_line.cu -- the line-window kernel: the FAST path for dense VGL /
// VGH batches (fp32 and fp64).  Same per-orbital arithmetic as
// spo_eval_tma.cu (bitwise), different data movement: stencil planes are
// shared between positions.
//
// Position p's 4x4x4 stencil is four planes i0..i0+3 of 4(j) x 4(k) rows.  Two
// positions on the same grid line (j0, k0) with i0 values less than 4 apart
// share planes.  So:
//
//  1. line_keys_kernel + cub radix sort + line_records_kernel +
//     line_runs_kernel: positions are sorted by (spatial block, j0, k0, i0) --
//     the 4x4x4 block order of spo_eval_tma.cu's bucketing for L2 locality,
//     and inside a block whole lines in increasing i0 -- into records (36
//     weights, cell, original index); every run of BPL sorted positions gets
//     the list of planes it needs in load order and each record the number of
//     its i0 plane within that list.
//  2. line_kernel: persistent CTAs (one per SM).  A work item is (unit u = a
//     512-byte slice of every table row: 128 fp32 / 64 fp64 lanes, run), handed
//     out by a global ticket in unit-major order.  A producer warp loads each
//     plane of the run ONCE (one 16-row TMA box) into a 24-slot shared-memory
//     ring; consumer warp g evaluates positions g, g + CONS, ... of the run
//     from the ring (warp-specialised: the producer warpgroup hands its
//     registers to the consumers with setmaxnreg).  With one position per cell along a line, a position
//     needs ~1.2 new planes instead of 4: L2->SM traffic drops ~3.4x.
//
// Synchronisation: one full mbarrier per slot (TMA complete_tx); the producer
// publishes how many planes are armed (`issued`), each consumer the first
// plane it will still need (`relw[g]`); see the kernel body for why neither
// side can alias an mbarrier phase or deadlock.
#include <cuda.h>

#include <cub/device/device_radix_sort.cuh>

#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "spo_common.cuh"
#include "spo_prologue.cuh"
#include "spo_tma.cuh"

namespace spo {
namespace line {

using namespace tma;

constexpr int ROWB = 512;                        // unit bytes per table row
constexpr int BOXB = 512;                        // TMA box width in bytes
static_assert(ROWB == BOXB, "one TMA box per plane");
constexpr int BOX = 16 * BOXB;                   // bytes per box (16 rows)
#ifndef SPO_LINE_BPL
#define SPO_LINE_BPL 64
#endif
#ifndef SPO_LINE_R32
#define SPO_LINE_R32 24
#endif
#ifndef SPO_LINE_R64
#define SPO_LINE_R64 22
#endif
constexpr int BPL = SPO_LINE_BPL;                // positions per item (run)
constexpr int PL = 4 * BPL + 4;                  // plane-list ints per run: count, planes, pad
constexpr int PLB = PL * 4;                      // plane-list bytes per run (16-byte multiple)
#ifndef SPO_WX_SMEM
#define SPO_WX_SMEM 0  // 1: every VGL / VGH consumer reads its x weights per slab from shared memory
#endif
#ifndef SPO_SPIN_NS
#define SPO_SPIN_NS 256
#endif
constexpr unsigned SPIN_NS = SPO_SPIN_NS;        // back-off of the issued / release polls
constexpr int PBATCH = 4;                        // planes issued together by the producer lanes
constexpr int WS_HEADER = 1024;                  // ticket @0
constexpr int NBK = 4;                           // spatial blocks per axis (as spo_eval_tma.cu)
constexpr int MAX_AXIS = 256;                    // cell indices fit the 10-bit fields of a plane entry

template <typename T>
struct LT;
// Warp-specialised with register reallocation (setmaxnreg, per warpgroup):
// warpgroup 0 is the producer group (warp 0 produces, warps 1-3 retire) and
// shrinks to PREG registers; the CONS = 4 x (WGS - 1) consumer warps grow to
// CREG.  Consumer warp w evaluates positions q = w (mod CONS) of every run
// over the whole unit (one 16-byte lane vector per thread: 4 fp32 / 2 fp64
// orbitals).  Budget: 128 x PREG + CONS x 32 x CREG <= the CTA's launch
// allocation (regs_fit below).
template <>
struct LT<float> {
    static constexpr int RECB = 36 * 4 + 16;
    static constexpr int WGS = 4;     // 12 consumer warps, 3 per SMSP
    static constexpr int PREG = 32, CREG = 160;
    static constexpr int R = SPO_LINE_R32;  // plane slots
};
template <>
struct LT<double> {
    static constexpr int RECB = 36 * 8 + 16;
    // 12 consumer warps at 160 registers, as fp32.  Round 1 ran fp64 on 8 at
    // 232 (its 36 weights are 72 registers); at two warps per SMSP the DFMA
    // chains were latency-bound (ncu: stall `wait` 3.1 per issue, FP64 pipe
    // 27% on config 5's V).  Measured with 12 (profiles/r02/f64v_split.md):
    // V -21% (with groups of 3), VGL -2..5%, VGH -1%, a few spilled bytes.
    static constexpr int WGS = 4;
    static constexpr int PREG = 32, CREG = 160;
    static constexpr int R = SPO_LINE_R64;  // plane slots (larger records)
};
// Warp split per table form.  The k-power form needs fewer registers (no z
// weights), but 16 consumer warps at 112 registers spill and ran 10% slower
// than 12 at 160 (31.8 vs 28.6 ms per 524,288-position launch), so both
// forms use LT's split.
template <typename T, bool KP>
struct LW {
    static constexpr int WGS = LT<T>::WGS, PREG = LT<T>::PREG, CREG = LT<T>::CREG;
};
template <typename T, bool KP = false>
constexpr int cons_warps() {
    return 4 * (LW<T, KP>::WGS - 1);
}
template <typename T, bool KP = false>
constexpr int threads() {
    return 128 * LW<T, KP>::WGS;
}
// The pool setmaxnreg redistributes is the CTA's launch allocation: threads x
// the per-thread count __launch_bounds__ gives (64K / threads, rounded down to
// a multiple of 8).  Growing past it would make TRY_ALLOC spin forever.
template <typename T, bool KP = false>
constexpr bool regs_fit() {
    return 128 * LW<T, KP>::PREG + 32 * cons_warps<T, KP>() * LW<T, KP>::CREG <=
           threads<T, KP>() * (65536 / threads<T, KP>() / 8 * 8);
}
static_assert(regs_fit<float>(), "fp32 register split exceeds the launch allocation");
static_assert(regs_fit<double>(), "fp64 register split exceeds the launch allocation");
static_assert(regs_fit<float, true>(), "fp32 k-power register split exceeds the launch allocation");
static_assert(regs_fit<double, true>(), "fp64 k-power register split exceeds the launch allocation");

struct LArgs {
    const unsigned char *recs;  // [n_pos][RECB], sorted
    const int *plist;           // [runs][PL]: plane count, then i | j << 10 | k << 20 per plane
    unsigned *ticket;
    long long n_pos;
    long long nbatch;           // ceil(n_pos / BPL)
    long long n_items;          // units * nbatch
    int nb;                     // table row length (lanes) per tile
    void *out;
    long long out_pos_stride, out_stream_stride;
    const long long *out_index;
    long long lane_limit;
    int evict_last;
    // fused ratio epilogue (RATIO kernels, spo_eval_ratios): per (unit,
    // position) partial dot products of every stream with the coefficient row
    const void *coef;           // [n_pos][coef_stride] in output-lane layout
    long long coef_stride;
    double *partials;           // [units][n_pos][S]
    // k-power tables (KP kernels): TMA row coordinate = kmul * k0 (4: four
    // power-basis rows per cell), z-derivative factors 1/dz and 2/dz^2
    int kmul;
    double dz, dz2;
    int rotate;                 // rotate the run's positions over the consumer warps
    int dynamic;                // consumers take positions from a shared per-run counter
    int vuni;                   // V groups: the unrolled same-cell path (SPO_VUNI=0 disables, for A/B)
    int pspin;                  // producer mbarrier waits: 1 = tight try_wait spin, 0 = test + nanosleep back-off
    int vgroup;                 // V positions per consumer warp (the group kernels' VGROUP)
    int cellgroups;             // V groups aligned to cells by line_runs_kernel (group starts in the records)
    int vdyn;                   // V groups taken from a shared per-run counter (SPO_VDYN=0: rotated static)
    long long cells;            // grid cells (positions per cell pick the V group size)
};

struct LItem {
    long long b0;
    int nb, u, valid, pad;
};

// ------------------------------------------------------------- prologue --
// Sort keys, dense: lines (win == 1) order by (spatial block, j0, k0, i0) with
// the cell coordinates taken relative to their block's first cell; windows
// (win > 1) by (j0 / win, k0 / win, i0).  Dense keys need few bits, so the
// radix sort runs over bits [0, key_bits) only (line_key_bits): 2-3 passes
// instead of 4.  A non-finite position gets the all-ones key, which sorts
// after every valid one (key_bits leaves it above the largest valid key).
// Window shapes: WIN = n is an n x n window of (j0, k0) cells (1: a line);
// WIN = 10 wj + wk (wj, wk < 10, two digits) is a wj x wk one, e.g. 21 = two
// lines along j with no halo sharing along k (planes of 5 j-rows x 4 k-rows).
__host__ __device__ constexpr int win_j(int w) { return w > 9 ? w / 10 : w; }
__host__ __device__ constexpr int win_k(int w) { return w > 9 ? w % 10 : w; }

struct KeyGeom {
    int3 nbk;   // spatial blocks per axis (lines)
    int3 ext;   // cells per block along i, j, k (lines: ceil(n / nbk)); windows: (nx, ceil(ny / wj), ceil(nz / wk))
    int win;    // window code (win_j / win_k)
};
__device__ __forceinline__ int block_start(int b, int n, int nbk) { return (b * n + nbk - 1) / nbk; }

__global__ void line_keys_kernel(GridArgs g, const double *__restrict__ pos, long long n, unsigned *__restrict__ keys,
                                 int *__restrict__ vals, int *__restrict__ status, KeyGeom kg) {
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n;
         p += (long long)gridDim.x * blockDim.x) {
        double t;
        const double x = pos[3 * p], y = pos[3 * p + 1], z = pos[3 * p + 2];
        const int i0 = map_axis(x, g.dinv[0], g.cnt[0], &t);
        const int j0 = map_axis(y, g.dinv[1], g.cnt[1], &t);
        const int k0 = map_axis(z, g.dinv[2], g.cnt[2], &t);
        unsigned key = 0xffffffffu;
        if (isfinite(x) && isfinite(y) && isfinite(z)) {
            if (kg.win > 1) {  // windows: all lines of a wj x wk window of (j0, k0) cells, in i0 order
                key = ((unsigned)(j0 / win_j(kg.win)) * kg.ext.z + (unsigned)(k0 / win_k(kg.win))) * kg.ext.x +
                      (unsigned)i0;
            } else {
                const int bi = i0 * kg.nbk.x / g.n[0], bj = j0 * kg.nbk.y / g.n[1], bk = k0 * kg.nbk.z / g.n[2];
                const unsigned b = (bi * kg.nbk.y + bj) * kg.nbk.z + bk;
                const unsigned il = i0 - block_start(bi, g.n[0], kg.nbk.x);
                const unsigned jl = j0 - block_start(bj, g.n[1], kg.nbk.y);
                const unsigned kl = k0 - block_start(bk, g.n[2], kg.nbk.z);
                key = ((b * kg.ext.y + jl) * kg.ext.z + kl) * kg.ext.x + il;
            }
        } else if (status) {
            atomicOr(status, 1);
        }
        keys[p] = key;
        vals[p] = (int)p;
    }
}

template <typename T>
__global__ void line_records_kernel(GridArgs g, const double *__restrict__ pos, const int *__restrict__ order,
                                    long long n, unsigned char *__restrict__ recs, int kpower) {
    constexpr int RECB = LT<T>::RECB;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n;
         q += (long long)gridDim.x * blockDim.x) {
        const long long p = order[q];
        const double x = pos[3 * p], y = pos[3 * p + 1], z = pos[3 * p + 2];
        double tx, ty, tz;
        int i0 = map_axis(x, g.dinv[0], g.cnt[0], &tx);
        const int j0 = map_axis(y, g.dinv[1], g.cnt[1], &ty);
        const int k0 = map_axis(z, g.dinv[2], g.cnt[2], &tz);
        T w[36];
        axis_weights<T>(tx, g.dinv[0], g.delta[0], w);
        axis_weights<T>(ty, g.dinv[1], g.delta[1], w + 12);
        axis_weights<T>(tz, g.dinv[2], g.delta[2], w + 24);
        if (kpower) w[24] = (T)tz;  // k-power tables: the z weight is t itself
        if (!(isfinite(x) && isfinite(y) && isfinite(z))) i0 = -1;
        unsigned char *dst = recs + q * RECB;
#pragma unroll
        for (int e = 0; e < 36 * (int)sizeof(T) / 16; ++e) {
            float4 v;
            memcpy(&v, reinterpret_cast<const unsigned char *>(w) + 16 * e, 16);
            reinterpret_cast<float4 *>(dst)[e] = v;
        }
        *reinterpret_cast<int4 *>(dst + 36 * sizeof(T)) = make_int4(i0, j0 | (k0 << 16), 0, (int)p);
    }
}

// ------------------------------------------------------- plane sequence --
// The planes a run (BPL consecutive sorted positions) needs, numbered in load
// order.  A position on the current line whose i0 lies inside the loaded
// range reuses planes i0..last; new planes (max(last+1, i0) .. i0+3) get the
// next numbers.  line_runs_kernel stores in every record the run-relative
// number of its plane i0 (its planes are that number + 0..3) and in the
// run's first record the run's plane count; the producer loads planes in
// that order and the consumers find their planes by number: plane number s
// lives in ring slot s % R, phase s / R.
// Windows (win > 1): a plane is the (win+3) x (win+3) rows at one i shared by
// every position of a win x win window of (j0, k0) cells, anchored at the
// window's first cell (plane entry: i | J << 10 | K << 20, J = win * (j0 / win));
// positions of one window follow each other in i0 order like a line's.
// One warp per run, two positions per lane.  With the run sorted, a
// position's stencil shares planes only with the position before it, and only
// on the same line / window (`same`); the loaded range of the current line is
// a running maximum of i0 + 3 restarted at every new line (a segmented max
// scan), a position appends max(0, i0 + 3 - last) planes (4 on a new line),
// and the plane numbers are the prefix sums of those counts.  That is the
// sequential rule above, restated as two warp scans.  Non-finite positions
// (i0 < 0, sorted last) append nothing; a run in which one precedes a finite
// position (not produced by the sort) takes the sequential walk in lane 0.
constexpr int RUNS_PER_BLOCK = 4;
template <typename T>
__global__ void __launch_bounds__(32 * RUNS_PER_BLOCK)
    line_runs_kernel(long long n, unsigned char *__restrict__ recs, int *__restrict__ plist, int win, int vgroup) {
    static_assert(BPL == 64, "two positions per lane");
    __shared__ unsigned char gs_all[RUNS_PER_BLOCK][BPL];  // vgroup > 0: start position of the run's group k
    constexpr int RECB = LT<T>::RECB;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long b = blockIdx.x * (long long)RUNS_PER_BLOCK + w;
    if (b * BPL >= n) return;
    const int nb = (int)min((long long)BPL, n - b * BPL);
    unsigned char *rc = recs + b * BPL * RECB + 36 * sizeof(T);
    int *pl = plist + b * PL;
    unsigned char *gs = gs_all[w];
    int i0[2], wj[2], wk[2], cy[2];
    bool ok[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const int q = 2 * lane + e;
        int4 c = make_int4(-1, 0, 0, 0);
        if (q < nb) c = *reinterpret_cast<const int4 *>(rc + q * RECB);
        ok[e] = c.x >= 0;
        i0[e] = c.x;
        cy[e] = c.y;
        gs[q] = 0xff;
        const int j0 = c.y & 0xffff, k0 = c.y >> 16;
        wj[e] = win_j(win) * (j0 / win_j(win));
        wk[e] = win_k(win) * (k0 / win_k(win));
    }
    const unsigned m0 = __ballot_sync(0xffffffffu, ok[0]), m1 = __ballot_sync(0xffffffffu, ok[1]);
    unsigned long long valid = 0;  // bit q: position q is finite
    for (int l = 0; l < 32; ++l)
        valid |= (unsigned long long)((m0 >> l) & 1) << (2 * l) | (unsigned long long)((m1 >> l) & 1) << (2 * l + 1);
    if ((valid & (valid + 1)) != 0) {  // not a prefix: the sequential walk
        if (lane == 0) {
            int cj = -1, ck = -1, last = -1, next = 0;
            for (int q = 0; q < nb; ++q) {
                int4 *c = reinterpret_cast<int4 *>(rc + q * RECB);
                const int4 cell = *c;
                int s = 0;
                if (cell.x >= 0) {
                    const int j0 = cell.y & 0xffff, k0 = cell.y >> 16, x0 = cell.x;
                    const int aj = win_j(win) * (j0 / win_j(win)), ak = win_k(win) * (k0 / win_k(win));
                    const bool same = aj == cj && ak == ck;
                    int lo;
                    if (same && x0 <= last) {
                        s = next - 1 - (last - x0);
                        lo = last + 1;
                    } else {
                        s = next;
                        lo = x0;
                    }
                    for (int t = lo; t <= x0 + 3; ++t) pl[1 + next++] = t | (aj << 10) | (ak << 20);
                    if (!same || x0 + 3 > last) last = x0 + 3;
                    cj = aj;
                    ck = ak;
                }
                c->z = s | (vgroup > 0 && q > 0 ? q << 16 : 0);  // cell groups: every position its own group
            }
            reinterpret_cast<int4 *>(rc)->z |= next << 16;
            pl[0] = next;
        }
        return;
    }
    // the previous position's anchor: element 0 from the lane before
    const int pj = __shfl_up_sync(0xffffffffu, wj[1], 1), pk = __shfl_up_sync(0xffffffffu, wk[1], 1);
    bool same[2];
    same[0] = lane > 0 && ok[0] && wj[0] == pj && wk[0] == pk;
    same[1] = ok[1] && wj[1] == wj[0] && wk[1] == wk[0];
    // segmented inclusive max of i0 + 3 (a new line starts a segment)
    const int v0 = i0[0] + 3, v1 = i0[1] + 3;
    const bool head0 = !same[0], head1 = !same[1];
    bool hf = head0 || head1;
    int hv = head1 ? v1 : max(v0, v1);
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int ov = __shfl_up_sync(0xffffffffu, hv, d);
        const bool of = __shfl_up_sync(0xffffffffu, hf, d);
        if (lane >= d) {
            if (!hf) hv = max(hv, ov);
            hf = hf || of;
        }
    }
    const int before = __shfl_up_sync(0xffffffffu, hv, 1);  // max over the lane's predecessors' segment
    const int run0 = head0 ? v0 : max(before, v0);
    const int lastp[2] = {before, run0};  // `last` before each element (used only when same)
    int cnt[2], lo[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        if (!ok[e]) {
            cnt[e] = 0;
            lo[e] = 0;
        } else if (same[e] && i0[e] <= lastp[e]) {
            lo[e] = lastp[e] + 1;
            cnt[e] = max(0, i0[e] + 3 - lastp[e]);
        } else {
            lo[e] = i0[e];
            cnt[e] = 4;
        }
    }
    // exclusive prefix sum of the counts
    int incl = cnt[0] + cnt[1];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int o = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += o;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    if (vgroup > 0) {
        // Cell-aligned V groups: a group starts at every new cell (a non-finite
        // position is a cell of its own) and after every vgroup positions of a
        // cell.  Position-in-cell = q - (start of q's cell), the start by a max
        // scan over the new-cell positions; the group number is the prefix sum
        // of the group-start flags; gs[k] = first position of group k.
        const int pi = __shfl_up_sync(0xffffffffu, i0[1], 1), py = __shfl_up_sync(0xffffffffu, cy[1], 1);
        bool nc[2];
        nc[0] = lane == 0 || !ok[0] || i0[0] != pi || cy[0] != py;
        nc[1] = !ok[1] || i0[1] != i0[0] || cy[1] != cy[0];
        int cs = nc[1] ? 2 * lane + 1 : (nc[0] ? 2 * lane : -1);  // last cell start in this lane
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int o = __shfl_up_sync(0xffffffffu, cs, d);
            if (lane >= d) cs = max(cs, o);
        }
        const int csb = __shfl_up_sync(0xffffffffu, cs, 1);  // last cell start before this lane
        const int st0 = nc[0] ? 2 * lane : csb;
        const int st1 = nc[1] ? 2 * lane + 1 : st0;
        bool gf[2];
        gf[0] = 2 * lane < nb && (2 * lane - st0) % vgroup == 0;
        gf[1] = 2 * lane + 1 < nb && (2 * lane + 1 - st1) % vgroup == 0;
        int gi = (int)gf[0] + (int)gf[1];
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int o = __shfl_up_sync(0xffffffffu, gi, d);
            if (lane >= d) gi += o;
        }
        const int g1 = gi - 1, g0 = g1 - (int)gf[1];  // group numbers of the lane's two positions
        __syncwarp();
        if (gf[0]) gs[g0] = (unsigned char)(2 * lane);
        if (gf[1]) gs[g1] = (unsigned char)(2 * lane + 1);
        __syncwarp();
    }
    int next = incl - cnt[0] - cnt[1];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const int q = 2 * lane + e;
        int s = 0;
        if (ok[e]) {
            s = (same[e] && i0[e] <= lastp[e]) ? next - 1 - (lastp[e] - i0[e]) : next;
            for (int t = 0; t < cnt[e]; ++t) pl[1 + next + t] = (lo[e] + t) | (wj[e] << 10) | (wk[e] << 20);
        }
        if (q < nb)
            reinterpret_cast<int4 *>(rc + q * RECB)->z =
                s | (q == 0 ? total << 16 : (vgroup > 0 ? (int)gs[q] << 16 : 0));
        next += cnt[e];
    }
    if (lane == 0) pl[0] = total;
}

// Plane slots: WIN = 1 (lines) R = LT<T>::R slots of 16 rows; windows of
// WIN x WIN cells: as many (WIN+3)^2-row slots as the budget holds.
constexpr size_t SMEM_BUDGET = 232448;
template <int WIN>
constexpr int plane_bytes() {
    return (win_j(WIN) + 3) * (win_k(WIN) + 3) * ROWB;
}
// Run slots (NRS): how many runs' records + plane lists a CTA holds.  Two let
// the producer fetch run r+1 while the consumers evaluate run r.  The V group
// kernels on lines take three (SPO_LINE_NRS_V; a V run is short, ~1.8 groups
// per warp, and with the groups handed out dynamically a third slot is worth
// 2.5% on config 5's V; four measured the same as three; the window rings
// have no room: scripts/micro/vdyn_ab.sh, profiles/r02/v_dynamic.md).
#ifndef SPO_LINE_NRS_V
#define SPO_LINE_NRS_V 3
#endif
template <typename T, int NRS = 2>
constexpr size_t smem_fixed() {
    return NRS * ((size_t)BPL * LT<T>::RECB + (size_t)PLB + sizeof(LItem) + 2 * 8);
}
template <typename T, int WIN, int NRS = 2>
constexpr int ring() {
    constexpr int fit = (int)((SMEM_BUDGET - smem_fixed<T, NRS>()) / (plane_bytes<WIN>() + 16));
    return WIN == 1 ? (LT<T>::R < fit ? LT<T>::R : fit) : fit;
}
// as many run slots (<= SPO_LINE_NRS_V) as leave the V group its ring: the 4 x
// VGROUP planes a group may span, the rest of the producer's last batch
// (ring_min below) and a few to load ahead
template <int KIND, typename T, int VGROUP, int WIN>
constexpr int rec_slots() {
    if (!(KIND == SPO_KIND_V && VGROUP > 1)) return 2;
    if (SPO_LINE_NRS_V >= 4 && ring<T, WIN, 4>() >= 4 * VGROUP + PBATCH + 3) return 4;
    if (SPO_LINE_NRS_V >= 3 && ring<T, WIN, 3>() >= 4 * VGROUP + PBATCH + 3) return 3;
    return 2;
}
// The smallest deadlock-free ring: the warp furthest behind holds planes from
// lo on and may wait for plane lo + 4 VGROUP - 1; the producer arms planes in
// batches of PBATCH and waits for ring space for a whole batch, so the batch
// that holds that plane can reach PBATCH - 1 planes past it.
constexpr int ring_min(int vgroup) { return 4 * vgroup + PBATCH - 1; }
template <typename T, int WIN = 1, int NRS = 2>
constexpr size_t smem_planes() {
    return (size_t)ring<T, WIN, NRS>() * plane_bytes<WIN>();
}
template <typename T, int WIN = 1, int NRS = 2>
constexpr size_t smem_bytes() {
    return smem_planes<T, WIN, NRS>() + smem_fixed<T, NRS>() + 2 * (size_t)ring<T, WIN, NRS>() * 8;
}
#ifndef SPO_WIN_CELLS
#define SPO_WIN_CELLS 2  // 2 and 3 within ~1-4% of each other, 2 ahead on most configs; 4 slower
#endif
constexpr int WIN_CELLS = SPO_WIN_CELLS;  // window side (cells) of the window variant
// V on windows: two lines along j (planes of 5 j-rows x 4 k-rows), where V
// position groups read a plane once for several positions with no k offset
// to select (win_k = 1)
constexpr int VWIN = 21;
// V groups aligned to cells from this many positions per cell (below, most
// same-cell runs are shorter than a group and the general path's plane sharing
// between neighbouring cells is worth more).  Measured with groups of 3
// (profiles/r02/v_cell_groups.md): fp64 -3.4% at 4.7 per cell, -4% at 7.1, -5% at
// 16.3 (config 5's V); fp32 +1% at 4, 0 at 6, -3% at 8 per cell.
#ifndef SPO_CELL_GROUPS_MIN32
#define SPO_CELL_GROUPS_MIN32 7.0
#endif
#ifndef SPO_CELL_GROUPS_MIN64
#define SPO_CELL_GROUPS_MIN64 4.5
#endif
static_assert(smem_bytes<float>() <= SMEM_BUDGET, "shared memory budget");
static_assert(smem_bytes<double>() <= SMEM_BUDGET, "shared memory budget");
static_assert(smem_bytes<float, WIN_CELLS>() <= SMEM_BUDGET, "shared memory budget");
static_assert(smem_bytes<double, WIN_CELLS>() <= SMEM_BUDGET, "shared memory budget");
static_assert(ring<double, WIN_CELLS>() >= 6, "a window ring must hold more than one position's planes");
static_assert(smem_bytes<float, VWIN>() <= SMEM_BUDGET && smem_bytes<double, VWIN>() <= SMEM_BUDGET, "budget");

// ---------------------------------------------------------------- kernel --
template <int KIND, typename T, bool RATIO, bool KP, int VGROUP = 1, int WIN = 1>
__global__ void __launch_bounds__(threads<T, KP>(), 1) line_kernel(const __grid_constant__ CUtensorMap tmap, const LArgs a) {
    constexpr int S = NS<KIND>::S;
    constexpr int CONSUMERS = cons_warps<T, KP>();
    constexpr int NRS = rec_slots<KIND, T, VGROUP, WIN>();  // run slots (records + plane list)
    constexpr int R = ring<T, WIN, NRS>();
    constexpr int PB = plane_bytes<WIN>();         // bytes per plane slot
    constexpr int RJ = win_k(WIN) + 3;             // k-rows per j-row of a slot
    static_assert(WIN == 1 || (!KP && (VGROUP == 1 || (KIND == SPO_KIND_V && win_k(WIN) == 1))),
                  "windows: B-spline form; V groups only on windows without k sharing");
    constexpr int W = 16 / (int)sizeof(T);         // lanes per thread (16-byte vector)
    constexpr int RECB = LT<T>::RECB;
    constexpr int ULANES = ROWB / (int)sizeof(T);  // lanes per unit
    constexpr int BOXL = BOXB / (int)sizeof(T);    // lanes per box = per consumer warp
    static_assert(32 * W == BOXL, "a consumer warp covers one box");
    using AV = typename Acc<T>::V;
    constexpr int AN = Acc<T>::N;

    extern __shared__ __align__(1024) unsigned char smem[];
    unsigned char *planes = smem;
    unsigned char *recs = smem + smem_planes<T, WIN, NRS>();
    int *plists = reinterpret_cast<int *>(recs + NRS * BPL * RECB);
    LItem *info = reinterpret_cast<LItem *>(plists + NRS * PL);
    unsigned long long *full = reinterpret_cast<unsigned long long *>(info + NRS);
    unsigned *relw = reinterpret_cast<unsigned *>(full + R);  // [CONSUMERS]: first plane each warp still needs
    unsigned *issued = relw + CONSUMERS;                      // planes armed so far
    unsigned long long *rfull = full + 2 * R;
    unsigned long long *rempty = rfull + NRS;
    unsigned *qnext = issued + 1;                             // [NRS]: next position of each run slot's run
    static_assert((CONSUMERS + 1 + NRS) * 4 <= R * 8, "release words fit");
    static_assert(ring_min(1) <= R, "a position's planes and the producer's batch must fit the ring");

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x < CONSUMERS + 1 + NRS) relw[threadIdx.x] = 0;  // and issued, qnext
    if (threadIdx.x == 0) {
        for (int s = 0; s < R; ++s) mbar_init(&full[s], 1);
        for (int s = 0; s < NRS; ++s) {
            mbar_init(&rfull[s], 1);
            mbar_init(&rempty[s], CONSUMERS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp < 4) {
        // ------------------------------------------------------ producer --
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(LW<T, KP>::PREG));
        if (warp != 0) return;
        // lane 0 takes tickets and loads run records + plane lists; lanes
        // 0..PBATCH-1 issue the run's planes PBATCH at a time (one slot each)
        const unsigned long long policy = l2_policy(a.evict_last);
        // The producer's mbarrier waits: a try_wait spin (default).  It takes
        // issue slots from the three consumer warps on its scheduler (ncu on
        // config 5's V: 2.7e8 spin iterations per launch, 14% of all
        // instructions executed), but a nanosleep back-off (SPO_PSPIN=0)
        // reacts later and measured slower; the consumers' dynamic position /
        // group counters absorb the imbalance instead.
        auto pwait = [&](unsigned long long *bar, unsigned par) {
            if (a.pspin) {
                mbar_wait(bar, par);
                return;
            }
            while (!mbar_test(bar, par)) __nanosleep(SPIN_NS);
        };
        auto fill = [&](int slot) {  // lane 0
            const unsigned long long k = atomicAdd(a.ticket, 1u);
            LItem it;
            it.valid = k < (unsigned long long)a.n_items;
            it.pad = 0;
            if (it.valid) {
                const long long u = (long long)k / a.nbatch;
                const long long b = (long long)k - u * a.nbatch;
                it.u = (int)u;
                it.b0 = b * BPL;
                it.nb = (int)min((long long)BPL, a.n_pos - it.b0);
                info[slot] = it;
                qnext[slot] = 0;  // published to the consumers by the arrive (release)
                mbar_arrive_expect_tx(&rfull[slot], (unsigned)(it.nb * RECB + PLB));
                bulk_load(recs + slot * BPL * RECB, a.recs + it.b0 * RECB, (unsigned)(it.nb * RECB), &rfull[slot]);
                bulk_load(plists + slot * PL, a.plist + b * PL, (unsigned)PLB, &rfull[slot]);
            } else {
                it.u = it.nb = 0;
                it.b0 = 0;
                info[slot] = it;
                mbar_arrive(&rfull[slot]);
            }
        };
        // the records slot of item r-1 is refilled (item r+1) once the
        // consumers release it: polled between plane batches
        int pend = -1;
        unsigned pend_par = 0;
        auto poll = [&](bool block) {  // lane 0
            if (pend < 0) return;
            if (block)
                pwait(&rempty[pend], pend_par);
            else if (!mbar_test(&rempty[pend], pend_par))
                return;
            fill(pend);
            pend = -1;
        };
        if (lane == 0) {
            for (int s = 0; s < NRS; ++s) fill(s);
        }
        __syncwarp();
        unsigned base = 0;  // plane number of the current run's first plane
        for (int r = 0;; ++r) {
            const int slot = r % NRS;
            pwait(&rfull[slot], (r / NRS) & 1);
            const LItem it = info[slot];
            if (!it.valid) break;
            if (r >= 1) {
                pend = (r - 1) % NRS;  // item r-1's slot, for item r-1+NRS
                pend_par = ((r - 1) / NRS) & 1;
            }
            const int *pl = plists + slot * PL;
            const int count = pl[0];
            const long long L = (long long)it.u * ULANES;  // the unit's first lane
            const int tile = (int)(L / a.nb), lt = (int)(L - (long long)tile * a.nb);
            for (int t0 = 0; t0 < count; t0 += PBATCH) {
                const int nbt = min(PBATCH, count - t0);
                const unsigned xlast = base + (unsigned)(t0 + nbt - 1);
                if (xlast >= (unsigned)R) {
                    // ring space: every consumer is done with the planes these slots held
                    const unsigned need = xlast - R + 1;
                    while (true) {
                        unsigned v = lane < CONSUMERS ? ld_acquire_shared(&relw[lane]) : 0xffffffffu;
                        v = __reduce_min_sync(0xffffffffu, v);
                        if (v >= need) break;
                        __nanosleep(SPIN_NS);
                    }
                }
                const int t = t0 + lane;
                if (lane < nbt) {
                    const unsigned s = base + (unsigned)t;
                    const int sl = (int)(s % R);
                    const unsigned n = s / R;
                    // the slot's previous plane has landed (the producer observes
                    // every plane in order, so the parity cannot alias)
                    if (n > 0) pwait(&full[sl], (n - 1) & 1);
                    const int c = pl[1 + t];
                    mbar_arrive_expect_tx(&full[sl], PB);
                    tma_load_5d(planes + (size_t)sl * PB, &tmap, &full[sl], lt, a.kmul * ((c >> 20) & 0x3ff),
                                (c >> 10) & 0x3ff, c & 0x3ff, tile, policy);
                }
                __syncwarp();
                if (lane == 0) {
                    st_release_shared(issued, base + (unsigned)(t0 + nbt));
                    poll(false);
                }
                __syncwarp();
            }
            base += (unsigned)count;
            if (r >= 1 && lane == 0) poll(true);
            __syncwarp();
        }
        return;
    }

    // -------------------------------------------------------- consumers --
    // warp g evaluates positions q = g (mod CONSUMERS) of every run (the TMA
    // kernel's contraction, one 16-byte lane vector per thread).  It waits
    // only on its own planes: `issued` says a plane's slot is armed (so the
    // parity wait is on the right phase), and relw[g] publishes the first
    // plane it will need next (all below are free for the producer).
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(LW<T, KP>::CREG));
    const int g = warp - 4;
    unsigned base = 0;
    // (Skipping this acquire poll for planes below an `issued` value already
    // observed is correct but measured 0.6-1.1% slower: scripts/micro/z2_ab.sh
    // run as an A/B, profiles/r02/README.md.)
    auto await_issued = [&](unsigned x) {
        while (ld_acquire_shared(issued) <= x) __nanosleep(SPIN_NS);
    };
    auto publish = [&](unsigned v) {
        __syncwarp();
        if (lane == 0) st_release_shared(&relw[g], v);
    };
    if constexpr (KIND == SPO_KIND_V && VGROUP > 1) {
        // V: groups of VGROUP consecutive sorted positions, group k of a run
        // to warp k mod CONSUMERS.  V has little math per plane, so a plane's
        // shared-memory read is most of its cost: the group reads each plane
        // of [lo, hi] (the union of its positions' planes, contiguous in load
        // order) once, and every position covering it consumes the registers
        // (v_rowgroup, bitwise the one-position sequence).  Ring safety as
        // below: the warp publishes lo, and hi <= lo + 4 VGROUP - 1 < lo + R.
        constexpr int VM = VGROUP;
        static_assert(ring_min(VM) <= R, "a group's planes and the producer's batch must fit the ring");
        using RV = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
        using TV = typename std::conditional<sizeof(T) == 4, float2, double>::type;
        for (int r = 0;; ++r) {
            const int slot = r % NRS;
            mbar_wait(&rfull[slot], (r / NRS) & 1);
            const LItem it = info[slot];
            if (!it.valid) break;
            const unsigned char *rc = recs + slot * BPL * RECB;
            const unsigned count = (unsigned)reinterpret_cast<const int4 *>(rc + 36 * sizeof(T))->z >> 16;
            auto first_plane = [&](int q) -> unsigned {  // base + count once q is past the run
                if (q >= it.nb) return base + count;
                const int4 c = *reinterpret_cast<const int4 *>(rc + q * RECB + 36 * sizeof(T));
                return c.x < 0 ? base + count : base + (unsigned)(c.z & 0xffff);
            };
            // group k of the run goes to warp (k + rotation) mod CONSUMERS; the
            // rotation advances by the run's group count so that every warp gets
            // the same share of groups over consecutive runs (64 / VM groups do
            // not divide evenly among the warps)
            const int rot = a.rotate ? (int)((long long)r * (BPL / VM) % CONSUMERS) : 0;
            // dynamic (SPO_VDYN, default): every warp takes the run's next group
            // from the run slot's counter, so a warp delayed on its SMSP (the
            // producer warp shares SMSP 0's issue slots) takes fewer groups
            // instead of holding the run back
            auto take = [&]() -> int {
                int v = 0;
                if (lane == 0) v = (int)atomicAdd(&qnext[slot], 1u);
                return __shfl_sync(0xffffffffu, v, 0);
            };
            // Groups: fixed (group k = positions k VM .. k VM + VM - 1 of the run),
            // or, on dense batches, aligned to cells by line_runs_kernel
            // (a.cellgroups): group k starts at the position stored in record k
            // (bits 16..23 of cell.z; 0xff: no such group) and holds up to VM
            // positions of ONE cell, so every group takes the unrolled same-cell
            // path below.
            auto gstart = [&](int k) -> int {
                if (k >= it.nb) return it.nb;
                if (k == 0) return 0;
                const int v = (reinterpret_cast<const int4 *>(rc + k * RECB + 36 * sizeof(T))->z >> 16) & 0xff;
                return v == 0xff ? it.nb : v;
            };
            auto qof = [&](int k) -> int { return a.cellgroups ? gstart(k) : k * VM; };
            int kcur = a.vdyn ? take() : (g + CONSUMERS - rot) % CONSUMERS;
            int q0 = qof(kcur);
            publish(first_plane(q0));
            const long long L0 = (long long)it.u * ULANES + lane * W;
            const int nv = (int)max(0LL, min((long long)W, a.lane_limit - L0));
            while (q0 < it.nb) {
                const int ng = a.cellgroups ? gstart(kcur + 1) - q0 : VM;  // positions of this group
                // The x weights are used once per plane: read from the record in
                // shared memory at that point (a broadcast load) instead of held
                // in 4 (fp64: 8) registers per position: fp32 V -10..12% at 2-4 per
                // cell, config 5's fp64 V -1..6%.  fp64 reads the y weights the
                // same way (once per row group; -1..2%; fp32 measured 4-7% slower
                // with it).  scripts/micro/wx_ab.sh, profiles/r02/v_dynamic.md.
                constexpr bool WY_SMEM = sizeof(T) == 8;
                T wy[WY_SMEM ? 1 : VM][4], wz[VM][4];
                const T *wxp[VM];
                auto wyj = [&](int m, int j) -> T {  // selects: j is a run-time value on windows
                    if constexpr (WY_SMEM) return wxp[m][12 + j];
                    const auto &w = wy[WY_SMEM ? 0 : m];
                    return j == 0 ? w[0] : (j == 1 ? w[1] : (j == 2 ? w[2] : w[3]));
                };
                unsigned s0[VM];
                int jj[VM];  // windows along j: the position's j-row offset in the plane
                bool live[VM];
                long long op[VM];
                AV acc[VM][1][AN];
                TV t00[VM][2];
                unsigned lo = 0xffffffffu, hi = 0;
#pragma unroll
                for (int m = 0; m < VM; ++m) {
                    const bool in = m < ng && q0 + m < it.nb;
                    const unsigned char *rec = rc + min(q0 + m, it.nb - 1) * RECB;
                    const int4 cell = *reinterpret_cast<const int4 *>(rec + 36 * sizeof(T));
                    live[m] = in && cell.x >= 0;
                    op[m] = !in ? -1 : (!RATIO && a.out_index ? a.out_index[cell.w] : cell.w);
                    // the a-rows of x, y, z: weights 0..3, 12..15, 24..27 (k-power: wz[0] = t_z)
                    wxp[m] = reinterpret_cast<const T *>(rec);
                    if constexpr (!WY_SMEM) load4(rec + 12 * sizeof(T), wy[m]);
                    load4(rec + 24 * sizeof(T), wz[m]);
                    s0[m] = base + (unsigned)(cell.z & 0xffff);
                    jj[m] = (cell.y & 0xffff) % win_j(WIN);
                    if (live[m]) {
                        lo = min(lo, s0[m]);
                        hi = max(hi, s0[m] + 3u);
                    }
#pragma unroll
                    for (int h = 0; h < AN; ++h) zero(acc[m][0][h]);
                    t00[m][0] = t00[m][1] = TV{};
                }
                // Dense batches: the group's positions mostly sit in one cell (same
                // first plane, same row offset), so all of them take the same four
                // planes row group by row group -- unrolled with no per-position
                // tests (the general loop below spends ~60% of its instructions on
                // them: ncu on config 5's V, profiles/r02/f64v_uniform.md).  Each
                // position sees exactly the general loop's sequence (bitwise).
                // the first NN positions of the group on the same four planes
                auto same_cell = [&](auto nn) {
                    constexpr int NN = decltype(nn)::value;
                    await_issued(hi);  // planes are armed in order: lo .. hi are all issued
                    const int roff = WIN == 1 ? 0 : jj[0] * 4 * BOXL;
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const unsigned x = lo + (unsigned)i;
                        const int sl = (int)(x % R);
                        mbar_wait(&full[sl], (x / R) & 1);
                        const T *p = reinterpret_cast<const T *>(planes + (size_t)sl * PB) + roff + lane * W;
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            RV c[4];
#pragma unroll
                            for (int k = 0; k < 4; ++k) c[k] = *reinterpret_cast<const RV *>(p + (j * 4 + k) * BOXL);
#pragma unroll
                            for (int m = 0; m < NN; ++m) v_rowgroup<KP>(c, wz[m], wyj(m, j), t00[m]);
                        }
#pragma unroll
                        for (int m = 0; m < NN; ++m) v_plane_done(wxp[m][i], t00[m], acc[m]);
                    }
                };
                if (a.cellgroups) {
                    // 1 .. VM positions of one cell (a non-finite position is a group of its own)
                    if (live[0]) {
                        if (ng >= VM) same_cell(std::integral_constant<int, VM>{});
                        else if (ng == 1) same_cell(std::integral_constant<int, 1>{});
                        else if (ng == 2) same_cell(std::integral_constant<int, (VM > 2 ? 2 : 1)>{});
                        else if (ng == 3) same_cell(std::integral_constant<int, (VM > 3 ? 3 : 1)>{});
                        else same_cell(std::integral_constant<int, (VM > 4 ? 4 : 1)>{});
                    }
                    lo = 0xffffffffu;  // done: skip the general loop
                } else {
                    bool uni = a.vuni && live[0];
#pragma unroll
                    for (int m = 1; m < VM; ++m)
                        uni = uni && live[m] && s0[m] == s0[0] && (WIN == 1 || jj[m] == jj[0]);
                    if (uni) {
                        same_cell(std::integral_constant<int, VM>{});
                        lo = 0xffffffffu;  // done: skip the general loop
                    }
                }
                for (unsigned x = lo; lo != 0xffffffffu && x <= hi; ++x) {
                    await_issued(x);
                    const int sl = (int)(x % R);
                    mbar_wait(&full[sl], (x / R) & 1);
                    const T *p = reinterpret_cast<const T *>(planes + (size_t)sl * PB) + lane * W;
                    // j-row by j-row (a line: its 4; a wj x 1 window: wj + 3, each
                    // position taking its row group j = r - jj, in increasing j
                    // as its own slab_contract would; no k offsets to select)
#pragma unroll
                    for (int r = 0; r < win_j(WIN) + 3; ++r) {
                        RV c[4];
#pragma unroll
                        for (int k = 0; k < 4; ++k) c[k] = *reinterpret_cast<const RV *>(p + (r * 4 + k) * BOXL);
#pragma unroll
                        for (int m = 0; m < VM; ++m) {
                            const int j = WIN == 1 ? r : r - jj[m];
                            if (!(live[m] && x - s0[m] < 4u) || j < 0 || j > 3) continue;
                            v_rowgroup<KP>(c, wz[m], wyj(m, j), t00[m]);
                        }
                    }
#pragma unroll
                    for (int m = 0; m < VM; ++m)
                        if (live[m] && x - s0[m] < 4u) {
                            const unsigned i = x - s0[m];
                            v_plane_done(wxp[m][i], t00[m], acc[m]);
                        }
                }
                kcur = a.vdyn ? take() : kcur + CONSUMERS;
                const int qn = qof(kcur);
                publish(first_plane(qn));  // this group's planes are read
#pragma unroll
                for (int m = 0; m < VM; ++m) {
                    if (op[m] < 0) continue;
                    if constexpr (RATIO) {
                        // the fused consumer: this unit's dot with the position's coefficient
                        // row (pad lanes hold 0), reduced over the warp, as the one-position path
                        double part[1] = {(double)NAN};
                        if (live[m]) {
                            const T *cf = reinterpret_cast<const T *>(a.coef) + op[m] * a.coef_stride + L0;
                            ratio_partials<1, 32>(acc[m], cf, true, part);
                        }
                        if (lane == 0) a.partials[(long long)it.u * a.n_pos + op[m]] = part[0];
                        continue;
                    }
                    T *o = reinterpret_cast<T *>(a.out) + op[m] * a.out_pos_stride + L0;
                    if (nv == W)
                        store_lane<1>(o, a.out_stream_stride, acc[m], live[m]);
                    else if (nv > 0)
                        store_lane_partial<1>(o, a.out_stream_stride, acc[m], live[m], nv);
                }
                q0 = qn;
            }
            base += count;
            __syncwarp();
            if (lane == 0) mbar_arrive(&rempty[slot]);
        }
        return;
    }
    for (int r = 0;; ++r) {
        const int slot = r % NRS;
        mbar_wait(&rfull[slot], (r / NRS) & 1);
        const LItem it = info[slot];
        if (!it.valid) break;
        const unsigned char *rc = recs + slot * BPL * RECB;
        const unsigned count = (unsigned)reinterpret_cast<const int4 *>(rc + 36 * sizeof(T))->z >> 16;
        auto first_plane = [&](int q) -> unsigned {
            if (q >= it.nb) return base + count;
            const int4 c = *reinterpret_cast<const int4 *>(rc + q * RECB + 36 * sizeof(T));
            return c.x < 0 ? base + count : base + (unsigned)(c.z & 0xffff);
        };
        // position q of the run goes to warp (q + rotation) mod CONSUMERS; the
        // rotation advances by BPL per run, so the warps take turns at the
        // BPL mod CONSUMERS extra positions (64 = 5 x 12 + 4: without it four
        // warps would always carry a sixth position and the rest would wait)
        const int rot = a.rotate ? (int)((long long)r * BPL % CONSUMERS) : 0;
        // dynamic: every warp takes the run's next position from a shared
        // counter, so the warps stay on neighbouring positions (one window of
        // planes) whatever their individual delays
        auto take = [&]() -> int {
            int v = 0;
            if (lane == 0) v = (int)atomicAdd(&qnext[slot], 1u);
            return __shfl_sync(0xffffffffu, v, 0);
        };
        const int q_first = a.dynamic ? take() : (g + CONSUMERS - rot) % CONSUMERS;
        publish(first_plane(q_first));
        const long long L0 = (long long)it.u * ULANES + lane * W;  // output lane
        const int nv = (int)max(0LL, min((long long)W, a.lane_limit - L0));
        for (int q = q_first, qn = 0; q < it.nb; q = qn) {
            const unsigned char *rec = rc + q * RECB;
            const int4 cell = *reinterpret_cast<const int4 *>(rec + 36 * sizeof(T));
            const long long op = a.out_index ? a.out_index[cell.w] : cell.w;
            T *o = reinterpret_cast<T *>(a.out) + op * a.out_pos_stride + L0;
            AV acc[S][AN], zs[4][AN];  // zs: fp32 z-second-derivative sums (slab_contract)
#pragma unroll
            for (int s = 0; s < S; ++s)
#pragma unroll
                for (int h = 0; h < AN; ++h) zero(acc[s][h]);
#pragma unroll
            for (int c = 0; c < 4; ++c)
#pragma unroll
                for (int h = 0; h < AN; ++h) zero(zs[c][h]);
            if (cell.x < 0) {
                qn = a.dynamic ? take() : q + CONSUMERS;
                publish(first_plane(qn));
                if constexpr (RATIO) {
                    if (lane == 0) {
                        double *dst = a.partials + ((long long)it.u * a.n_pos + cell.w) * S;
#pragma unroll
                        for (int s = 0; s < S; ++s) dst[s] = (double)NAN;
                    }
                } else if (nv == W) {
                    store_lane<S>(o, a.out_stream_stride, acc, false);
                } else if (nv > 0) {
                    store_lane_partial<S>(o, a.out_stream_stride, acc, false, nv);
                }
                continue;
            }
            const unsigned s0 = base + (unsigned)(cell.z & 0xffff);
            // the position's 4 x 4 rows inside its slot (windows: offset by its cell in the window)
            const int corner =
                WIN == 1 ? 0 : (((cell.y & 0xffff) % win_j(WIN)) * RJ + (cell.y >> 16) % win_k(WIN)) * BOXL;
            T wx[12], wy[12], wz[12];  // k-power tables: wz[0] = t_z, the rest unused
            load_weights(rec, wx, wy, wz);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const unsigned x = s0 + (unsigned)i;
                await_issued(x);
                const int sl = (int)(x % R);
                mbar_wait(&full[sl], (x / R) & 1);
                const T *p = reinterpret_cast<const T *>(planes + (size_t)sl * PB) + corner + lane * W;
                // fp64 VGH: the x weights of slab i from the record in shared memory
                // (three broadcast loads per slab) instead of 24 registers: -2.7%,
                // its spills gone.  fp32 (+0.8%) and fp64 VGL (+0.5%) keep them in
                // registers (scripts/micro/wxs_ab.sh; -DSPO_WX_SMEM=1 forces all).
                constexpr bool WXS = SPO_WX_SMEM || (sizeof(T) == 8 && KIND == SPO_KIND_VGH);
                const T *wr = reinterpret_cast<const T *>(rec);
                const T ax = WXS ? wr[i] : wx[i], dax = WXS ? wr[4 + i] : wx[4 + i],
                        d2ax = WXS ? wr[8 + i] : wx[8 + i];
                if constexpr (KP) {
                    const T dz = (T)a.dz, dz2 = (T)a.dz2;
                    slab_contract_kp<KIND, BOXL>(p, wy, wz[0], ax, dax, d2ax, mul_rn(ax, dz), mul_rn(dax, dz),
                                                 mul_rn(ax, dz2), acc);
                } else if constexpr (sizeof(T) == 4) {
                    slab_contract<KIND, BOXL, RJ>(p, wy, wz, ax, dax, d2ax, acc, zs);
                } else {
                    slab_contract<KIND, BOXL, RJ>(p, wy, wz, ax, dax, d2ax, acc);
                }
            }
            if constexpr (!KP && sizeof(T) == 4) finish_z2<KIND>(wz, zs, acc);
            // (Claiming the next position at the start of this one, to take the
            // counter / shuffle / record-lookup chain off the gap between two
            // positions, measured +0.3..1.4% slower for VGH and 5-35% slower for
            // V groups: scripts/micro/early_ab.sh, profiles/r02/v_dynamic.md.)
            qn = a.dynamic ? take() : q + CONSUMERS;
            publish(first_plane(qn));  // this position's planes are read
            if constexpr (RATIO) {
                // the warp's 32 lanes are this position's unit: dot with the
                // coefficient row, reduced over the warp (as spo_eval_tma.cu)
                const T *cf = reinterpret_cast<const T *>(a.coef) + (long long)cell.w * a.coef_stride + L0;
                double part[S];
                ratio_partials<S, 32>(acc, cf, true, part);
                if (lane == 0) {
                    double *dst = a.partials + ((long long)it.u * a.n_pos + cell.w) * S;
#pragma unroll
                    for (int s = 0; s < S; ++s) dst[s] = part[s];
                }
            } else if (nv == W) {
                store_lane<S>(o, a.out_stream_stride, acc, true);
            } else if (nv > 0) {
                store_lane_partial<S>(o, a.out_stream_stride, acc, true, nv);
            }
        }
        base += count;
        __syncwarp();
        if (lane == 0) mbar_arrive(&rempty[slot]);
    }
}

template <int KIND, typename T, bool RATIO, bool KP, int VGROUP = 1, int WIN = 1>
static int launch1(const CUtensorMap &map, const LArgs &a, int sms, cudaStream_t st) {
    constexpr size_t sm = smem_bytes<T, WIN, rec_slots<KIND, T, VGROUP, WIN>()>();
    static_assert(sm <= SMEM_BUDGET, "shared memory budget");
    int grid = (int)min((long long)sms, a.n_items);
    if (grid < 1) grid = 1;
    cudaFuncSetAttribute(line_kernel<KIND, T, RATIO, KP, VGROUP, WIN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sm);
    line_kernel<KIND, T, RATIO, KP, VGROUP, WIN><<<grid, threads<T, KP>(), sm, st>>>(map, a);
    return check_launch("spo_eval (line) launch");
}
// V positions per consumer warp (the VGROUP the V launch is instantiated with;
// chosen before the prologue, which aligns the groups to cells on dense
// batches).  SPO_VGROUP=1..5 forces; sizes the plane ring cannot hold
// (ring_min) fall back to the next smaller one.
//  * 2 x 1 windows (profiles/r02/v_window.md): fp32 2 below 1.75 positions per
//    cell, else 4; fp64 3.
//  * lines (scripts/micro/vm_sweep.py, profiles/r01/v_groups.jsonl; with dynamic
//    groups and the x weights in shared memory, profiles/r02/v_dynamic.md): fp32
//    3 below 8 per cell (22.7 ms at 4 per cell against 23.2 / 23.3 at 2 / 4),
//    else 4; fp64 k-power 4; fp64 B-spline 1 below 4 per cell, else 3; with
//    cell-aligned groups (cell): 3 (groups of 4 and 5 aligned to cells measured
//    8-70% slower than fixed ones, profiles/r02/v_cell_groups.md).
#ifndef SPO_CELL_VGROUP32
#define SPO_CELL_VGROUP32 3
#endif
#ifndef SPO_CELL_VGROUP64
#define SPO_CELL_VGROUP64 3
#endif
template <typename T>
static int v_group_size(bool kp, int win, double dens, bool cell) {
    const char *e = getenv("SPO_VGROUP");
    if (!kp && win > 1 && win != VWIN) return 1;  // the 2 x 2 window: no groups
    int v;
    if (!kp && win == VWIN) {
        v = e ? atoi(e) : (sizeof(T) == 4 ? (dens < 1.75 ? 2 : 4) : 3);
        v = v < 1 ? 1 : (v > 5 ? 5 : v);
        if (v == 5 && !(ring_min(5) <= ring<T, VWIN, rec_slots<SPO_KIND_V, T, 5, VWIN>()>())) v = 4;
        if (v == 4 && !(ring_min(4) <= ring<T, VWIN, rec_slots<SPO_KIND_V, T, 4, VWIN>()>())) v = 3;
        return v;
    }
    v = e ? atoi(e)
          : (cell ? (sizeof(T) == 4 ? SPO_CELL_VGROUP32 : SPO_CELL_VGROUP64)
                  : (sizeof(T) == 4 ? (dens < 8.0 ? 3 : 4) : (kp ? 4 : (dens < 4.0 ? 1 : 3))));
    v = v < 1 ? 1 : (v > 5 ? 5 : v);
    if (v == 5 && !(ring_min(5) <= ring<T, 1, rec_slots<SPO_KIND_V, T, 5, 1>()>())) v = 4;
    return v;
}

template <int KIND, typename T, bool RATIO, bool KP>
static int launch(const CUtensorMap &map, const LArgs &a, int sms, cudaStream_t st, int win) {
    if constexpr (!KP && KIND == SPO_KIND_V && !RATIO) {
        if (win == VWIN) {
            const int v = a.vgroup;  // v_group_size(): a size this ring holds
            if (v == 1) return launch1<KIND, T, RATIO, false, 1, VWIN>(map, a, sms, st);
            if (v == 2) return launch1<KIND, T, RATIO, false, 2, VWIN>(map, a, sms, st);
            if (v == 3) return launch1<KIND, T, RATIO, false, 3, VWIN>(map, a, sms, st);
            // group sizes whose planes fit the window ring (ring_min; fp64: up to 3)
            if constexpr (ring_min(5) <= ring<T, VWIN, rec_slots<KIND, T, 5, VWIN>()>())
                if (v == 5) return launch1<KIND, T, RATIO, false, 5, VWIN>(map, a, sms, st);
            if constexpr (ring_min(4) <= ring<T, VWIN, rec_slots<KIND, T, 4, VWIN>()>())
                return launch1<KIND, T, RATIO, false, 4, VWIN>(map, a, sms, st);
            return launch1<KIND, T, RATIO, false, 3, VWIN>(map, a, sms, st);
        }
    }
    if constexpr (!KP) {
        if (win > 1) return launch1<KIND, T, RATIO, false, 1, WIN_CELLS>(map, a, sms, st);
    }
    if constexpr (KIND == SPO_KIND_V) {
        const int v = a.vgroup;  // v_group_size(); the ratio epilogue has groups on lines only (win = 1)
        if (v == 2) return launch1<KIND, T, RATIO, KP, 2>(map, a, sms, st);
        if (v == 4) return launch1<KIND, T, RATIO, KP, 4>(map, a, sms, st);
        if (v == 3) return launch1<KIND, T, RATIO, KP, 3>(map, a, sms, st);
        if constexpr (ring_min(5) <= ring<T, 1, rec_slots<KIND, T, 5, 1>()>())
            if (v == 5) return launch1<KIND, T, RATIO, KP, 5>(map, a, sms, st);
    }
    return launch1<KIND, T, RATIO, KP>(map, a, sms, st);
}
template <int KIND, typename T>
static int launch_r(bool ratio, bool kp, const CUtensorMap &map, const LArgs &a, int sms, cudaStream_t st, int win) {
    if (kp)
        return ratio ? launch<KIND, T, true, true>(map, a, sms, st, 1) : launch<KIND, T, false, true>(map, a, sms, st, 1);
    return ratio ? launch<KIND, T, true, false>(map, a, sms, st, win)
                 : launch<KIND, T, false, false>(map, a, sms, st, win);
}

static size_t pad256(size_t b) { return (b + 255) / 256 * 256; }

// Bits the radix sort must look at: the key range [0, keys) of valid
// positions plus the all-ones key of non-finite ones, which must stay above
// it: bit_length(keys) bits (keys itself is not a valid key).
static int line_key_bits(const KeyGeom &kg, const TableGeom &geo) {
    const long long blocks = kg.win > 1 ? 1 : (long long)kg.nbk.x * kg.nbk.y * kg.nbk.z;
    const long long keys = blocks * kg.ext.x * kg.ext.y * kg.ext.z;
    int bits = 0;
    while (bits < 32 && (keys >> bits) != 0) ++bits;
    (void)geo;
    return bits < 1 ? 1 : bits;
}

}  // namespace line

// Workspace of the line path: [header][keys in/out][order in/out][cub temp]
// [records].  The radix-sort temp size is only known on a device; the bound
// below covers it (checked at call time).
// Radix-sort temp storage: exact when a device answers cub's size query
// (the double-buffer variant: ping-pong in our key/value buffers, the temp
// holds histograms and look-back state only), else a generous bound.
static long long line_cub_bytes(long long n) {
    size_t bytes = 0;
    cub::DoubleBuffer<unsigned> keys(nullptr, nullptr);
    cub::DoubleBuffer<int> vals(nullptr, nullptr);
    if (n > 0 && n < (1LL << 31) &&
        cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys, vals, (int)n, 0, 32) == cudaSuccess)
        return (long long)line::pad256(bytes);
    cudaGetLastError();
    return (8LL << 20) + (long long)line::pad256((size_t)n);
}

long long eval_line_workspace_bytes(int dtype, long long n_pos) {
    using namespace line;
    const long long recb = dtype == SPO_F64 ? LT<double>::RECB : LT<float>::RECB;
    const long long runs = (n_pos + BPL - 1) / BPL;
    return WS_HEADER + 4 * (long long)pad256(4 * n_pos) + line_cub_bytes(n_pos) + (long long)pad256(n_pos * recb) +
           runs * PLB;
}

// Whether the line path can take this request (layout, grid, workspace).
bool eval_line_eligible(int dtype, const TableGeom &geo, long long n_pos, long long ws_bytes) {
    using namespace line;
    const int E = dtype == SPO_F64 ? 8 : 4;
    const long long row = (long long)geo.nb * E;
    if (row % BOXB) return false;                                       // boxes must not straddle tiles
    if (((long long)geo.nb * geo.n_tiles * E) % ROWB) return false;     // whole units
    if (geo.nx > MAX_AXIS || geo.ny > MAX_AXIS || geo.nz > MAX_AXIS) return false;
    if (n_pos >= (1LL << 31)) return false;
    return ws_bytes >= eval_line_workspace_bytes(dtype, n_pos);
}

int line_window_cells() { return line::WIN_CELLS; }
int line_v_window() { return line::VWIN; }

// Returns -1 when the request is not taken (the caller falls back).
int ratio_reduce(int kind, const double *partials, long long units, long long n_pos, double *ratios,
                 cudaStream_t st);

int eval_line(int kind, int dtype, const void *table, const TableGeom &geo, const GridArgs &g, const double *pos,
              long long n_pos, void *out, long long ops, long long oss, const long long *out_index, int *status,
              void *workspace, long long ws_bytes, cudaStream_t st, long long lane_limit, const void *coef,
              long long coef_stride, double *ratios, long long ratio_bytes, int win) {
    using namespace line;
    const bool ratio = ratios != nullptr;
    if (!eval_line_eligible(dtype, geo, n_pos, ws_bytes - ratio_bytes) || !aligned16(workspace)) return -1;
    // windows: the B-spline form; the 2 x 1 window for V only
    if (win != 1 && ((win != WIN_CELLS && !(win == VWIN && kind == SPO_KIND_V && !ratio)) || geo.kmul != 1))
        return -1;
    if (!tensor_map_encoder()) return -1;
    const int E = dtype == SPO_F64 ? 8 : 4;
    const int boxl = BOXB / E;

    unsigned char *ws = static_cast<unsigned char *>(workspace);
    const size_t vec = pad256(4 * (size_t)n_pos);
    unsigned *keys_in = reinterpret_cast<unsigned *>(ws + WS_HEADER);
    unsigned *keys_out = reinterpret_cast<unsigned *>(ws + WS_HEADER + vec);
    int *vals_in = reinterpret_cast<int *>(ws + WS_HEADER + 2 * vec);
    int *vals_out = reinterpret_cast<int *>(ws + WS_HEADER + 3 * vec);
    unsigned char *temp = ws + WS_HEADER + 4 * vec;
    cub::DoubleBuffer<unsigned> keys(keys_in, keys_out);
    cub::DoubleBuffer<int> vals(vals_in, vals_out);
    size_t temp_bytes = 0;
    if (cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, keys, vals, (int)n_pos, 0, 32, st) != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    const long long temp_room = line_cub_bytes(n_pos);
    if ((long long)temp_bytes > temp_room) return -1;
    unsigned char *recs = temp + temp_room;
    int *plist = reinterpret_cast<int *>(recs + pad256((size_t)n_pos * (dtype == SPO_F64 ? LT<double>::RECB
                                                                                          : LT<float>::RECB)));
    CUtensorMap map;
    const int r = table_tensor_map(&map, table, geo, dtype, boxl, win_k(win) + 3, win_j(win) + 3);
    if (r) return fail(SPO_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", r);

    if (cudaMemsetAsync(ws, 0, WS_HEADER, st) != cudaSuccess) return check_launch("workspace reset");
    const Grid1D pg = prologue_grid(n_pos);
    // spatial blocks per axis: k-power rows have no halo along z, so blocks
    // flat in z cut the i/j halo re-reads (profiles/r01/nbk_sweep.txt)
    int3 nbk = geo.kmul != 1 ? make_int3(2, 2, 4) : make_int3(NBK, NBK, NBK);
    if (const char *e = getenv("SPO_NBK")) {  // experiment: blocks per axis "i,j,k"
        sscanf(e, "%d,%d,%d", &nbk.x, &nbk.y, &nbk.z);
        if (nbk.x * nbk.y * nbk.z > 255) nbk = make_int3(NBK, NBK, NBK);
    }
    KeyGeom kg;
    kg.nbk = nbk;
    kg.win = win;
    if (win > 1)
        kg.ext = make_int3(geo.nx, (geo.ny + win_j(win) - 1) / win_j(win), (geo.nz + win_k(win) - 1) / win_k(win));
    else
        kg.ext = make_int3((geo.nx + nbk.x - 1) / nbk.x, (geo.ny + nbk.y - 1) / nbk.y, (geo.nz + nbk.z - 1) / nbk.z);
    const int key_bits = line_key_bits(kg, geo);
    line_keys_kernel<<<pg.blocks, pg.threads, 0, st>>>(g, pos, n_pos, keys_in, vals_in, status, kg);
    if (cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys, vals, (int)n_pos, 0, key_bits, st) != cudaSuccess)
        return check_launch("spo_eval (line sort)");
    const int *order = vals.Current();  // the sorted original indices (either buffer)
    // V groups: size, and whether line_runs_kernel aligns them to cells (dense
    // batches: most groups then sit in one cell; SPO_VCELL=0/1 forces)
    const bool kpower = geo.kmul != 1;
    const double dens = (double)n_pos / ((double)geo.nx * geo.ny * geo.nz);
    int vgroup = 1, cellgroups = 0;
    if (kind == SPO_KIND_V && (!ratio || win == 1)) {
        const char *env_cell = getenv("SPO_VCELL");
        // (fp32 k-power tables keep fixed groups of 4: aligned groups of 3 measured +2..4% there,
        // fp64 k-power -9%)
        const bool cell = env_cell ? env_cell[0] == '1'
                                   : dens >= (dtype == SPO_F64 ? SPO_CELL_GROUPS_MIN64 : SPO_CELL_GROUPS_MIN32) &&
                                         !(kpower && dtype != SPO_F64);
        vgroup = dtype == SPO_F64 ? v_group_size<double>(kpower, win, dens, cell)
                                  : v_group_size<float>(kpower, win, dens, cell);
        cellgroups = cell && vgroup > 1 ? vgroup : 0;
    }
    const unsigned run_blocks = (unsigned)((n_pos + (long long)BPL * RUNS_PER_BLOCK - 1) / ((long long)BPL * RUNS_PER_BLOCK));
    if (dtype == SPO_F64) {
        line_records_kernel<double><<<pg.blocks, pg.threads, 0, st>>>(g, pos, order, n_pos, recs, geo.kmul != 1);
        line_runs_kernel<double><<<run_blocks, 32 * RUNS_PER_BLOCK, 0, st>>>(n_pos, recs, plist, win, cellgroups);
    } else {
        line_records_kernel<float><<<pg.blocks, pg.threads, 0, st>>>(g, pos, order, n_pos, recs, geo.kmul != 1);
        line_runs_kernel<float><<<run_blocks, 32 * RUNS_PER_BLOCK, 0, st>>>(n_pos, recs, plist, win, cellgroups);
    }
    int rc = check_launch("spo_eval (line prologue)");
    if (rc) return rc;

    LArgs a;
    a.recs = recs;
    a.plist = plist;
    a.ticket = reinterpret_cast<unsigned *>(ws);
    a.n_pos = n_pos;
    a.nbatch = (n_pos + BPL - 1) / BPL;
    const long long units = (long long)geo.nb * geo.n_tiles * E / ROWB;
    a.n_items = a.nbatch * units;
    if (a.n_items >= (1LL << 32)) return -1;
    a.nb = geo.nb;
    a.out = out;
    a.out_pos_stride = ops;
    a.out_stream_stride = oss;
    a.out_index = out_index;
    a.lane_limit = lane_limit;
    static const char *env_hint = getenv("SPO_L2HINT");
    a.evict_last = !(env_hint && env_hint[0] == '0');
    a.coef = coef;
    a.coef_stride = coef_stride;
    a.partials = ratio ? reinterpret_cast<double *>(ws + eval_line_workspace_bytes(dtype, n_pos)) : nullptr;
    const bool kp = geo.kmul != 1;
    a.kmul = geo.kmul;
    a.cells = (long long)geo.nx * geo.ny * geo.nz;
    const char *env_rot = getenv("SPO_ROTATE");  // experiment: 0 = fixed position-to-warp assignment
    a.rotate = !(env_rot && env_rot[0] == '0');
    // positions from a shared per-run counter (default; SPO_DYNAMIC=0: the
    // rotated static assignment).  +0.3-1% (scripts/micro/dynamic_ab.sh)
    const char *env_dyn = getenv("SPO_DYNAMIC");
    a.dynamic = !(env_dyn && env_dyn[0] == '0');
    const char *env_uni = getenv("SPO_VUNI");
    a.vuni = !(env_uni && env_uni[0] == '0');
    a.vgroup = vgroup;
    a.cellgroups = cellgroups;
    const char *env_vdyn = getenv("SPO_VDYN");
    a.vdyn = !(env_vdyn && env_vdyn[0] == '0');
    // the producer's mbarrier waits spin on try_wait (default); SPO_PSPIN=0:
    // test_wait + nanosleep back-off, measured 1.6% slower on config 5's V
    // (profiles/r02/v_dynamic.md)
    const char *env_pspin = getenv("SPO_PSPIN");
    a.pspin = !(env_pspin && env_pspin[0] == '0');
    a.dz = g.dinv[2];
    a.dz2 = 2.0 * g.dinv[2] * g.dinv[2];

    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (dtype == SPO_F64)
        rc = kind == SPO_KIND_V     ? launch_r<SPO_KIND_V, double>(ratio, kp, map, a, sms, st, win)
             : kind == SPO_KIND_VGL ? launch_r<SPO_KIND_VGL, double>(ratio, kp, map, a, sms, st, win)
                                    : launch_r<SPO_KIND_VGH, double>(ratio, kp, map, a, sms, st, win);
    else
        rc = kind == SPO_KIND_V     ? launch_r<SPO_KIND_V, float>(ratio, kp, map, a, sms, st, win)
             : kind == SPO_KIND_VGL ? launch_r<SPO_KIND_VGL, float>(ratio, kp, map, a, sms, st, win)
                                    : launch_r<SPO_KIND_VGH, float>(ratio, kp, map, a, sms, st, win);
    if (rc || !ratio) return rc;
    return ratio_reduce(kind, a.partials, units, n_pos, ratios, st);
}

}  // namespace spo
