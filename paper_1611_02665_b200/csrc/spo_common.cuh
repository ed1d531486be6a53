// spo_common.cuh -- shared host/device helpers for libspo_b200.so.
#pragma once
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/spo_b200.h"

namespace spo {

// Thread-local last-error text (spo_last_error).
inline std::string &last_error_slot() {
    static thread_local std::string s;
    return s;
}

inline int fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    last_error_slot() = buf;
    return code;
}

inline int ok() {
    last_error_slot().clear();
    return SPO_OK;
}

// The library links its own static CUDA runtime, whose current device is
// independent of the caller's (torch's) runtime.  Before launching, make it
// follow the device that owns the buffer the launch writes.
inline int bind_device(const void *ptr) {
    if (!ptr) return SPO_OK;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
        cudaGetLastError();
        return fail(SPO_ERR_CONTRACT, "pointer %p is not a CUDA allocation", ptr);
    }
    if (at.type != cudaMemoryTypeDevice && at.type != cudaMemoryTypeManaged)
        return fail(SPO_ERR_CONTRACT, "pointer %p is not device memory", ptr);
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess || cur != at.device) {
        if (cudaSetDevice(at.device) != cudaSuccess) {
            cudaGetLastError();
            return fail(SPO_ERR_CUDA, "cudaSetDevice(%d) failed", at.device);
        }
    }
    return SPO_OK;
}

// Every device buffer of a call must live on the device bind_device picked:
// a foreign pointer would fault inside the kernel, so reject it up front.
inline int check_on_device(const void *ptr, const char *what) {
    if (!ptr) return SPO_OK;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
        cudaGetLastError();
        return fail(SPO_ERR_CONTRACT, "%s (%p) is not a CUDA allocation", what, ptr);
    }
    int cur = -1;
    cudaGetDevice(&cur);
    if ((at.type != cudaMemoryTypeDevice && at.type != cudaMemoryTypeManaged) || at.device != cur)
        return fail(SPO_ERR_CONTRACT, "%s (%p) is not memory of device %d", what, ptr, cur);
    return SPO_OK;
}

// `out` of spo_eval_lanes: memory of the current device, or of a peer the
// current device can reach over NVLink/PCIe (peer access is enabled here; an
// IPC mapping opened with lazy peer access is already reachable).
inline int check_reachable(const void *ptr, const char *what) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
        cudaGetLastError();
        return fail(SPO_ERR_CONTRACT, "%s (%p) is not a CUDA allocation", what, ptr);
    }
    if (at.type != cudaMemoryTypeDevice && at.type != cudaMemoryTypeManaged)
        return fail(SPO_ERR_CONTRACT, "%s (%p) is not device memory", what, ptr);
    int cur = -1;
    cudaGetDevice(&cur);
    if (at.device == cur || at.type == cudaMemoryTypeManaged) return SPO_OK;
    int can = 0;
    if (cudaDeviceCanAccessPeer(&can, cur, at.device) != cudaSuccess || !can) {
        cudaGetLastError();
        return fail(SPO_ERR_CONTRACT, "%s (%p) lives on device %d, which device %d cannot reach", what, ptr,
                    at.device, cur);
    }
    const cudaError_t e = cudaDeviceEnablePeerAccess(at.device, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
        return fail(SPO_ERR_CUDA, "cudaDeviceEnablePeerAccess(%d) from %d failed", at.device, cur);
    }
    cudaGetLastError();
    return SPO_OK;
}

inline int check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(SPO_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
    return ok();
}

inline bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

inline int dtype_size(int dtype) { return dtype == SPO_F64 ? 8 : 4; }

// Launch shape of the one-thread-per-position prologue kernels (mapping,
// weights, sort keys).  Their fp64 arithmetic is ALU-bound per SM, so a small
// batch gets smaller blocks, enough of them to reach every SM: 256 threads
// from 2 x 148 x 256 positions, down to 64.
struct Grid1D {
    unsigned blocks;
    int threads;
};
inline Grid1D prologue_grid(long long n) {
    int threads = 256;
    while (threads > 64 && (n + threads - 1) / threads < 2 * 148) threads >>= 1;
    long long blocks = (n + threads - 1) / threads;
    if (blocks > 148LL * 16) blocks = 148LL * 16;
    if (blocks < 1) blocks = 1;
    return Grid1D{(unsigned)blocks, threads};
}

// Device table geometry shared by the eval, pack and fill kernels.
// B-spline form: rows k' < nz + 3 per (i', j'), the stencil of cell k0 is
// rows k0..k0+3.  k-power form (SPO_TABLE_KPOWER): rows 4*k0 + r (r < 4) hold
// the power-basis coefficients q_r of cell k0 along z, nzp = 4 nz, kmul = 4.
struct TableGeom {
    int nx, ny, nz;        // reference grid counts
    int nxp, nyp, nzp;     // wrap-padded counts (n + 3); k-power: nzp = 4 nz
    int nb;                // row length (lanes) per tile
    int n_tiles;
    long long tile_stride; // elements per tile
    int kmul;              // row of cell k0's first stencil row = kmul * k0
};

inline int make_geom(const int32_t *n3, int32_t nb, int32_t n_tiles, int dtype, TableGeom *g,
                     bool kpower = false) {
    if (!n3) return fail(SPO_ERR_CONTRACT, "grid counts pointer is NULL");
    for (int a = 0; a < 3; ++a)
        if (n3[a] < 4) return fail(SPO_ERR_CONFIG, "grid count %d on axis %d must be >= 4", n3[a], a);
    const int quantum = dtype == SPO_F64 ? 16 : 32;  // 128-byte rows
    if (nb <= 0 || nb % quantum)
        return fail(SPO_ERR_CONTRACT, "row length nb=%d must be a positive multiple of %d", nb,
                    quantum);
    if (n_tiles <= 0) return fail(SPO_ERR_CONFIG, "n_tiles=%d must be >= 1", n_tiles);
    g->nx = n3[0];
    g->ny = n3[1];
    g->nz = n3[2];
    g->nxp = n3[0] + 3;
    g->nyp = n3[1] + 3;
    g->nzp = kpower ? 4 * n3[2] : n3[2] + 3;
    g->kmul = kpower ? 4 : 1;
    g->nb = nb;
    g->n_tiles = n_tiles;
    g->tile_stride = (long long)g->nxp * g->nyp * g->nzp * nb;
    return SPO_OK;
}

}  // namespace spo
