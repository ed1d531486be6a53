// umma_probe.cu -- feasibility probe for a tensor-core (tcgen05, kind::tf32)
// formulation of the plane contraction (next steps).  Not part
// of the library.
//
// One CTA: A = one table plane (128 lanes x 16 rows fp32) in several smem
// layouts, B = 16 x N weights (K-major, no swizzle), D in TMEM (M = 128
// lanes, N columns).  Checks D against a host fp64 product of the
// tf32-truncated operands and times back-to-back MMAs (MACs per SM clock).
// Findings (one B200): MN-major tf32 A works only in the "128B swizzle with
// 32-byte atoms" layout (descriptor layout type 1, LBO = next 32 lanes,
// SBO = next 4 k-rows; TMA's CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) -- the
// plain 128B-swizzle and no-swizzle MN layouts leave D at zero; K-major A
// works; 2048 MACs/clk at N = 256, 1364 at N = 64, 364 at N = 16.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_probe umma_probe.cu && ./umma_probe
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e = (x);                                                               \
        if (e != cudaSuccess) {                                                            \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            exit(1);                                                                       \
        }                                                                                  \
    } while (0)

constexpr int M = 128, K = 16;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// A (m, k) byte offset in the TMA SW128 plane layout: box m/32 at 2 KB, rows
// k at 128 B (8-row atoms of 1 KB), 16-byte chunks XOR-swizzled by row % 8.
__host__ __device__ inline uint32_t a_offset(int m, int k) {
    const int box = m >> 5, mm = m & 31;
    const int chunk = (mm >> 2) ^ (k & 7);
    return box * 2048 + (k >> 3) * 1024 + (k & 7) * 128 + chunk * 16 + (mm & 3) * 4;
}
// B (k, n) byte offset, K-major no swizzle: 8x16B core matrices; LBO = 128 B
// (next 4 k), SBO = 512 B (next 8 n).
__host__ __device__ inline uint32_t b_offset(int k, int n) {
    return (n >> 3) * 512 + (k >> 2) * 128 + (n & 7) * 16 + (k & 3) * 4;
}

__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3fff);
    d |= (uint64_t)((lbo >> 4) & 0x3fff) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3fff) << 32;
    d |= (uint64_t)1 << 46;  // version 1 (sm_100)
    d |= (uint64_t)(layout & 7) << 61;
    return d;
}

__host__ __device__ constexpr uint32_t instr_desc(int m, int n, bool ak) {
    return (1u << 4)               // D f32
           | (2u << 7)             // A tf32
           | (2u << 10)            // B tf32
           | ((ak ? 0u : 1u) << 15)  // A MN-major (or K-major)
           | (0u << 16)            // B K-major
           | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

// A (m, k), MN-major no swizzle: core = 8 k-rows x 16 B (4 m), SBO = 128 B
// (next 4 m), LBO = 4096 B (next 8 k)
__host__ __device__ inline uint32_t ami_offset(int m, int k) {
    return (k >> 3) * 4096 + (m >> 2) * 128 + (k & 7) * 16 + (m & 3) * 4;
}
// A (m, k), MN-major "128B swizzle, 32-byte atoms" (the only MN-major layout
// for 32-bit operands): 4 k-rows of 128 B per 512 B atom, 32-byte granules
// XOR-swizzled by k % 4; atoms of 32 lanes at 2 KB (one TMA box of 16 rows)
__host__ __device__ inline uint32_t a32_offset(int m, int k) {
    const int mm = m & 31;
    return (m >> 5) * 2048 + (k >> 2) * 512 + (k & 3) * 128 + (((mm >> 3) ^ (k & 3)) << 5) + (mm & 7) * 4;
}
// A (m, k), K-major no swizzle (same core-matrix scheme as B)
__host__ __device__ inline uint32_t ak_offset(int m, int k) {
    return (m >> 3) * 512 + (k >> 2) * 128 + (m & 7) * 16 + (k & 3) * 4;
}

template <int N, int VAR>
__global__ void probe(const float *A, const float *B, float *D, int iters, long long *cycles) {
    extern __shared__ unsigned char smem_raw[];
    // swizzle atoms need 1024-byte alignment of the shared-memory address
    unsigned char *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    unsigned char *sa = smem;          // 8 KB
    unsigned char *sb = smem + 8192;   // K x N x 4
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    for (int e = tid; e < M * K; e += blockDim.x) {
        const int m = e % M, k = e / M;
        const uint32_t off = VAR == 1 ? ak_offset(m, k) : VAR == 3 ? ami_offset(m, k)
                             : VAR >= 4 ? a32_offset(m, k) : a_offset(m, k);
        *reinterpret_cast<float *>(sa + off) = A[k * M + m];
    }
    for (int e = tid; e < K * N; e += blockDim.x) {
        const int n = e % N, k = e / N;
        *reinterpret_cast<float *>(sb + b_offset(k, n)) = B[k * N + n];
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                     "r"(N < 32 ? 32 : N));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> tensor core reads
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_base;

    if (iters < 0) {  // TMEM store/load self-test: D[row][col] = row * 1000 + col
        for (int c = 0; c < N; c += 8) {
            uint32_t v[8];
            for (int e = 0; e < 8; ++e) v[e] = __float_as_uint((float)((32 * warp + lane) * 1000 + c + e));
            asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                             tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)c),
                         "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        if (tid == 0)
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bar)));
    }
    constexpr uint32_t idesc = instr_desc(M, N, VAR == 1);
    const uint32_t a0 = smem_u32(sa), b0 = smem_u32(sb);
    long long t0 = 0, t1 = 0;
    if (tid == 0 && iters >= 0) {
        t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) {  // K = 16 as two K = 8 steps
                const uint64_t da = VAR == 1   ? smem_desc(a0 + ks * 256, 128, 512, 0)
                                    : VAR == 0 ? smem_desc(a0 + ks * 1024, 2048, 1024, 2)
                                    : VAR == 2 ? smem_desc(a0 + ks * 1024, 1024, 2048, 2)
                                    : VAR == 3 ? smem_desc(a0 + ks * 4096, 4096, 128, 0)
                                    : VAR == 4 ? smem_desc(a0 + ks * 1024, 2048, 512, 1)
                                               : smem_desc(a0 + ks * 1024, 512, 2048, 1);
                const uint64_t db = smem_desc(b0 + ks * 256, 128, 512, 0);     // no swizzle
                const uint32_t acc = (it > 0 || ks > 0) ? 1u : 0u;
                asm volatile(
                    "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                    "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                    "l"(da), "l"(db), "r"(idesc), "r"(acc));
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(&bar)));
    }
    asm volatile(
        "{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(
            smem_u32(&bar)));
    if (tid == 0 && iters >= 0) {
        t1 = clock64();
        *cycles = t1 - t0;
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // D: warp w reads TMEM lanes 32w..32w+31, N columns, 8 at a time
    for (int c = 0; c < N; c += 8) {
        uint32_t r[8];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
            : "r"(tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)c));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int e = 0; e < 8; ++e) D[(32 * warp + lane) * N + c + e] = __uint_as_float(r[e]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(N < 32 ? 32 : N));
}

static float tf32(float x) {
    uint32_t u;
    memcpy(&u, &x, 4);
    u &= 0xffffe000u;
    float y;
    memcpy(&y, &u, 4);
    return y;
}

template <int N, int VAR>
static int run(int iters) {
    std::vector<float> A(M * K), B(K * N), D(M * N);
    srand(1);
    for (auto &x : A) x = (float)rand() / RAND_MAX * 2 - 1;
    for (auto &x : B) x = (float)rand() / RAND_MAX * 2 - 1;
    float *dA, *dB, *dD;
    long long *dc, cyc = 0;
    CK(cudaMalloc(&dA, A.size() * 4));
    CK(cudaMalloc(&dB, B.size() * 4));
    CK(cudaMalloc(&dD, D.size() * 4));
    CK(cudaMalloc(&dc, 8));
    CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
    const size_t sm = 8192 + K * N * 4 + 1024;
    CK(cudaFuncSetAttribute(probe<N, VAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    probe<N, VAR><<<1, 128, sm>>>(dA, dB, dD, iters, dc);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost));
    double worst = 0, mag = 0;
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
            double ref = 0;
            for (int k = 0; k < K; ++k) ref += (double)tf32(A[k * M + m]) * tf32(B[k * N + n]);
            ref *= iters;
            worst = fmax(worst, fabs(D[m * N + n] - ref));
            mag = fmax(mag, fabs(ref));
        }
    const double macs = (double)M * N * K * iters;
    if (worst / mag > 1e-4) {
        for (int q = 0; q < 4; ++q) {
            double ref = 0;
            for (int k = 0; k < K; ++k) ref += (double)tf32(A[k * M + q]) * tf32(B[k * N + 1]);
            printf("  D[%d][1] = %g  ref %g\n", q, D[q * N + 1], ref * iters);
        }
    }
    printf("A %s N=%3d iters=%6d  max|D-ref|/max|ref| = %.3e  cycles=%lld  MACs/clk=%.1f\n",
           VAR == 1 ? "K-major " : VAR == 0 ? "MN-SW128" : VAR == 2 ? "MN-SW128s" : VAR == 3 ? "MN-none "
           : VAR == 4 ? "MN-SW128-32B" : "MN-SW128-32Bs", N, iters,
           worst / mag, cyc,
           macs / (double)cyc);
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dD);
    cudaFree(dc);
    return worst / mag < 1e-4 ? 0 : 1;
}

static int selftest() {
    constexpr int N = 64;
    float *dD;
    long long *dc;
    std::vector<float> D(M * N);
    CK(cudaMalloc(&dD, D.size() * 4));
    CK(cudaMalloc(&dc, 8));
    const size_t sm = 8192 + K * N * 4 + 1024;
    CK(cudaFuncSetAttribute(probe<N, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    float *dA, *dB;
    CK(cudaMalloc(&dA, M * K * 4));
    CK(cudaMalloc(&dB, K * N * 4));
    CK(cudaMemset(dA, 0, M * K * 4));
    CK(cudaMemset(dB, 0, K * N * 4));
    probe<N, 0><<<1, 128, sm>>>(dA, dB, dD, -1, dc);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) bad += D[m * N + n] != (float)(m * 1000 + n);
    printf("TMEM st/ld self-test: %d mismatches (D[5][3] = %g)\n", bad, D[5 * N + 3]);
    return bad != 0;
}

int main() {
    int bad = selftest();
    bad |= run<64, 1>(1);
    run<64, 4>(1);
    run<64, 5>(1);
    bad |= run<64, 4>(4096) & run<64, 5>(4096);
    run<256, 4>(4096);
    printf(bad ? "FAIL\n" : "OK\n");
    return bad;
}
