// Minimal tcgen05 kind::tf32 GEMM probe (round-2 groundwork for the chi = 32 stages):
// D[128 x N] = A[128 x K] * B[N x K]^T with K-major SWIZZLE_NONE operands in shared memory,
// the accumulator in TMEM, read back with tcgen05.ld.32x32b.  Checks against a CPU reference
// on TF32-rounded inputs and times back-to-back MMAs.
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

constexpr int M = 128;
#ifndef PN
#define PN 64
#endif
#ifndef PK
#define PK 32
#endif
constexpr int N = PN, K = PK;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// K-major, no swizzle: core matrix = 8 rows x 16 B (4 tf32 along K); LBO = stride between the
// K-adjacent core matrices, SBO = stride between 8-row groups.
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;   // version (Blackwell)
  return d;                  // base_offset 0, lbo_mode 0, layout SWIZZLE_NONE (0)
}

__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n) {
  return (1u << 4)            // D format F32
       | (2u << 7)            // A TF32
       | (2u << 10)           // B TF32
       | (0u << 15) | (0u << 16)   // A, B K-major
       | ((uint32_t)(n >> 3) << 17)
       | ((uint32_t)(m >> 4) << 24);
}

// offset (in floats) of element (row, k) in the K-major interleaved layout
__host__ __device__ inline int koff(int row, int k, int kdim) {
  const int r = row >> 3, i = row & 7, c = k >> 2, j = k & 3;
  const int lbo = 32;                 // floats: 128 B between K-adjacent core matrices
  const int sbo = (kdim / 4) * 32;    // floats: all K chunks of one 8-row group
  return r * sbo + c * lbo + i * 4 + j;
}

__global__ void umma_probe(const float* A, const float* B, float* D, int reps, long long* cycles) {
  __shared__ __align__(1024) float sa[M * K];
  __shared__ __align__(1024) float sb[N * K];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < M * K; e += blockDim.x) sa[koff(e / K, e % K, K)] = A[e];
  for (int e = tid; e < N * K; e += blockDim.x) sb[koff(e / K, e % K, K)] = B[e];
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" :: "r"(smem_u32(&tmem_base)), "n"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" :: "r"(smem_u32(&mbar)));
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tmem_base;
  const uint32_t idesc = idesc_tf32(M, N);
  long long t0 = clock64();
  uint32_t phase = 0;
  for (int rep = 0; rep < reps; ++rep) {
    if (tid == 0) {
      for (int s = 0; s < K / 8; ++s) {
        const uint64_t da = smem_desc(smem_u32(sa) + s * 2 * 128, 128, (K / 4) * 128);
        const uint64_t db = smem_desc(smem_u32(sb) + s * 2 * 128, 128, (K / 4) * 128);
        const uint32_t acc = s > 0 ? 1u : 0u;
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
                     :: "r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];\n" :: "r"(smem_u32(&mbar)));
    }
    // every thread waits for the MMA group to complete
    asm volatile("{\n\t.reg .pred done;\n\tLAB_WAIT:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
                 "@!done bra LAB_WAIT;\n\t}\n" :: "r"(smem_u32(&mbar)), "r"(phase));
    phase ^= 1;
  }
  long long t1 = clock64();
  // pipelined: 4*reps MMAs back to back (accumulating), one commit at the end
  if (tid == 0) {
    for (int rep = 0; rep < reps; ++rep)
      for (int s = 0; s < K / 8; ++s) {
        const uint64_t da = smem_desc(smem_u32(sa) + s * 2 * 128, 128, (K / 4) * 128);
        const uint64_t db = smem_desc(smem_u32(sb) + s * 2 * 128, 128, (K / 4) * 128);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
                     :: "r"(tmem + 64), "l"(da), "l"(db), "r"(idesc), "r"(1u));
      }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];\n" :: "r"(smem_u32(&mbar)));
  }
  asm volatile("{\n\t.reg .pred done;\n\tLAB_WAIT2:\n\t"
               "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
               "@!done bra LAB_WAIT2;\n\t}\n" :: "r"(smem_u32(&mbar)), "r"(phase));
  long long t2 = clock64();
  if (tid == 0) cycles[1] = t2 - t1;
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  // warp w reads TMEM lanes 32w..32w+31 (rows), 16 columns at a time
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t v[16];
    const uint32_t addr = tmem + ((uint32_t)(warp * 32) << 16) + c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                 : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n");
    for (int j = 0; j < 16; ++j) D[(warp * 32 + lane) * N + c0 + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" :: "r"(tmem), "n"(128));
  if (tid == 0) *cycles = t1 - t0;
}

static float tf32r(float x) {   // round-to-nearest onto 10 mantissa bits
  uint32_t u; memcpy(&u, &x, 4);
  u = (u + 0x1000u) & 0xFFFFE000u;
  float y; memcpy(&y, &u, 4); return y;
}

int main() {
  std::vector<float> A(M * K), B(N * K), D(M * N), R(M * N);
  for (int i = 0; i < M * K; ++i) A[i] = tf32r(std::sin(0.37f * i) * 0.5f);
  for (int i = 0; i < N * K; ++i) B[i] = tf32r(std::cos(0.11f * i + 0.3f));
  for (int r = 0; r < M; ++r)
    for (int c = 0; c < N; ++c) {
      double s = 0; for (int k = 0; k < K; ++k) s += double(A[r * K + k]) * B[c * K + k];
      R[r * N + c] = float(s);
    }
  float *dA, *dB, *dD; long long* dc;  // dc[0]: per-rep round trips, dc[1]: pipelined
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4); cudaMalloc(&dc, 16);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  for (int reps : {1, 1000}) {
    umma_probe<<<1, 128>>>(dA, dB, dD, reps, dc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("CUDA error: %s\n", cudaGetErrorString(e)); return 1; }
    long long cycs[2]; cudaMemcpy(cycs, dc, 16, cudaMemcpyDeviceToHost);
    const long long cyc = cycs[0];
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0;
    for (int i = 0; i < M * N; ++i) { maxerr = fmax(maxerr, fabs(D[i] - R[i])); maxref = fmax(maxref, fabs(R[i])); }
    printf("reps=%d  max|D-ref|=%.3e (max|ref| %.3f)  D[0]=%f ref=%f D[5*N+7]=%f ref=%f  cycles/rep=%.1f (%d MMAs of 128x%dx8 each)\n",
           reps, maxerr, maxref, D[0], R[0], D[5 * N + 7], R[5 * N + 7], double(cyc) / reps, K / 8, N);
    const double fl = 2.0 * M * N * K * reps;
    printf("   pipelined: %.1f cycles per 128x%dx%d group -> %.0f TF32 flop/cycle/SM\n", double(cycs[1]) / reps, N, K, fl / double(cycs[1]));
  }
  return 0;
}
