// tq_debug.cuh — race / uninitialised-read stress instrumentation (diagnostic build only).
//
// compute-sanitizer is closed on this GPU pool, so the shared-memory pipelines are checked by
// perturbation instead (tools/race_stress.py): built with -DTQ_DEBUG_RACE,
//   * every dynamic shared-memory byte is poisoned with 0xFF (a NaN pattern) at kernel entry,
//     so a read of a slot nothing wrote turns the result non-finite;
//   * every barrier (__syncthreads, __syncwarp, the sweeps' team_sync) is preceded by a
//     pseudo-random sleep of 0..~2 us per thread, which reorders warps and stretches every
//     cp.async / store -> load window, so a missing barrier or wait shows up as a run-to-run
//     or build-to-build difference.
// The production build defines nothing here.
#pragma once

#ifdef TQ_DEBUG_RACE
__device__ __forceinline__ void tq_dbg_delay() {
  unsigned long long c;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(c));
  unsigned h = (unsigned)c ^ (threadIdx.x * 0x9E3779B9u) ^ (blockIdx.x * 0x85EBCA6Bu);
  h ^= h >> 13; h *= 0xC2B2AE35u; h ^= h >> 16;
  __nanosleep(h & 2047u);
}
#define __syncthreads() do { tq_dbg_delay(); __syncthreads(); } while (0)
#define __syncwarp(...) do { tq_dbg_delay(); __syncwarp(__VA_ARGS__); } while (0)
#define TQ_SMEM_POISON(buf)                                                            \
  do {                                                                                 \
    unsigned _sz;                                                                      \
    asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(_sz));                      \
    for (unsigned _i = threadIdx.x * 4u; _i + 4u <= _sz; _i += blockDim.x * 4u)        \
      *reinterpret_cast<unsigned*>((buf) + _i) = 0xFFFFFFFFu;                          \
    __syncthreads();                                                                   \
  } while (0)
#else
#define TQ_SMEM_POISON(buf) do { } while (0)
#endif
