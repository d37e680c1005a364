// Test helpers (TEST INFRASTRUCTURE, not part of the product library): a kernel that holds
// SMs until a device flag is set -- the shape of an NCCL kernel on a comm stream that waits on
// its peers -- so a GPU test can run the long-K GEMMs (wave barriers) against SM contention.
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// One block per SM (the dynamic shared memory makes each block exclusive): spin until *flag
// != 0 or the safety timeout, then record in status[0] whether the timeout released it.
// times (globaltimer ns, optional): times[0] = first holder start, times[1] = last holder end
__global__ void k_hold(volatile int* flag, uint64_t timeout_ns, int* status, int* started,
                       unsigned long long* times) {
  extern __shared__ uint8_t smem[];
  smem[threadIdx.x] = 0;
  const uint64_t t0 = gtimer();
  if (threadIdx.x == 0) {
    atomicAdd(started, 1);
    if (times) atomicMin(times, (unsigned long long)t0);
    while (*flag == 0) {
      __nanosleep(1000);
      if (gtimer() - t0 > timeout_ns) {
        atomicExch(status, 1);
        break;
      }
    }
    if (times) atomicMax(times + 1, (unsigned long long)gtimer());
  }
  __syncthreads();
}

// sets the flag; times[2] (optional) = when
__global__ void k_set(int* flag, unsigned long long* times) {
  if (times) times[2] = gtimer();
  __threadfence();
  *reinterpret_cast<volatile int*>(flag) = 1;
}

extern "C" {

int th_hold_sms(int n_blocks, int smem_bytes, int* flag, long long timeout_ns, int* status, int* started,
                unsigned long long* times, void* stream) {
  if (cudaFuncSetAttribute(k_hold, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes) != cudaSuccess)
    return 1;
  k_hold<<<n_blocks, 32, smem_bytes, static_cast<cudaStream_t>(stream)>>>(flag, (uint64_t)timeout_ns, status,
                                                                          started, times);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

int th_set_flag(int* flag, unsigned long long* times, void* stream) {
  k_set<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(flag, times);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

}  // extern "C"
