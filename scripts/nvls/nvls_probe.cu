// NVLS (NVSwitch in-switch reduction) bandwidth probe — an experiment for
// SURVEY.md §8(f) NEXT-2, not on the product path.  One CTA grid per call:
//   ar : each GPU reduces its 1/W slice through the multicast address
//        (multimem.ld_reduce) and broadcasts it back (multimem.st) = a flat
//        one-shot NVLS All-Reduce;
//   rs : ld_reduce of the own slice, stored locally (the RS half alone);
//   ag : multimem.st of the own slice (the AG half alone).
// Host code supplies the multicast / unicast pointers (torch symmetric memory)
// and orders calls with process-group barriers (bandwidth probe only).
#include <cstdint>

__device__ __forceinline__ void ld_reduce_v4(const float* mc, float4& v) {
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(mc) : "memory");
}
__device__ __forceinline__ void st_v4_mc(float* mc, const float4& v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};"
               :: "l"(mc), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}

__global__ void nvls_kernel(float* mc, float* local, uint64_t n, int rank, int world, int mode) {
  const uint64_t per = n / world, v0 = (uint64_t)rank * per / 4, v1 = ((uint64_t)rank + 1) * per / 4;
  for (uint64_t i = v0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < v1; i += (uint64_t)gridDim.x * blockDim.x) {
    float4 v;
    if (mode == 2) {  // ag: broadcast the own slice
      v = reinterpret_cast<const float4*>(local)[i];
      st_v4_mc(mc + 4 * i, v);
      continue;
    }
    ld_reduce_v4(mc + 4 * i, v);
    if (mode == 0)
      st_v4_mc(mc + 4 * i, v);  // ar
    else
      reinterpret_cast<float4*>(local)[i] = v;  // rs
  }
}

extern "C" int nvls_launch(void* mc, void* local, uint64_t n, int rank, int world, int mode, int blocks, void* stream) {
  nvls_kernel<<<blocks, 512, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<float*>(mc), static_cast<float*>(local),
                                                                     n, rank, world, mode);
  return (int)cudaGetLastError();
}
