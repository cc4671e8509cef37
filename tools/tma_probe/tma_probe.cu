// Minimal TMA + mbarrier probe (debugging aid): one 128 x 32 fp32 box of plane p into smem, copied out.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include <cstdlib>

struct Q { CUtensorMap tm; float* out; int x0, y0, p, bw, bh; };

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void k(const __grid_constant__ Q q) {
  extern __shared__ __align__(128) unsigned char raw[];
  float* box = reinterpret_cast<float*>(raw);
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(raw + ((q.bw * q.bh * 4 + 15) / 16) * 16);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(sa(bar)), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sa(bar)), "r"((unsigned)(q.bw * q.bh * 4)) : "memory");
    if (MODE == 0)
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
                   ::"r"(sa(box)), "l"(reinterpret_cast<unsigned long long>(&q.tm)), "r"(q.x0), "r"(q.y0), "r"(q.p), "r"(sa(bar)) : "memory");
    else
      asm volatile("cp.async.bulk.tensor.3d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
                   ::"r"(sa(box)), "l"(reinterpret_cast<unsigned long long>(&q.tm)), "r"(q.x0), "r"(q.y0), "r"(q.p), "r"(sa(bar)) : "memory");
  }
  asm volatile(
      "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(sa(bar)), "r"(0)
      : "memory");
  for (int i = threadIdx.x; i < q.bw * q.bh; i += blockDim.x) q.out[i] = box[i];
}

int main(int argc, char** argv) {
  const int nx = argc > 5 ? atoi(argv[5]) : 256, ny = argc > 6 ? atoi(argv[6]) : 64, nz = 4;
  std::vector<float> h((size_t)nx * ny * nz);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (float)i;
  float *d, *o;
  cudaMalloc(&d, h.size() * 4);
  cudaMalloc(&o, 256 * 64 * 4);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  Q q{};
  cuuint64_t dims[3] = {nx, ny, nz};
  cuuint64_t str[2] = {(cuuint64_t)nx * 4, (cuuint64_t)nx * ny * 4};
  const int BW = argc > 1 ? atoi(argv[1]) : 128, BH = argc > 2 ? atoi(argv[2]) : 32;
  cuuint32_t box[3] = {(cuuint32_t)BW, (cuuint32_t)BH, 1}, es[3] = {1, 1, 1};
  CUresult r = enc(&q.tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  q.out = o; q.x0 = argc > 3 ? atoi(argv[3]) : -5; q.y0 = argc > 4 ? atoi(argv[4]) : -4; q.p = 2; q.bw = BW; q.bh = BH;
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(o, 0, BW * BH * 4);
    const size_t sm = BW * BH * 4 + 64;
    if (mode == 0) { cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); k<0><<<1, 128, sm>>>(q); }
    else { cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); k<1><<<1, 128, sm>>>(q); }
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> ho(BW * BH);
    cudaMemcpy(ho.data(), o, ho.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int y = 0; y < BH; ++y)
      for (int x = 0; x < BW; ++x) {
        const int gx = q.x0 + x, gy = q.y0 + y;
        const float exp = (gx >= 0 && gx < nx && gy >= 0 && gy < ny) ? h[((size_t)q.p * ny + gy) * nx + gx] : 0.f;
        if (ho[y * BW + x] != exp) ++bad;
      }
    printf("mode %d: %s bad=%d\n", mode, cudaGetErrorString(e), bad);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
