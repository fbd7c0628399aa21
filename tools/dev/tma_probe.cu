// Minimal TMA probe: loads one 3-D uint8 box through vf::tma helpers and checks it.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cudaTypedefs.h>
#include "../../paper_1009_0959_b200/csrc/vf_tma.cuh"

__global__ void probe(const __grid_constant__ CUtensorMap map, uint8_t* out, int c0, int c1, int c2) {
  __shared__ alignas(128) uint8_t buf[10 * 112];
  __shared__ alignas(8) uint64_t bar;
  if (threadIdx.x == 0) {
    vf::tma::mbar_init(&bar, 1);
    vf::tma::fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    vf::tma::mbar_expect_tx(&bar, 10 * 112);
    vf::tma::load_3d(buf, &map, &bar, c0, c1, c2);
  }
  vf::tma::mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < 10 * 112; i += blockDim.x) out[i] = buf[i];
}

int main(int argc, char** argv) {
  const int W = 64, H = 20, B = 2;
  const size_t rb = W * 3;
  std::vector<uint8_t> h(B * H * rb);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (uint8_t)(i * 7 + 3);
  uint8_t *d, *o;
  cudaMalloc(&d, h.size()); cudaMalloc(&o, 1120);
  cudaMemcpy(d, h.data(), h.size(), cudaMemcpyHostToDevice);
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
  CUtensorMap map;
  cuuint64_t dims[3] = {rb, (cuuint64_t)H, (cuuint64_t)B};
  cuuint64_t strides[2] = {rb, rb * H};
  cuuint32_t box[3] = {112, 10, 1}, es[3] = {1, 1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  int cs[1][3] = {{atoi(argv[1]), atoi(argv[2]), atoi(argv[3])}};
  for (auto& c : cs) {
    probe<<<1, 128>>>(map, o, c[0], c[1], c[2]);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<uint8_t> g(1120);
    cudaMemcpy(g.data(), o, 1120, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int rr = 0; rr < 10; ++rr)
      for (int cc = 0; cc < 112; ++cc) {
        int gy = c[1] + rr, gx = c[0] + cc;
        uint8_t want = (gy >= 0 && gy < H && gx >= 0 && gx < (int)rb) ? h[(size_t)c[2] * H * rb + gy * rb + gx] : 0;
        bad += g[rr * 112 + cc] != want;
      }
    printf("coords (%d,%d,%d): %s, mismatches %d\n", c[0], c[1], c[2], cudaGetErrorString(e), bad);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
