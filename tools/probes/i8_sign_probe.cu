// Does tcgen05.mma kind::i8 honour per-operand signedness (idesc bits 7 / 10)?
// A = 128 x 32 bytes of 0xC8 (200 as u8, -56 as s8), B = 64 x 32 bytes of 0x01.
// Every element is equal, so the smem layout does not matter: D = 32 * a * b.
// Expected: A u8 -> 6400, A s8 -> -1792; B = 0xFF: u8 255, s8 -1.
#include <cstdio>
#include "../../paper_2604_12163_b200/csrc/common.cuh"
using namespace nimg;

__global__ void probe(int* out, uint32_t idesc, uint8_t aval, uint8_t bval) {
  // K-major, 128-B swizzle: rows are 128 B apart even though one MMA reads 32 B of each
  __shared__ __align__(1024) uint8_t a[128 * 128];
  __shared__ __align__(1024) uint8_t b[64 * 128];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 128 * 128; i += blockDim.x) a[i] = aval;
  for (int i = threadIdx.x; i < 64 * 128; i += blockDim.x) b[i] = bval;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  fence_proxy_async_smem();
  if (threadIdx.x < 32) tmem_alloc(&slot, 64);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot;
  if (threadIdx.x == 0) {
    umma_i8(tm, make_sdesc_k128(smem_u32(a)), make_sdesc_k128(smem_u32(b)), idesc, 0u);
    umma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  uint32_t r[4];
  tmem_ld4(tm + ((uint32_t)((threadIdx.x / 32) * 32) << 16), r);
  tmem_ld_wait();
  if (threadIdx.x == 0) out[0] = (int)r[0];
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tm, 64); }
}

int main() {
  int* d;
  cudaMalloc(&d, 4);
  const uint32_t base = (2u << 4) | ((uint32_t)(64 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  struct { const char* name; uint32_t bits; uint8_t a, b; int want; } cases[] = {
      {"A s8 B s8", (1u << 7) | (1u << 10), 0xC8, 0x01, -1792},
      {"A u8 B s8", (1u << 10), 0xC8, 0x01, 6400},
      {"A s8 B u8", (1u << 7), 0xC8, 0xFF, -56 * 255 * 32},
      {"A u8 B u8", 0u, 0xC8, 0xFF, 200 * 255 * 32},
  };
  int bad = 0;
  for (auto& c : cases) {
    probe<<<1, 128>>>(d, base | c.bits, c.a, c.b);
    int h = 0;
    cudaError_t e = cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost);
    printf("%s: got %d want %d %s (%s)\n", c.name, h, c.want, h == c.want ? "OK" : "MISMATCH", cudaGetErrorString(e));
    bad += h != c.want;
  }
  return bad;
}
