// i8_probe.cu — tcgen05.mma kind::i8 with A in TMEM, B in shared memory (K-major, no swizzle):
// (1) correctness of the assumed operand layouts (A: TMEM lane = row, 32-bit column = 4
//     consecutive k bytes; B: 8-row x 16-byte core matrices, LBO = K stride, SBO = N stride),
// (2) issue cost of back-to-back M = 128, N = 16/32/64, K = 32 MMAs from one thread.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/i8_probe tools/i8_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

template <int N>
__global__ void k_probe(const uint8_t* A, const int8_t* B, int K, int reps, int* D, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&slot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 32) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // B: [k/16][n/8][n%8][16 B]
  for (int i = threadIdx.x; i < N * K; i += blockDim.x) {
    const int n = i / K, k = i % K;
    sm[(k / 16) * (N * 16) + (n / 8) * 128 + (n % 8) * 16 + (k % 16)] = static_cast<uint8_t>(B[n * K + k]);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tb = slot;
  if (warp < 4) {
    const int r = warp * 32 + lane;
    for (int c0 = 0; c0 < K / 4; c0 += 16) {
      uint32_t v[16];
      for (int j = 0; j < 16; ++j) {
        const uint8_t* p = A + r * K + 4 * (c0 + j);
        v[j] = p[0] | (p[1] << 8) | (p[2] << 16) | (static_cast<uint32_t>(p[3]) << 24);
      }
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
              tb + (static_cast<uint32_t>(warp * 32) << 16) + c0),
          "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
          "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
          : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t idesc = (2u << 4) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) | (8u << 24);
  const uint64_t dhi = (static_cast<uint64_t>((N * 16) >> 4) << 16) | (static_cast<uint64_t>(128 >> 4) << 32) | (1ull << 46);
  const uint32_t dcol = tb + 128;
  if (warp == 4) {
    long long t0 = 0;
    for (int rep = 0; rep < reps + 1; ++rep) {
      if (rep == 1) t0 = clock64();
      for (int ks = 0; ks < K / 32; ++ks) {
        const uint64_t bd = dhi | static_cast<uint64_t>(((su32(sm) + ks * N * 32) >> 4) & 0x3FFF);
        const uint32_t acc = (ks > 0) ? 1u : 0u;
        asm volatile(
            "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
            "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(dcol),
            "r"(tb + ks * 8), "l"(bd), "r"(idesc), "r"(acc)
            : "memory");
      }
    }
    asm volatile(
        "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(su32(&bar))
        : "memory");
    long long t1 = clock64();
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n" ::"r"(su32(&bar))
        : "memory");
    long long t2 = clock64();
    if (lane == 0) {
      cyc[0] = t1 - t0;  // issue time of reps * K/32 MMAs
      cyc[1] = t2 - t0;  // to completion
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp < 4) {
    const int r = warp * 32 + lane;
    for (int c0 = 0; c0 < N; c0 += 16) {
      uint32_t v[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
            "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
          : "r"(dcol + (static_cast<uint32_t>(warp * 32) << 16) + c0));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int j = 0; j < 16; ++j) D[r * N + c0 + j] = static_cast<int>(v[j]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(256));
}

template <int N>
int run(int K, int reps) {
  std::vector<uint8_t> A(128 * K);
  std::vector<int8_t> B(N * K);
  srand(7 + N);
  for (auto& a : A) a = rand() % 16;
  for (auto& b : B) b = static_cast<int8_t>(rand() % 255 - 127);
  uint8_t* dA;
  int8_t* dB;
  int* dD;
  long long* dc;
  cudaMalloc(&dA, A.size());
  cudaMalloc(&dB, B.size());
  cudaMalloc(&dD, 128 * N * 4);
  cudaMalloc(&dc, 16);
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
  const int smem = N * K + 1024;
  cudaFuncSetAttribute(k_probe<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_probe<N><<<1, 160, smem>>>(dA, dB, K, reps, dD, dc);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("N=%d error %s\n", N, cudaGetErrorString(e));
    return 1;
  }
  std::vector<int> D(128 * N);
  long long c[2];
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(c, dc, 16, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int r = 0; r < 128; ++r)
    for (int n = 0; n < N; ++n) {
      long long s = 0;
      for (int k = 0; k < K; ++k) s += static_cast<long long>(A[r * K + k]) * B[n * K + k];
      if (s != D[r * N + n] && bad++ < 3) printf("  mismatch r=%d n=%d got %d want %lld\n", r, n, D[r * N + n], s);
    }
  const double nm = static_cast<double>(reps) * (K / 32);
  printf("N=%d K=%d: %s (%d bad); issue %.1f cycles/MMA, completion %.1f cycles/MMA\n", N, K, bad ? "WRONG" : "exact", bad,
         c[0] / nm, c[1] / nm);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dD);
  cudaFree(dc);
  return bad != 0;
}

int main() {
  int bad = 0;
  bad += run<16>(512, 200);
  bad += run<32>(512, 200);
  bad += run<64>(512, 200);
  bad += run<32>(256, 400);
  return bad;
}
