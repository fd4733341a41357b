// Microbenchmark: MUFU-bound exp pass of one warp per sub-partition while the other warp of the
// sub-partition runs the softmax's other work (FMNMX max pass, tcgen05.ld, st.shared, nothing).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I../../paper_2511_21095_b200/csrc -o exp_interf exp_interf.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"

using namespace gesr;

__device__ __forceinline__ void ffma2(float& d0, float& d1, float a0, float a1, float b0, float b1,
                                      float c0, float c1) {
  asm("{\n .reg .b64 a, b, c, d;\n mov.b64 a, {%2, %3};\n mov.b64 b, {%4, %5};\n"
      " mov.b64 c, {%6, %7};\n fma.rn.f32x2 d, a, b, c;\n mov.b64 {%0, %1}, d;\n}"
      : "=f"(d0), "=f"(d1) : "f"(a0), "f"(a1), "f"(b0), "f"(b1), "f"(c0), "f"(c1));
}
__device__ __forceinline__ void fadd2(float& d0, float& d1, float a0, float a1, float b0, float b1) {
  asm("{\n .reg .b64 a, b, d;\n mov.b64 a, {%2, %3};\n mov.b64 b, {%4, %5};\n"
      " add.rn.f32x2 d, a, b;\n mov.b64 {%0, %1}, d;\n}"
      : "=f"(d0), "=f"(d1) : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}

// 2^x for a pair on the FMA pipe only (no min/max, no MUFU): clamp x to [-126, 126] with a
// saturating FFMA, split x = j + f with the 1.5*2^23 magic add, degree-3 polynomial for 2^f,
// exponent added with an IMAD.
__device__ __forceinline__ void exp2_fma2(float& y0, float& y1, float x0, float x1) {
  float u0, u1;
  asm("fma.rn.sat.f32 %0, %1, %2, %3;" : "=f"(u0) : "f"(x0), "f"(1.0f / 252.0f), "f"(0.5f));
  asm("fma.rn.sat.f32 %0, %1, %2, %3;" : "=f"(u1) : "f"(x1), "f"(1.0f / 252.0f), "f"(0.5f));
  constexpr float kMagic = 12582912.0f;   // 1.5 * 2^23
  float t0, t1, s0, s1, f0, f1, p0, p1;
  ffma2(t0, t1, u0, u1, 252.0f, 252.0f, kMagic - 126.0f, kMagic - 126.0f);   // round(x') in low bits
  fadd2(s0, s1, -t0, -t1, kMagic - 126.0f, kMagic - 126.0f);                   // -126 - round(x')
  ffma2(f0, f1, u0, u1, 252.0f, 252.0f, s0, s1);                                // f = x' - round(x')
  ffma2(p0, p1, f0, f1, 0.054848f, 0.054848f, 0.24180661f, 0.24180661f);
  ffma2(p0, p1, p0, p1, f0, f1, 0.6932482f, 0.6932482f);
  ffma2(p0, p1, p0, p1, f0, f1, 0.99998866f, 0.99998866f);
  y0 = __int_as_float(__float_as_int(t0) * (1 << 23) + __float_as_int(p0));
  y1 = __int_as_float(__float_as_int(t1) * (1 << 23) + __float_as_int(p1));
}

template <int MODE>
__global__ void __launch_bounds__(256, 1) k(uint32_t* out, int iters, float sl2, long long* clk) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t mbar_s;
  const int warp = threadIdx.x / 32;
  if (warp == 0) { tmem_alloc(&slot, 512); tmem_relinquish(); }
  if (threadIdx.x == 0) { mbar_init(&mbar_s, 1); fence_mbar_init(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  uint32_t r[128];
  for (int i = 0; i < 128; ++i) r[i] = __float_as_uint((threadIdx.x * 128 + i) * 1e-5f);
  uint32_t sink = 0;
  if (warp < 4 && MODE >= 8) {
    // the kernel's exp pass variants (one warp per SMSP, other warps idle)
    float m = 0.5f;
    const uint32_t prow = smem_u32(smem) + threadIdx.x * 128;
    const uint32_t taddr = tmem + (((warp & 3) * 32) << 16);
    uint32_t sink2 = 0;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      uint32_t x[128];
#pragma unroll
      for (int i = 0; i < 128; ++i) x[i] = r[i];
      if (MODE == 13 || MODE == 14) {
        // pack in place into x[0..63], then store after the loop
#pragma unroll
        for (int kk = 0; kk < 64; ++kk) {
          const float p0 = ex2(__uint_as_float(x[2 * kk]) - m), p1 = ex2(__uint_as_float(x[2 * kk + 1]) - m);
          const int a = (kk & 3) * 2;
          fadd2(acc[a], acc[a + 1], acc[a], acc[a + 1], p0, p1);
          x[kk] = pack_bf16x2(p0, p1);
        }
        if (MODE == 13) {
#pragma unroll
          for (int q = 0; q < 16; ++q)
            st_shared_v4(prow + (q >> 3) * 16384 + (((q & 7) ^ (threadIdx.x & 7)) << 4), x[4 * q], x[4 * q + 1], x[4 * q + 2], x[4 * q + 3]);
        } else {
          tmem_st32(taddr, x);
          tmem_st32(taddr + 32, x + 32);
          tmem_st_wait();
        }
      } else {
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          uint32_t pw[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int kk = q * 4 + u;
            float p0, p1;
            if (MODE >= 10 && MODE <= 12 && (kk % (MODE - 8)) == 0) {
              exp2_fma2(p0, p1, __uint_as_float(x[2 * kk]) - m, __uint_as_float(x[2 * kk + 1]) - m);
            } else {
              p0 = ex2(__uint_as_float(x[2 * kk]) - m);
              p1 = ex2(__uint_as_float(x[2 * kk + 1]) - m);
            }
            const int a = (kk & 3) * 2;
            fadd2(acc[a], acc[a + 1], acc[a], acc[a + 1], p0, p1);
            pw[u] = pack_bf16x2(p0, p1);
          }
          st_shared_v4(prow + (q >> 3) * 16384 + (((q & 7) ^ (threadIdx.x & 7)) << 4), pw[0], pw[1], pw[2], pw[3]);
        }
      }
      sink2 += x[0] ^ x[5];
      m += (((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]))) * 1e-9f;
    }
    const long long t1 = clock64();
    sink ^= sink2;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
  } else if (warp < 4) {
    float m = 0.5f;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      const float nm = -m;
#pragma unroll
      for (int kk = 0; kk < 64; ++kk) {
        float x0, x1;
        ffma2(x0, x1, __uint_as_float(r[2 * kk]), __uint_as_float(r[2 * kk + 1]), sl2, sl2, nm, nm);
        const float p0 = ex2(x0), p1 = ex2(x1);
        const int a = (kk & 3) * 2;
        fadd2(acc[a], acc[a + 1], acc[a], acc[a + 1], p0, p1);
        r[kk] = pack_bf16x2(p0, p1) ^ r[kk + 64];
      }
      m += (((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]))) * 1e-9f;
    }
    const long long t1 = clock64();
    for (int i = 0; i < 128; ++i) sink ^= r[i];
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
  } else {
    const uint32_t taddr = tmem + (((warp & 3) * 32) << 16);
    const uint32_t srow = smem_u32(smem) + (threadIdx.x - 128) * 128;
    for (int it = 0; it < iters * 4; ++it) {
      if (MODE == 1) {         // FMNMX max pass
        float mx[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) mx[e] = -1e30f;
#pragma unroll
        for (int kk = 0; kk < 128; ++kk) mx[kk & 7] = fmaxf(mx[kk & 7], __uint_as_float(r[kk]));
        sink += __float_as_uint(fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                                      fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7]))));
        r[it & 127] += 1;
      } else if (MODE == 4) {  // 3-input max (max.f32 a, b, c)
        float mx[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) mx[e] = -1e30f;
#pragma unroll
        for (int kk = 0; kk < 128; kk += 2) {
          float y;
          asm("max.f32 %0, %1, %2, %3;" : "=f"(y) : "f"(mx[(kk / 2) & 7]), "f"(__uint_as_float(r[kk])), "f"(__uint_as_float(r[kk + 1])));
          mx[(kk / 2) & 7] = y;
        }
        sink += __float_as_uint(fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                                      fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7]))));
        r[it & 127] += 1;
      } else if (MODE == 5) {  // integer max on the raw bits (IMNMX)
        int mx[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) mx[e] = -2147483647;
#pragma unroll
        for (int kk = 0; kk < 128; ++kk) mx[kk & 7] = max(mx[kk & 7], static_cast<int>(r[kk]));
        sink += max(max(max(mx[0], mx[1]), max(mx[2], mx[3])), max(max(mx[4], mx[5]), max(mx[6], mx[7])));
        r[it & 127] += 1;
      } else if (MODE == 6) {  // packed bf16x2 max (HMNMX2) on the raw high halves
        uint32_t mx[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) mx[e] = 0xff80ff80u;
#pragma unroll
        for (int kk = 0; kk < 64; ++kk) {
          uint32_t y;
          asm("max.bf16x2 %0, %1, %2;" : "=r"(y) : "r"(mx[kk & 7]), "r"(__byte_perm(r[2 * kk], r[2 * kk + 1], 0x7632)));
          mx[kk & 7] = y;
        }
        sink += mx[0] ^ mx[1] ^ mx[2] ^ mx[3] ^ mx[4] ^ mx[5] ^ mx[6] ^ mx[7];
        r[it & 127] += 1;
      } else if (MODE == 7) {  // FFMA stream (issue competition only)
        float a0 = __uint_as_float(r[0]), a1 = __uint_as_float(r[1]), a2 = __uint_as_float(r[2]), a3 = __uint_as_float(r[3]);
#pragma unroll
        for (int kk = 0; kk < 32; ++kk) { a0 = a0 * 1.0001f + 0.1f; a1 = a1 * 1.0001f + 0.1f; a2 = a2 * 1.0001f + 0.1f; a3 = a3 * 1.0001f + 0.1f; }
        sink += __float_as_uint(a0 + a1 + a2 + a3);
      } else if (MODE == 2) {  // tcgen05.ld 128 columns
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld32(taddr + c * 32, r + c * 32);
        tmem_ld_wait();
        sink += r[it & 127];
      } else if (MODE == 9) {  // kernel-like overhead: ld 128 cols + 16 STS, then ~1000 clk idle
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld32(taddr + c * 32, r + c * 32);
        tmem_ld_wait();
        const long long w0 = clock64();
        while (clock64() - w0 < 1200) {}
        sink += r[it & 127];
      } else if (MODE == 15) {  // tcgen05 MMA stream (SS M=128 N=128 K=16) into columns 256..383
        if (threadIdx.x == 128) {
          const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 16384);
          const uint32_t idesc = make_idesc_bf16(128, 128, 0, 0);
#pragma unroll 1
          for (int rep = 0; rep < 64; ++rep)
#pragma unroll
            for (int ks = 0; ks < 4; ++ks)
              mma_ss(tmem + 256, make_sdesc(sa + ks * 32, 16, 1024, 2), make_sdesc(sb + ks * 32, 16, 1024, 2), idesc, 1u);
          mma_commit(&mbar_s);
          mbar_wait(&mbar_s, it & 1);
        }
        __syncwarp();
      } else if (MODE == 3) {  // 16 x st.shared.v4
#pragma unroll
        for (int c = 0; c < 16; ++c) st_shared_v4(srow + ((c * 16) & 127) + (c / 8) * 16384, r[c], r[c + 1], r[c + 2], sink);
        fence_proxy_async_smem();
        sink += 1;
      }
    }
  }
  if (sink == 0x1234567u) out[threadIdx.x] = sink;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

int main() {
  uint32_t* d;
  long long* c;
  cudaMalloc(&d, 4096);
  cudaMalloc(&c, 4096 * 8);
  const char* names[16] = {"alone", "+FMNMX max pass", "+tcgen05.ld x128", "+16 STS.128 + proxy fence",
                          "+3-input max.f32", "+IMNMX on bits", "+max.bf16x2", "+FFMA stream",
                          "kernel loop (STS inside), alone", "kernel loop + ld/1.2k clk",
                          "kernel loop, poly 1 in 2", "kernel loop, poly 1 in 3", "kernel loop, poly 1 in 4",
                          "pack in place, 16 STS after loop", "pack in place, 2 tcgen05.st after", "kernel loop + MMA stream (other warp)"};
  for (int mode = 0; mode < 16; ++mode) {
    const int iters = 400;
    auto launch = [&] {
      if (mode == 0) k<0><<<148, 256, 40000>>>(d, iters, 0.1f, c);
      if (mode == 1) k<1><<<148, 256, 40000>>>(d, iters, 0.1f, c);
      if (mode == 2) k<2><<<148, 256, 40000>>>(d, iters, 0.1f, c);
      if (mode == 3) k<3><<<148, 256, 40000>>>(d, iters, 0.1f, c);
      if (mode == 4) k<4><<<148, 256, 40000>>>(d, iters, 0.1f, c);
      if (mode == 5) k<5><<<148, 256, 40000>>>(d, iters, 0.1f, c);
      if (mode == 6) k<6><<<148, 256, 40000>>>(d, iters, 0.1f, c);
      if (mode == 7) k<7><<<148, 256, 40000>>>(d, iters, 0.1f, c);
      if (mode == 8) k<8><<<148, 256, 40000>>>(d, iters, 0.1f, c);
      if (mode == 9) k<9><<<148, 256, 40000>>>(d, iters, 0.1f, c);
      if (mode == 10) k<10><<<148, 256, 40000>>>(d, iters, 0.1f, c);
      if (mode == 11) k<11><<<148, 256, 40000>>>(d, iters, 0.1f, c);
      if (mode == 12) k<12><<<148, 256, 40000>>>(d, iters, 0.1f, c);
      if (mode == 13) k<13><<<148, 256, 40000>>>(d, iters, 0.1f, c);
      if (mode == 14) k<14><<<148, 256, 40000>>>(d, iters, 0.1f, c);
      if (mode == 15) k<15><<<148, 256, 40000>>>(d, iters, 0.1f, c);
    };
    launch();
    cudaError_t e = cudaDeviceSynchronize();
    launch();
    e = cudaDeviceSynchronize();
    long long h;
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("exp pass (128 exps/thread, 1 warp/SMSP) %-28s %.0f clk (MUFU bound 1024) %s\n", names[mode],
           double(h) / iters, cudaGetErrorString(e));
  }
  return 0;
}
