// Host decode-loop microbenchmark (tools only): g++ -O3 tools/decode_bench.cpp -o tools/decode_bench -lpthread
// args: threads mode(0 = chained permute, 1 = independent block sums) fence-per-chunk(0/1)
#include <immintrin.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <thread>
#include <vector>
#include <cstring>
__attribute__((target("avx512f"))) void chunk_old(const uint32_t* d, uint64_t* out, uint32_t len, uint64_t acc, bool fence){
  out[0]=acc; uint32_t i=1;
  while (i < len && (reinterpret_cast<uintptr_t>(out + i) & 63u)) { acc += d[i]; out[i++] = acc; }
  const __m512i z=_mm512_setzero_si512(), last=_mm512_set1_epi64(7); __m512i run=_mm512_set1_epi64(acc);
  for (; i + 8 <= len; i += 8) {
    __m512i x=_mm512_cvtepu32_epi64(_mm256_loadu_si256((const __m256i*)(d+i)));
    x=_mm512_add_epi64(x,_mm512_alignr_epi64(x,z,7)); x=_mm512_add_epi64(x,_mm512_alignr_epi64(x,z,6)); x=_mm512_add_epi64(x,_mm512_alignr_epi64(x,z,4));
    x=_mm512_add_epi64(x,run); run=_mm512_permutexvar_epi64(last,x); _mm512_stream_si512((__m512i*)(out+i),x);
  }
  acc=(uint64_t)_mm_cvtsi128_si64(_mm512_castsi512_si128(run));
  for (; i < len; ++i) { acc += d[i]; out[i] = acc; }
  if (fence) _mm_sfence();
}
__attribute__((target("avx512f"))) void chunk_new(const uint32_t* d, uint64_t* out, uint32_t len, uint64_t acc, bool fence){
  out[0]=acc; uint32_t i=1;
  while (i < len && (reinterpret_cast<uintptr_t>(out + i) & 63u)) { acc += d[i]; out[i++] = acc; }
  const __m512i z=_mm512_setzero_si512(), last=_mm512_set1_epi64(7); __m512i run=_mm512_set1_epi64(acc);
  for (; i + 8 <= len; i += 8) {
    __m512i x=_mm512_cvtepu32_epi64(_mm256_loadu_si256((const __m256i*)(d+i)));
    x=_mm512_add_epi64(x,_mm512_alignr_epi64(x,z,7)); x=_mm512_add_epi64(x,_mm512_alignr_epi64(x,z,6)); x=_mm512_add_epi64(x,_mm512_alignr_epi64(x,z,4));
    const __m512i b=_mm512_permutexvar_epi64(last,x);
    _mm512_stream_si512((__m512i*)(out+i),_mm512_add_epi64(x,run)); run=_mm512_add_epi64(run,b);
  }
  acc=(uint64_t)_mm_cvtsi128_si64(_mm512_castsi512_si128(run));
  for (; i < len; ++i) { acc += d[i]; out[i] = acc; }
  if (fence) _mm_sfence();
}
int main(int argc,char**argv){
  int T=atoi(argv[1]); int mode=atoi(argv[2]); bool fence=atoi(argv[3]);
  uint64_t N=1ull<<29; uint32_t* d=(uint32_t*)aligned_alloc(64,N*4); uint64_t* o=(uint64_t*)aligned_alloc(64,N*8+64);
  memset(d,1,N*4); memset(o,0,N*8);
  uint64_t* oo=o+3; // misaligned output like the real buffer
  for(int rep=0;rep<3;rep++){
  auto t0=std::chrono::steady_clock::now(); std::vector<std::thread> th;
  for(int t=0;t<T;t++) th.emplace_back([=]{ uint64_t per=(N/T)/4096*4096, lo=t*per;
     const uint64_t ring=1<<20; // 4 MiB per-thread input window (LLC)
     for(uint64_t s=0;s<per;s+=4096){ const uint32_t* src=d+(uint64_t)t*ring+(s%ring);
       if(mode==0) chunk_old(src,oo+lo+s,4096,s,fence); else chunk_new(src,oo+lo+s,4096,s,fence);} _mm_sfence(); });
  for(auto&x:th)x.join();
  double dt=std::chrono::duration<double>(std::chrono::steady_clock::now()-t0).count();
  printf("T=%d mode=%d fence=%d: out %.1f GB/s\n",T,mode,(int)fence,(N/T/4096*4096*T)*8/dt/1e9);}
}
