// Host-side fp64 <-> fp32 conversion rate with T threads (measurement for the
// e2e path: would a narrowed model over PCIe beat the fp64 DMA?).
// gcc -O3 -mavx2 -pthread tools/hostconv.c -o /tmp/hostconv
#define _GNU_SOURCE
#include <immintrin.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static double *src; static float *dst; static double *back; static size_t N; static int T;
static double now(void){struct timespec t;clock_gettime(CLOCK_MONOTONIC,&t);return t.tv_sec+1e-9*t.tv_nsec;}
static void *narrow(void *a){size_t id=(size_t)a,b=N/T*id,e=id==T-1?N:N/T*(id+1);
  for(size_t i=b;i+8<=e;i+=8){__m128 lo=_mm256_cvtpd_ps(_mm256_loadu_pd(src+i));__m128 hi=_mm256_cvtpd_ps(_mm256_loadu_pd(src+i+4));
    _mm256_stream_ps(dst+i,_mm256_set_m128(hi,lo));}
  _mm_sfence();return 0;}
static void *widen(void *a){size_t id=(size_t)a,b=N/T*id,e=id==T-1?N:N/T*(id+1);
  for(size_t i=b;i+8<=e;i+=8){__m256 v=_mm256_loadu_ps(dst+i);
    _mm256_stream_pd(back+i,_mm256_cvtps_pd(_mm256_castps256_ps128(v)));_mm256_stream_pd(back+i+4,_mm256_cvtps_pd(_mm256_extractf128_ps(v,1)));}
  _mm_sfence();return 0;}
static void *copy(void *a){size_t id=(size_t)a,b=N/T*id,e=id==T-1?N:N/T*(id+1);memcpy(back+b,src+b,(e-b)*8);return 0;}
static double run(void*(*f)(void*)){pthread_t th[64];double t0=now();for(int i=0;i<T;i++)pthread_create(&th[i],0,f,(void*)(size_t)i);for(int i=0;i<T;i++)pthread_join(th[i],0);return now()-t0;}
int main(int argc,char**argv){N=132800000/T*0+132800000; 
  src=aligned_alloc(64,N*8);dst=aligned_alloc(64,N*4);back=aligned_alloc(64,N*8);
  for(size_t i=0;i<N;i++){src[i]=(double)(float)(i*1e-7);} memset(dst,0,N*4);memset(back,0,N*8);
  int ts[]={1,2,4,8,16,32};
  for(int k=0;k<6;k++){T=ts[k];double a=1e9,b=1e9,c=1e9;for(int r=0;r<3;r++){double x=run(narrow);if(x<a)a=x;x=run(widen);if(x<b)b=x;x=run(copy);if(x<c)c=x;}
    printf("threads %2d: narrow %.1f ms (%.1f GB/s of fp64 in)  widen %.1f ms (%.1f GB/s of fp64 out)  memcpy %.1f ms (%.1f GB/s)\n",T,a*1e3,N*8/a/1e9,b*1e3,N*8/b/1e9,c*1e3,N*8/c/1e9);}
  return memcmp(src,back,N*8)!=0;}
