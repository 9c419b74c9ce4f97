#include <cstdio>
#include <cstdint>
__global__ void spin(uint64_t ns){uint64_t t0,t;asm volatile("mov.u64 %0, %%globaltimer;":"=l"(t0));do{asm volatile("mov.u64 %0, %%globaltimer;":"=l"(t));}while(t-t0<ns);}
__global__ void tick(uint64_t* out){uint64_t t0,t;asm volatile("mov.u64 %0, %%globaltimer;":"=l"(t0));
  uint64_t mn=~0ull; int changes=0; uint64_t prev=t0;
  for(int i=0;i<2000000 && changes<64;i++){asm volatile("mov.u64 %0, %%globaltimer;":"=l"(t)); if(t!=prev){ if(t-prev<mn) mn=t-prev; prev=t; changes++;}}
  out[0]=mn; out[1]=prev-t0; out[2]=changes;}
__global__ void empty(){}
int main(){uint64_t* d; cudaMalloc(&d,64); tick<<<1,1>>>(d); uint64_t h[3]; cudaMemcpy(h,d,24,cudaMemcpyDeviceToHost);
 printf("globaltimer min increment %llu ns, span %llu ns over %llu changes\n",(unsigned long long)h[0],(unsigned long long)h[1],(unsigned long long)h[2]);
 cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b); cudaStream_t s; cudaStreamCreateWithFlags(&s,cudaStreamNonBlocking);
 for(uint64_t ns: {0ull,1000ull,5000ull,10000ull,20000ull,40000ull,100000ull}){ float tot=0; int R=50; float mn=1e9;
  for(int r=0;r<R;r++){cudaEventRecord(a,s); if(ns) spin<<<1,32,0,s>>>(ns); else empty<<<1,32,0,s>>>(); cudaEventRecord(b,s); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms,a,b); tot+=ms; if(ms<mn) mn=ms;}
  printf("spin %6llu ns: mean %.2f us min %.2f us\n",(unsigned long long)ns, tot/R*1e3, mn*1e3);}
 return 0;}
