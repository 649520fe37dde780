#include <cstdio>
#include <cstring>
#include <cmath>
__global__ void k(const float* a, const float* b, float* o, int n) {
  int i = threadIdx.x;
  if (i < n) {
    float mn, mx;
    asm("min.f32 %0, %1, %2;" : "=f"(mn) : "f"(a[i]), "f"(b[i]));
    asm("max.f32 %0, %1, %2;" : "=f"(mx) : "f"(a[i]), "f"(b[i]));
    o[4*i] = mn; o[4*i+1] = mx; o[4*i+2] = fminf(a[i], b[i]); o[4*i+3] = fmaxf(a[i], b[i]);
  }
}
unsigned u(float f){unsigned x; memcpy(&x,&f,4); return x;}
int main(){
  float qn = nanf(""); float nqn = -qn;
  float A[] = {0.0f, -0.0f, 1.0f, qn, qn, -0.0f, nqn, 2.0f};
  float B[] = {-0.0f, 0.0f, qn, 1.0f, qn, nqn, -0.0f, nqn};
  int n = 8; float *da,*db,*dout; float out[32];
  cudaMalloc(&da,64); cudaMalloc(&db,64); cudaMalloc(&dout,128);
  cudaMemcpy(da,A,32,cudaMemcpyHostToDevice); cudaMemcpy(db,B,32,cudaMemcpyHostToDevice);
  k<<<1,32>>>(da,db,dout,n); cudaMemcpy(out,dout,128,cudaMemcpyDeviceToHost);
  for(int i=0;i<n;i++) printf("a=%08x b=%08x  min=%08x max=%08x fminf=%08x fmaxf=%08x\n", u(A[i]),u(B[i]),u(out[4*i]),u(out[4*i+1]),u(out[4*i+2]),u(out[4*i+3]));
}
