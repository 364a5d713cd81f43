#include <cstdio>
#include <cstdint>
#include <cstring>
__global__ void k(const double* a, const double* b, double* c, int n){ int i=threadIdx.x; if(i<n){ double x=a[i], y=b[i]; double r; asm("add.rn.f64 %0, %1, %2;" : "=d"(r) : "d"(x), "d"(y)); c[i]=r; } }
static double bits(uint64_t u){ double d; memcpy(&d,&u,8); return d; }
static uint64_t ub(double d){ uint64_t u; memcpy(&u,&d,8); return u; }
int main(){
  const int n=8;
  double a[n]={bits(0x7ff8000000000000ull), 1.0, bits(0xfff8000000000000ull), bits(0x7ff0000000000000ull), -0.0, 0.0, bits(0x7ff8000000001234ull), bits(0x7ff0000000000001ull)};
  double b[n]={1.0, bits(0x7ff8000000000000ull), bits(0x7ff8000000000000ull), bits(0xfff0000000000000ull), 0.0, -0.0, bits(0xfff8000000005678ull), 1.0};
  double *da,*db,*dc; cudaMalloc(&da,64);cudaMalloc(&db,64);cudaMalloc(&dc,64);
  cudaMemcpy(da,a,64,cudaMemcpyHostToDevice);cudaMemcpy(db,b,64,cudaMemcpyHostToDevice);
  k<<<1,32>>>(da,db,dc,n); double c[n]; cudaMemcpy(c,dc,64,cudaMemcpyDeviceToHost);
  for(int i=0;i<n;i++){ volatile double x=a[i], y=b[i]; double h = x + y; printf("%d a=%016llx b=%016llx gpu=%016llx cpu=%016llx\n",i,(unsigned long long)ub(a[i]),(unsigned long long)ub(b[i]),(unsigned long long)ub(c[i]),(unsigned long long)ub(h)); }
  return 0; }
