// Max abs error of ss_atan2f vs float64 atan2 on a dense circle (GPU): nvcc -gencode arch=compute_100a,code=sm_100a -O3 -Iinclude -o /tmp/at tools/atan2_check.cu
#include <cstdio>
#include <cmath>
#include "../paper_2605_05876_b200/csrc/ss_common.cuh"
#include "../paper_2605_05876_b200/csrc/shading.cuh"
__global__ void k(int n, double *err) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double ang = -3.14159265358979 + 6.28318530717959 * (i + 0.5) / n;
    float y = (float)sin(ang) * 0.7f, x = (float)cos(ang) * 0.7f;
    double ref = atan2((double)y, (double)x);
    double e = fabs((double)ss_atan2f(y, x) - ref);
    double e2 = fabs((double)atan2f(y, x) - ref);
    atomicMax((unsigned long long*)err, __double_as_longlong(e));
    atomicMax((unsigned long long*)(err+1), __double_as_longlong(e2));
}
int main(){ double *e; cudaMallocManaged(&e, 16); e[0]=e[1]=0; int n=1<<24; k<<<n/256,256>>>(n,e); cudaDeviceSynchronize(); printf("max err fast %.3e  atan2f %.3e\n", e[0], e[1]);
  // special cases on host-side via device
  return 0; }
