// expf_ref_check.c -- exhaustive check of the host-side replication of
// glibc's expf (the algorithm csrc/common.cuh expf_ref evaluates on the GPU)
// against the host libm: every float in (-130, 88), plus monotonicity over
// [-103, 0].  gcc -O2 -ffp-contract=off tools/expf_ref_check.c -lm && ./a.out
#include <math.h>
#include <stdio.h>
#include <stdint.h>
#include <string.h>
static uint64_t asu(double d){uint64_t u;memcpy(&u,&d,8);return u;}
static double asd(uint64_t u){double d;memcpy(&d,&u,8);return d;}
#define N 32
static const double invln2N = 0x1.71547652b82fep0 * N;
static const double shift = 0x1.8p+52;
static const double C0 = 0x1.c6af84b912394p-5 / N / N / N, C1 = 0x1.ebfce50fac4f3p-3 / N / N, C2 = 0x1.62e42ff0c52d6p-1 / N;
static uint64_t Ttab[N];
float my_expf(float x) {
  double xd = x, z = invln2N * xd, kd = z + shift; uint64_t ki = asu(kd); kd -= shift;
  double r = z - kd; uint64_t t = Ttab[ki % N]; t += ki << (52 - 5); double s = asd(t);
  double zz = fma(C0, r, C1), y = fma(C2, r, 1.0), r2 = r*r; y = fma(zz, r2, y); y = y * s; return (float)y;
}
int main(){
  for (int i=0;i<N;i++){ double v = exp2((double)i/N); Ttab[i] = asu(v) - ((uint64_t)i << 52)/N; }
  long nonmono=0; float prev=0; int first=1;
  for (uint32_t u = 0; u < 0xffffffffu; u+=1) {
    float x; memcpy(&x,&u,4);
    if (!(x > -130.0f && x < 88.0f)) continue;
    float g = expf(x), m = my_expf(x);
    if (m != g) printf("mismatch x=%a glibc=%a mine=%a\n", x, g, m);
  }
  // monotone over increasing x in [-103, 0]
  for (float x = -103.0f; x <= 0.0f; x = nextafterf(x, 1.0f)) { float m = my_expf(x); if (!first && m < prev) nonmono++; prev=m; first=0; }
  printf("nonmono=%ld\n", nonmono);
  printf("T0=%a\n", asd(Ttab[1]));
}
