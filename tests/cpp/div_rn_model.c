/* Host model of the device quotient div_rn / div_rn_wide
 * (paper_2008_01440_b200/csrc/kernels.cuh), the same operations with C99 fma():
 * checks it against the IEEE division x / b bit for bit over random operands of
 * every class (normal, subnormal, tiny, huge, around 2^960, arbitrary bit
 * patterns incl. inf / NaN) for six divisors. Usage: div_rn_model [samples/divisor]
 * Built and run by tests/test_host.py (compiled with -ffp-contract=off). */
#include <stdlib.h>
#include <math.h>
#include <stdio.h>
#include <stdint.h>
#include <string.h>
static uint64_t s=88172645463325252ULL;
static uint64_t rnd(){ s^=s<<13; s^=s>>7; s^=s<<17; return s; }
static double bits(uint64_t u){ double d; memcpy(&d,&u,8); return d; }
static uint64_t ubits(double d){ uint64_t u; memcpy(&u,&d,8); return u; }
static double wide(double x, double b, double inv) {
  const double ax = fabs(x);
  const int tiny = ax < 0x1p-960, huge = ax > 0x1p960;
  const double sc = tiny ? 0x1p1000 : (huge ? 0x1p-100 : 1.0);
  const double us = tiny ? 0x1p-1000 : (huge ? 0x1p100 : 1.0);
  const double xs = x * sc; const double q0 = xs * inv;
  const double r0 = fma(-q0, b, xs); const double q1 = fma(r0, inv, q0);
  double y = q1 * us;
  if (tiny) { const double rem = fma(-q1, b, xs); const double dd = q1 - y * sc;
    if (fabs(dd) == 0x1p-75 && rem != 0.0) y = (q1 + copysign(0x1p-75, rem)) * us; }
  return (ax > 0.0 && ax <= 0x1.fffffffffffffp1023) ? y : x * inv;
}
static double div_rn_plain(double x, double b, double inv) {
  const double q0 = x * inv; const double r = fma(-q0, b, x); double q = fma(r, inv, q0);
  uint64_t u = ubits(x); unsigned e = (unsigned)((u >> 52) & 0x7ff);
  if (e - 63u > 1920u) q = wide(x, b, inv);
  return q;
}
static double div_rn(double x, double b, double inv) {  /* div_rn_z */
  const double q0 = x * inv; const double r = fma(-q0, b, x); double q = fma(r, inv, q0);
  uint64_t u = ubits(x); unsigned e = (unsigned)((u >> 52) & 0x7ff);
  if (e - 63u > 1920u && x != 0.0) q = wide(x, b, inv);
  return x == 0.0 ? x : q;
}
int main(int argc, char** argv){
  long bad=0, n=0;
  const long per = argc > 1 ? atol(argv[1]) : 40000000;
  double thetas[6]={1.0010000002, 1.001*(4.7891255047772946e-05+1.9999521087449521)*0.5, 3.7, 0.5000001, 1.2345e-3, 977.25};
  for (int t=0;t<6;t++){
    double b=thetas[t], inv=1.0/b;
    for (long i=0;i<per;i++){
      uint64_t u=rnd(); double x; int mode=i%6;
      if(mode==0) x=bits(u);
      else if(mode==1) x=bits(u & 0x800FFFFFFFFFFFFFULL);
      else if(mode==2) x=bits((u & 0x800FFFFFFFFFFFFFULL) | ((uint64_t)(1+(rnd()%70))<<52));
      else if(mode==3) x=bits((u & 0x800FFFFFFFFFFFFFULL) | ((uint64_t)(2046-(rnd()%90))<<52));
      else if(mode==4) x=bits((u & 0x800FFFFFFFFFFFFFULL) | ((uint64_t)(1980+(rnd()%6))<<52)); // around 2^960
      else x=((double)(int64_t)u)*0x1p-63;
      double a=x/b, c=div_rn(x,b,inv), c2=div_rn_plain(x,b,inv); n++;
      if (ubits(a)!=ubits(c2) && !(isnan(a)&&isnan(c2))) { if(bad<10) printf("plain x=%a b=%a ieee=%a got=%a\n",x,b,a,c2); bad++; }
      if (ubits(a)!=ubits(c) && !(isnan(a)&&isnan(c))) { if(bad<10) printf("x=%a b=%a ieee=%a got=%a\n",x,b,a,c); bad++; }
    }
  }
  printf("n=%ld bad=%ld\n",n,bad);
  return bad != 0;
}
