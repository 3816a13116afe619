/* Exhaustive check of the division-by-3 used by exact_score (eca_strip.cuh:
   div3): for every RGB sum 0..765, q1 = fma(fma(-q0, 3, x), 1/3, q0) with
   q0 = x * RN(1/3) equals the correctly rounded x / 3.0 bit for bit.
   gcc -O2 -ffp-contract=off tools/div3_check.c -lm && ./a.out  (prints bad=0) */
#include <stdio.h>
#include <math.h>
int main(){
  const double c = 1.0/3.0;
  int bad=0;
  for (int x=0;x<=765;++x){
    double xd=x, q=x/3.0;
    double q0 = xd*c;
    double r = fma(-q0, 3.0, xd);
    double q1 = fma(r, c, q0);
    if (q1!=q) {bad++; if(bad<5) printf("x=%d q=%.17g q1=%.17g\n",x,q,q1);}
  }
  // also 2*x/3 style values? pre_sum/3 uses same ints (0..765)
  printf("bad=%d\n",bad);
}
