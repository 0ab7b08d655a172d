// Worst fp32 error of the rotated Chebyshev phasor chain (j <= 32) when a photon may run in
// frame A only if |sin theta| >= tau and in frame B (theta + pi/2) only if |cos theta| >= tau
// (the class-routed sketch, csrc/sketch_routed.cu), for every x < T at the tested T; plus the
// fraction of bins forced into each frame.  gcc -O2 tools/sim_cheb_tau.c -lm && ./a.out
#include <stdio.h>
#include <math.h>
// worst fp32 Chebyshev phasor error over x<T, j<=32, when a photon may run in frame A (theta)
// iff |cos| >= tau fails... frame A allowed iff |sin theta| >= tau; frame B (theta+pi/2) allowed iff |cos theta| >= tau
static double chain_err(int x, int T, int rot){
  int rc=(2*x>T)?x-T:x; double sn=sin(M_PI*2.0*rc/T), cs=cos(M_PI*2.0*rc/T);
  float c=(float)cs, s=(float)sn;
  float c1=rot? -s: c, s1=rot? c: s; float C=2.0f*c1;
  float pc=1.0f,ps=0.0f,qc=c1,qs=s1; double w=0;
  for(int j=1;j<=32;j++){ float vc,vs; if(j==1){vc=qc;vs=qs;} else {vc=fmaf(C,qc,-pc); vs=fmaf(C,qs,-ps); pc=qc;ps=qs;qc=vc;qs=vs;}
    float oc=vc,os=vs; if(rot){int jm=j&3; if(jm==1){oc=vs;os=-vc;} else if(jm==2){oc=-vc;os=-vs;} else if(jm==3){oc=-vs;os=vc;}}
    long long r=((long long)j*x)%T; int rr=(2*r>T)?(int)r-T:(int)r; double ec=cos(2*M_PI*rr/T), es=sin(2*M_PI*rr/T);
    double e=fmax(fabs(oc-ec),fabs(os-es)); if(e>w) w=e; }
  return w;
}
int main(){ int Ts[]={1024,2500,4096,4613,8192,23800,65535}; double taus[]={0.15,0.2,0.25,0.3,0.383,0.5};
  for(int ti=0;ti<6;ti++){ double tau=taus[ti]; double worst=0; double fa=0,fb=0;
    for(int k=0;k<7;k++){int T=Ts[k]; for(int x=0;x<T;x++){ int rc=(2*x>T)?x-T:x; double sn=sin(M_PI*2.0*rc/T), cs=cos(M_PI*2.0*rc/T);
      float c=(float)cs,s=(float)sn; int okA = fabsf(s)>=tau, okB=fabsf(c)>=tau;
      if(okA){double e=chain_err(x,T,0); if(e>worst) worst=e;}
      if(okB){double e=chain_err(x,T,1); if(e>worst) worst=e;}
      if(T==8192){ if(!okB) fa++; if(!okA) fb++; }
    }}
    printf("tau=%.3f worst err j<=32: %.2e   A-only frac %.3f B-only frac %.3f\n",tau,worst,fa/8192,fb/8192);
  }
}
