#include <stdio.h>
#include <math.h>
#include <stdlib.h>
// Emulate rotated Chebyshev phasor recurrence in fp32 (fmaf) for every x<T.
int main(int argc,char**argv){
  int Ts[]={1024,4613,2500,4096,8192,65536,65535,17,40000,3};
  for(int ti=0;ti<10;ti++){int T=Ts[ti]; int M=64; double worst[65]={0}; int wx=0;
    for(int x=0;x<T;x++){
      int rc = (2*x>T)? x-T : x; double sn,cs; sn=sin(M_PI*2.0*rc/T); cs=cos(M_PI*2.0*rc/T);
      float c=(float)cs, s=(float)sn; int k = fabsf(s) < fabsf(c);
      float c1 = k? -s : c, s1 = k? c : s; float C = 2.0f*c1;
      float pc=1.0f, ps=0.0f, qc=c1, qs=s1; // v_{j-1}=q, v_{j-2}=p
      for(int j=1;j<=M;j++){
        float vc,vs;
        if(j==1){vc=qc;vs=qs;} else { vc=fmaf(C,qc,-pc); vs=fmaf(C,qs,-ps); pc=qc;ps=qs;qc=vc;qs=vs; }
        // rotate (-i)^j if k
        float oc=vc, os=vs;
        if(k){ int jm=j&3; if(jm==1){oc=vs;os=-vc;} else if(jm==2){oc=-vc;os=-vs;} else if(jm==3){oc=-vs;os=vc;} }
        long long r=((long long)j*x)%T; int rr=(2*r>T)? (int)r-T:(int)r; double ec=cos(2*M_PI*rr/T), es=sin(2*M_PI*rr/T);
        double e=fmax(fabs(oc-ec),fabs(os-es)); if(e>worst[j]){worst[j]=e; if(j==32) wx=x;}
      }
    }
    double w32=0,w64=0; for(int j=1;j<=32;j++) w32=fmax(w32,worst[j]); for(int j=1;j<=64;j++) w64=fmax(w64,worst[j]);
    printf("T=%d worst j<=8 %.2e j<=16 %.2e j<=32 %.2e (x=%d) j<=64 %.2e\n",T,worst[8],worst[16],w32,wx,w64);
  }
}
