#!/bin/bash
# SASS evidence that the contractions run on tcgen05 / TMEM / TMA (no GPU needed): per kernel of
# libsvgear.so, the count of UTCHMMA (tcgen05.mma), LDTM/STTM (tcgen05.ld/st), UTMALDG (TMA tensor
# loads), LDGSTS (cp.async) and HMMA (mma.sync — expected 0) instructions.
LIB=${1:-paper_2603_08982_b200/libsvgear.so}
cuobjdump -sass $LIB | awk '
  /Function :/ { name=$3 }
  /UTCHMMA/ { mma[name]++ } /LDTM|STTM/ { tm[name]++ } /UTMALDG/ { tma[name]++ } /LDGSTS/ { cpa[name]++ } /[ \t]HMMA/ { hm[name]++ }
  END { printf "%-100s %8s %9s %8s %7s %5s\n", "kernel (mangled)", "UTCHMMA", "LDTM/STTM", "UTMALDG", "LDGSTS", "HMMA";
        for (n in mma) printf "%-100s %8d %9d %8d %7d %5d\n", substr(n,1,100), mma[n], tm[n], tma[n], cpa[n], hm[n] }' | sort
