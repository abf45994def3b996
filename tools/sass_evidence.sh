#!/bin/bash
# Per-kernel counts of the SASS instructions that prove tcgen05 / TMEM / TMA use (B200_PROFILING.md).
LIB=${1:-paper_2602_03921_b200/lib/libspecmd_b200.so}
echo "cuobjdump -sass $LIB: per kernel, count of UTC*MMA (tcgen05.mma), LDTM (tcgen05.ld), UTMALDG/UTMASTG (TMA), UBLKCP (bulk copy), SYNCS (mbarrier), REDG (global reductions), FFMA2 (packed fp32 FMA, the decode GEMV)"
cuobjdump -sass "$LIB" | awk '
  /Function :/ { if (name != "") printf "%-64s UTCMMA %3d  LDTM %3d  UTMALDG %3d  UTMASTG %2d  UBLKCP %2d  SYNCS %3d  REDG %3d  FFMA2 %3d\n", substr(name,1,64), mma, ldtm, ldg, stg, blk, syncs, red, f2;
                 name = $3; mma = ldtm = ldg = stg = blk = syncs = red = f2 = 0 }
  /UTC[A-Z]*MMA/ { mma++ } /LDTM/ { ldtm++ } /UTMALDG/ { ldg++ } /UTMASTG/ { stg++ } /UBLKCP/ { blk++ } /SYNCS\./ { syncs++ } /REDG/ { red++ } /FFMA2/ { f2++ }
  END { printf "%-64s UTCMMA %3d  LDTM %3d  UTMALDG %3d  UTMASTG %2d  UBLKCP %2d  SYNCS %3d  REDG %3d  FFMA2 %3d\n", substr(name,1,64), mma, ldtm, ldg, stg, blk, syncs, red, f2 }' \
  | grep -E "ffn|gemm" 
