#!/bin/bash
# K1 grid oversubscription sweep (CHFSI_K1_OVERSUB = CTAs per resident slot)
for o in 1 2 3 4; do
  CHFSI_K1_OVERSUB=$o python tools/k1_sweep.py --no-cublas --variants 64x32,64x16 \
    --shapes 2048x37,2048x64,2048x100,2048x160,2048x200,4096x160,5000x250,8192x160 | sed "s/^/{\"os\": $o, \"r\": /; s/$/}/"
done
