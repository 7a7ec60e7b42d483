#!/bin/bash
O=gpurun_out/${OUTD:-sweep_build}; mkdir -p $O
for c in ${CONFIGS:-mag:0 imdb:1 freebase:1 dblp:1}; do
  timeout 600 python scripts/sweep_build.py $c >> $O/sweep.txt 2>&1; echo "rc=$? $c" >> $O/sweep.txt
done
