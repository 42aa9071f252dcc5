#!/bin/bash
# A/B timing of C2 pass 0 (profile_update.py) for the working-tree library ("cur")
# and the variants named in VARIANTS (paper_2007_14394_b200/_variants/NAME).
VARIANTS=${VARIANTS:-head}
for i in 1 2; do
for v in $VARIANTS cur; do
  if [ $v = cur ]; then unset SDFGI_LIB; else export SDFGI_LIB=paper_2007_14394_b200/_variants/$v/libsdfgi_b200.so; fi
  echo -n "$v "; python scripts/profile_update.py f64 1 3
  echo -n "$v "; python scripts/profile_update.py f32 1 3
done; done
unset SDFGI_LIB
