#!/bin/bash
# A/B of the C2 step for the variants in VARIANTS (paper_2007_14394_b200/_variants/NAME) and the working tree.
for i in 1 2; do
for v in ${VARIANTS:-} cur; do
  if [ $v = cur ]; then unset SDFGI_LIB; else export SDFGI_LIB=paper_2007_14394_b200/_variants/$v/libsdfgi_b200.so; fi
  python scripts/ab_step.py ${PREC:-f64} 5
  if [ $v = cur ] && [ -n "$FUSED_TOO" ]; then FUSED=1 python scripts/ab_step.py ${PREC:-f64} 5; fi
  if [ $v = cur ] && [ -n "$ASYNC_TOO" ]; then ASYNC=1 python scripts/ab_step.py ${PREC:-f64} 5; fi
done; done
