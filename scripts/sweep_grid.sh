#!/bin/bash
# C2 pass 0 (profile_update.py) over candidate-grid sizes and margins.
CELLS=${CELLS:-"16777216 33554432"}; MARGINS=${MARGINS:-"0.6 1.0"}
for cells in $CELLS; do
  for m in $MARGINS; do
    for prec in f64 f32; do
      echo -n "cells=$cells margin=$m "; SDFGI_GRID_CELLS=$cells SDFGI_GRID_MARGIN=$m python scripts/profile_update.py $prec 1 3
    done
  done
done
