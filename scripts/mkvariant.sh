#!/bin/bash
# Build the library of git revision REV (default HEAD) into paper_2007_14394_b200/_variants/NAME
# for A/B timing against the working tree (SDFGI_LIB=.../_variants/NAME/libsdfgi_b200.so).
set -e
cd "$(dirname "$0")/.."
NAME=${1:-head}; REV=${2:-HEAD}
WT=/tmp/sdfgi_wt_$NAME
rm -rf $WT; git worktree prune; git worktree add -f $WT $REV >/dev/null 2>&1
(cd $WT && bash scripts/build_variants.sh $NAME "" >/dev/null)
mkdir -p paper_2007_14394_b200/_variants/$NAME
cp $WT/paper_2007_14394_b200/_variants/$NAME/libsdfgi_b200.so paper_2007_14394_b200/_variants/$NAME/
git worktree remove --force $WT
echo built _variants/$NAME from $(git rev-parse --short $REV)
