#!/bin/bash
# Build the library from a git rev (or WT = working tree) with extra nvcc flags into ab/<name>.so
# usage: bash tools/build_variant.sh name rev [EXTRA flags]
set -e
NAME=$1; REV=$2; shift 2
D=$(mktemp -d)
if [ "$REV" == "WT" ]; then cp -r paper_2502_00356_b200 include $D/; else git archive $REV paper_2502_00356_b200 include | tar -x -C $D; fi
make -s -C $D/paper_2502_00356_b200 -B EXTRA="$*" > /dev/null
mkdir -p ab && cp $D/paper_2502_00356_b200/libbesselgp_sm100a.so ab/$NAME.so
rm -rf $D
echo "built ab/$NAME.so"
