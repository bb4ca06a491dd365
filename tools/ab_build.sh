#!/bin/bash
# Builds A/B variants of the library with sum-factorisation launch overrides.
# usage: tools/ab_build.sh name1 "PI_SF_4_1 true,1,5,..." name2 "..." ...
# -> paper_1310_1191_b200/libprism_b200_ab_<name>.so (run with PRISM_B200_LIB=libprism_b200_ab_<name>.so)
cd "$(dirname "$0")/../paper_1310_1191_b200"
mkdir -p ab
while [ $# -ge 2 ]; do
  name=$1; def=$2; shift 2
  echo "#define $def" > ab/$name.h
  ( make -s LIB=libprism_b200_ab_$name.so OBJ=build_ab_$name NVEXTRA="-DPI_SF_OVERRIDE=\\\"$PWD/ab/$name.h\\\"" > /tmp/ab_$name.log 2>&1 \
      && echo "built $name" || { echo "FAILED $name"; tail -5 /tmp/ab_$name.log; } ) &
done
wait
