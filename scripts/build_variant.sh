#!/bin/bash
# build_variant.sh NAME "-DFLAG=1 ..." : an experiment build of libfvv.so in _variants/NAME
set -e
cd "$(dirname "$0")/../paper_1903_11785_b200/csrc"
make -s -j8 BUILD=../../_variants/$1/_build LIB=../../_variants/$1/libfvv.so EXTRA="$2"
