#!/bin/bash
# usage: tools/build_variant.sh NAME [--full] -DFOO=1 ...  -> paper_1612_00595_b200/_lib/variants/NAME.so
# (development build: the fp32 row-only production kernels only, unless --full; load it with
#  SEIS_LIB=...; the .so travels to the GPU box, tools/ab2.sh compares builds)
name=$1; shift
fast=--fast
if [ "$1" = "--full" ]; then fast=; shift; fi
cd "$(dirname "$0")/.."
python -m paper_1612_00595_b200.build $fast "$@" --out paper_1612_00595_b200/_lib/variants/$name.so
