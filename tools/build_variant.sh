#!/bin/bash
# build libpdssm.so tuning variants with extra -D defines into paper_2605_19150_b200/variants/NAME.so
# (selected at import with PDSSM_LIB_VARIANT=NAME); usage: bash tools/build_variant.sh NAME "DEFINES" [NAME "DEFINES" ...]
cd "$(dirname "$0")/.."
while [ $# -ge 2 ]; do python paper_2605_19150_b200/_build.py --variant "$1" $2; shift 2; done
