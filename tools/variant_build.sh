#!/bin/bash
# Build an experiment variant of libpolar.so with its own code list and nvcc flags:
#   tools/variant_build.sh <name> <codes file> [extra nvcc flags...]
# -> variants/<name>/libpolar.so ; select it at run time with POLAR_LIB=variants/<name>/libpolar.so
NAME=$1; CODES=$(realpath $2); shift 2
mkdir -p variants/$NAME
POLAR_BUILD_DIR=$PWD/variants/$NAME/build POLAR_LIB_OUT=$PWD/variants/$NAME/libpolar.so POLAR_CODES=$CODES \
POLAR_NVCC_EXTRA="$*" python -c "from paper_1504_00353_b200.build import build; build(verbose=False)"
# the library travels to the GPU box from vlibs/ (variants/ holds the build trees and is gpurun-ignored)
mkdir -p vlibs && cp variants/$NAME/libpolar.so vlibs/$NAME.so
