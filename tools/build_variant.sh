# build_variant.sh <name> [extra nvcc flags...] -> exp/libffdp_<name>.so (A/B experiments via FFDP_LIB)
set -e
name=$1; shift
cd "$(dirname "$0")/.."
mkdir -p exp
C=paper_2509_25044_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fvisibility=hidden -shared \
  -Iinclude "$@" -o exp/libffdp_$name.so $C/capi.cu $C/sampler.cu $C/lncc.cu $C/mi.cu $C/step_lncc.cu $C/step_lncc2.cu $C/step_mi.cu
