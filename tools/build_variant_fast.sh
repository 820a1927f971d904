# build_variant_fast.sh <name> "<sources to recompile>" [extra nvcc flags...] -> exp/libffdp_<name>.so
# Recompiles only the named csrc files with the extra flags and links them with the
# objects of the last in-tree build (paper_2509_25044_b200/build_obj, python -m paper_2509_25044_b200.build).
set -e
name=$1; shift; files=$1; shift
cd "$(dirname "$0")/.."
mkdir -p exp/obj_$name
O=paper_2509_25044_b200/build_obj
objs=""
for o in $O/*.o; do
  b=$(basename $o .o)
  if [[ " $files " == *" $b "* ]]; then
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fvisibility=hidden "$@" \
      -c -o exp/obj_$name/$b.o paper_2509_25044_b200/csrc/$b.cu
    objs="$objs exp/obj_$name/$b.o"
  else
    objs="$objs $o"
  fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o exp/libffdp_$name.so $objs -ldl
