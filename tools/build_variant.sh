# build_variant.sh <name> [extra nvcc flags...] -> exp/libffdp_<name>.so (A/B experiments via FFDP_LIB)
# SRC=<repo root> builds another checkout's sources (e.g. a git worktree of an older commit).
set -e
name=$1; shift
cd "$(dirname "$0")/.."
mkdir -p exp
S=${SRC:-.}
C=$S/paper_2509_25044_b200/csrc
srcs=$(python -c "import sys; sys.path.insert(0,'$S'); from paper_2509_25044_b200 import build as b; print(' '.join('$C/'+x for x in b.SOURCES))")
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fvisibility=hidden -shared \
  -I$S/include "$@" -o exp/libffdp_$name.so $srcs
