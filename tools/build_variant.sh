#!/bin/bash
# Build an A/B variant of libsynperf.so into variants/lib_<name>.so.
#   tools/build_variant.sh <name> [<git-rev>:<csrc file> ...] [-- extra nvcc flags]
# Each <git-rev>:<file> replaces that csrc file with its content at <git-rev>.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
name=$1; shift
tmp=$(mktemp -d)
cp -r "$ROOT/paper_2601_14910_b200/csrc" "$tmp/csrc"
extra=()
while [ $# -gt 0 ]; do
  if [ "$1" = "--" ]; then shift; extra=("$@"); break; fi
  rev=${1%%:*}; f=${1#*:}
  git -C "$ROOT" show "$rev:paper_2601_14910_b200/csrc/$f" > "$tmp/csrc/$f"
  shift
done
mkdir -p "$ROOT/variants"
nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC,-O2 \
  --expt-relaxed-constexpr -shared -I"$ROOT/include" "${extra[@]}" -o "$ROOT/variants/lib_$name.so" "$tmp"/csrc/*.cu
rm -rf "$tmp"
echo "$ROOT/variants/lib_$name.so"
