#!/bin/bash
# Build paper_2101_10994_b200/variants/libnglod_<name>.so from the same
# sources with extra nvcc flags (compile-time knobs such as -DNG_TT_RAYS=64);
# select it at run time with NG_LIB_VARIANT=<name>.
#   tools/build_variant.sh NAME "-DKNOB=VALUE ..."
set -e
name=$1; extra=$2
root=$(cd "$(dirname "$0")/.." && pwd)
csrc=$root/paper_2101_10994_b200/csrc
out=$root/paper_2101_10994_b200/variants
tmp=$root/.vb/$name  # depth 2 below the root: the sources include ../../include
rm -rf "$tmp"; mkdir -p "$tmp"
mkdir -p "$out"
cp "$csrc"/*.cu "$csrc"/*.cuh "$csrc"/Makefile "$tmp"/
sed -i "s#^OUT := .*#OUT := $out/libnglod_$name.so#" "$tmp/Makefile"
make -s -C "$tmp" -j8 EXTRA="$extra" > /dev/null
grep -h -A3 "k_traverse_tiles" "$tmp"/traverse.o.ptxas.log | grep -E "Used|spill" | head -2
rm -rf "$tmp"
