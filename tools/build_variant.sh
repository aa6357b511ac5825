#!/bin/bash
# profiling tool: build_variant.sh NAME "-DFOO=1 ..." -> build_variants/NAME.so from the current csrc
set -e
name=$1; shift
rm -rf /tmp/vb_$name && mkdir -p /tmp/vb_$name/p /tmp/vb_$name/include /root/repo/build_variants
cp /root/repo/include/rinshan.h /tmp/vb_$name/include/
cp -r /root/repo/paper_2605_20577_b200/csrc /tmp/vb_$name/p/csrc
cd /tmp/vb_$name/p/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr "$@" -shared -o /root/repo/build_variants/$name.so rs_abi.cu rs_tables.cpp 2> ptxas.log || (grep -i error ptxas.log; exit 1)
grep -A2 "Function properties.*k_rollout" ptxas.log | tail -2 | sed "s/^/$name: /"
