#!/bin/bash
# on the GPU box: make variant $1 (tools/build_variant.py) the loaded libfrwgpu.so
# ("default" restores the default build, kept as lib/variants/default)
L=paper_2507_09730_b200/lib
[ -f $L/variants/default/libfrwgpu.so ] || { mkdir -p $L/variants/default; cp $L/libfrwgpu.so $L/variants/default/; }
cp $L/variants/$1/libfrwgpu.so $L/libfrwgpu.so
