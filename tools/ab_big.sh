#!/bin/bash
for v in $1; do tools/use_variant.sh $v; echo "== $v"; python tools/big_walks.py 2>&1 | grep walks=; done
tools/use_variant.sh default
