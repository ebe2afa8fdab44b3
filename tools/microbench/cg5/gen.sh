#!/bin/bash
# builds proto_codegen5 variants: name R W KC S PF opt
cd "$(dirname "$0")"
while read name R W KC S PF opt; do
  python ../../proto_codegen5.py $R 4096 $W $KC $S $PF $name.ptx 0.1 > $name.info
  ptxas -arch=sm_100a -$opt $name.ptx -o $name.cubin -v 2> $name.ptxas
  rm -f $name.ptx
done
