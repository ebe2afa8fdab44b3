#!/bin/bash
# builds proto_codegen6 variants: name R W KC S PF opt rotate
cd "$(dirname "$0")"
while read name R W KC S PF opt rot; do
  python ../../proto_codegen6.py $R 4096 $W $KC $S $PF $name.ptx 0.1 $rot > $name.info
  ptxas -arch=sm_100a -$opt $name.ptx -o $name.cubin -v 2> $name.ptxas
  rm -f $name.ptx
done
