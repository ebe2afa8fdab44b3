# proto_codegen5 sweep (one panel, N = 262144, uniform 10 % density, K = 4096)
cd tools/microbench/cg5
while read name R W KC S PF opt; do
  nnz=$(awk '{print $2}' $name.info); smem=$(awk '{print $6}' $name.info)
  echo "== $name R=$R W=$W KC=$KC S=$S PF=$PF $opt $(grep -o 'Used [0-9]* registers' $name.ptxas)"
  timeout 60 ./run_cg5 $name.cubin $nnz 262144 $W $KC $S $R
done < ${1:-variants.txt}
