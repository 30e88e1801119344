# round-2 batch aa: exp2 split across MUFU / FMA (FA4) on the single-pass softmax
L=$PWD/paper_2602_01077_b200/lib
for v in p01 p11 pb11; do
timeout 900 bash tools/ab_lib.sh $L/libpisa_b200.so $L/libpisa_b200_$v.so gaussian clustered >> gpurun_out/ab_k3_aa.log 2>&1
done
