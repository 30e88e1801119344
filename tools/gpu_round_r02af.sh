# round-2 batch af: MMA warp waits with a nanosleep backoff (frees issue slots on its sub-partition)
L=$PWD/paper_2602_01077_b200/lib
for v in mw16 mw64; do
timeout 1200 bash tools/ab_lib.sh $L/libpisa_b200.so $L/libpisa_b200_$v.so gaussian clustered >> gpurun_out/ab_k3_af.log 2>&1
done
