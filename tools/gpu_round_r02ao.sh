# round-2 batch ao: hardware-suspended waits (try_wait with a time-limit hint) for the MMA warp / the softmax warps
L=$PWD/paper_2602_01077_b200/lib
for v in mwsus smsus bothsus; do
timeout 1200 bash tools/ab_lib.sh $L/libpisa_b200.so $L/libpisa_b200_$v.so clustered gaussian >> gpurun_out/ab_k3_ao.log 2>&1
done
