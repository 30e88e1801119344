# round-2 batch av: pair_candidates without local-memory candidate lists
set -x
timeout 900 python -m pytest tests/test_gpu.py -m gpu -q -x -k "pair or qrange or fused or golden" 2>&1 | tail -3 > gpurun_out/gpu_tests_av.log
cat > /tmp/pcmp.py <<'PY'
import os, sys, torch, ctypes as C
sys.path.insert(0, os.getcwd())
import paper_2602_01077_b200 as P
H, L, d = 8, 75600, 128
for kind in ("gaussian", "clustered"):
    gen = P.gen_clustered if kind == "clustered" else P.gen_gaussian
    q, k, v = (x.reshape(1, H, L, d).cuda() for x in gen(0, H, L, d))
    o = P.fwd(q, k, v, sparsity=0.875)
    torch.cuda.synchronize()
    torch.save(o.cpu(), f"/tmp/o_{kind}_{os.environ.get('TAG','x')}.pt")
PY
L=$PWD/paper_2602_01077_b200/lib
TAG=old PISA_B200_LIB=$L/libpisa_b200_pairold.so python /tmp/pcmp.py
TAG=new python /tmp/pcmp.py
python -c "
import torch
for k in ('gaussian','clustered'):
    a=torch.load(f'/tmp/o_{k}_old.pt'); b=torch.load(f'/tmp/o_{k}_new.pt'); print(k, 'bit-identical', torch.equal(a,b))
" >> gpurun_out/gpu_tests_av.log 2>&1
timeout 900 bash tools/ab_lib.sh $L/libpisa_b200_pairold.so $L/libpisa_b200.so gaussian clustered > gpurun_out/ab_pair_av.log 2>&1
