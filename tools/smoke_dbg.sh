for e in "X=1" "HEB_MODUP_CONCURRENT=0" "HEB_MODUP_SPLIT=1"; do
  env $e CUDA_LAUNCH_BLOCKING=1 timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1 | cut -c1-200 | sed "s/^/$e: /"
done
for m in 512 1024 2048 4096; do
  CUDA_LAUNCH_BLOCKING=1 timeout 120 python - $m <<'PY' 2>&1 | tail -1 | cut -c1-200
import sys, numpy as np
sys.path.insert(0, ".")
from paper_2102_00319_b200.backend import B200Backend
from paper_2102_00319_b200.params import derive_params
m = int(sys.argv[1])
be = B200Backend(derive_params(m, 300, 35, seed=7))
k = be.keygen(); be.set_eval_key(k)
x = be.encrypt(np.zeros(be.slots), k, entropy=1)
print(m, be.chain.primes.bit_length() if hasattr(be.chain.primes,'bit_length') else [int(p).bit_length() for p in be.chain.primes])
be.mul_ct_ct(x, x); import torch; torch.cuda.synchronize(); print(m, "ok")
PY
done
