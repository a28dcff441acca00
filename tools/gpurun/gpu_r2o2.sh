# round-2 call O2: fwd gather with whole-row tiles + 3 row buffers (CCT_TUNE_GATHER = 3) vs default
O=gpurun_out/r2o2; mkdir -p $O
timeout 300 python - > $O/parity.log 2>&1 <<'PY'
import sys, torch
sys.path.insert(0, '.')
import paper_1504_04343_b200 as cct
from paper_1504_04343_b200 import conv
dev = torch.device('cuda')
for (n, k, d, o, b, s, p) in [(227, 11, 3, 96, 8, 4, 0), (224, 11, 3, 64, 3, 4, 2), (63, 11, 3, 96, 2, 4, 5)]:
    desc = cct.ConvDesc(n, k, d, o, b, s, p, cct.NHWC)
    g = torch.Generator(device=dev).manual_seed(n)
    x = torch.rand((b, n, n, d), generator=g, device=dev) * 2 - 1
    w = torch.rand((o, k, k, d), generator=g, device=dev) * 2 - 1
    y1 = conv.conv_fwd(x, w, desc, 1)
    with cct.tuning(gather=3):
        y3 = conv.conv_fwd(x, w, desc, 1)
    print(n, k, d, o, 'bitwise equal' if torch.equal(y1, y3) else f'DIFF {float((y1-y3).abs().max())}', flush=True)
PY
echo "parity rc $?" >> $O/parity.log
for i in 1 2; do for t in "gather=1" "gather=3"; do
  timeout 120 python tools/pass_time.py --layer conv1 --pass fwd --layout 1 --reps 20 --tune $t >> $O/time.log 2>&1
done; done
for i in 1 2; do for t in "gather=1" "gather=3"; do
  timeout 300 python bench.py --no-cpu --no-e2e --no-configs --steps 20 --tune $t >> $O/bench.jsonl 2>> $O/bench.err
done; done
