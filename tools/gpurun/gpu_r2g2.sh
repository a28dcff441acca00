# round-2 call G2: merged N = 2 BN narrow tiles (CCT_TUNE_A_TMEM = 3) -- parity, then conv2 backward-data forms
O=gpurun_out/r2g2; mkdir -p $O
timeout 300 python - > $O/mg_parity.log 2>&1 <<'PY'
import sys, torch
sys.path.insert(0, '.')
import paper_1504_04343_b200 as cct
from paper_1504_04343_b200 import conv
dev = torch.device('cuda')
for (n, k, d, o, b, s, p) in [(27, 5, 96, 256, 8, 1, 2), (13, 3, 64, 96, 4, 1, 1), (9, 3, 32, 64, 2, 1, 1)]:
    desc = cct.ConvDesc(n, k, d, o, b, s, p, cct.NHWC)
    g = torch.Generator(device=dev).manual_seed(n + d)
    x = torch.rand((b, n, n, d), generator=g, device=dev) * 2 - 1
    w = torch.rand((o, k, k, d), generator=g, device=dev) * 2 - 1
    dy = torch.rand((b, desc.m, desc.m, o), generator=g, device=dev) * 2 - 1
    xr = x.double().permute(0, 3, 1, 2).requires_grad_(True)
    wr = w.double().permute(0, 3, 1, 2)
    yr = torch.nn.functional.conv2d(xr, wr, padding=p)
    yr.backward(dy.double().permute(0, 3, 1, 2))
    ref = xr.grad.permute(0, 2, 3, 1)
    for tune in ({}, {'dgrad_swap': 0}, {'dgrad_swap': 0, 'a_tmem': 3}, {'dgrad_swap': 0, 'a_tmem': 3, 'cta_pairs': 1}):
        with cct.tuning(implicit_bwd=2, **tune):
            dx = conv.conv_bwd_data(dy, w, desc, 1)
        e = float((dx.double() - ref).norm() / ref.norm())
        print(n, k, d, o, tune, f'{e:.2e}', 'OK' if e <= 1e-4 else 'FAIL', flush=True)
PY
echo "parity rc $?" >> $O/mg_parity.log
for t in "" "dgrad_swap=0" "dgrad_swap=0,a_tmem=3" "dgrad_swap=0,a_tmem=3,cta_pairs=1" "dgrad_swap=0,cta_pairs=1"; do
  echo "tune=$t" >> $O/time.log
  timeout 120 python tools/pass_time.py --layer conv2 --pass dgrad --layout 1 --reps 20 --tune "$t" >> $O/time.log 2>&1
done
