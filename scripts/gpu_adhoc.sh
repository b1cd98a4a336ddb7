timeout 300 python -m pytest tests/test_gpu_umma.py -x -q 2>&1 | tail -30 > gpurun_out/umma_s37.log
timeout 120 python - >> gpurun_out/umma_s37.log 2>&1 <<'PY'
import torch
from paper_2511_20048_b200 import spa
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn((128, 128), generator=g, device="cuda").to(torch.bfloat16)
k = torch.randn((32, 128), generator=g, device="cuda").to(torch.bfloat16)
v = torch.randn((32, 128), generator=g, device="cuda").to(torch.bfloat16)
s, o = spa.umma_selftest(q, k, v)
torch.cuda.synchronize()
s_ref = (q.double() @ k.double().T)
print("S err", (s.double() - s_ref).abs().max().item())
print("S[0,:4]", s[0, :4].tolist(), "ref", s_ref[0, :4].tolist())
print("S[1,:4]", s[1, :4].tolist(), "ref", s_ref[1, :4].tolist())
print("S[0,16:20]", s[0, 16:20].tolist(), "ref", s_ref[0, 16:20].tolist())
# find permutation of columns / rows
for name, ref in [("S", s_ref)]:
    import itertools
    sd = s.double()
    best = [(ref[:, j] - sd[:, 0]).abs().max().item() for j in range(32)]
    print("col0 best match", min(range(32), key=lambda j: best[j]), min(best))
    bestr = [(ref[i, :] - sd[0, :]).abs().max().item() for i in range(128)]
    print("row0 best match", min(range(128), key=lambda i: bestr[i]), min(bestr))
o_ref = s.to(torch.bfloat16).double() @ v.double()
print("O err", (o.double() - o_ref).abs().max().item(), "scale", o_ref.abs().max().item())
print("O[0,:4]", o[0, :4].tolist(), "ref", o_ref[0, :4].tolist())
PY
