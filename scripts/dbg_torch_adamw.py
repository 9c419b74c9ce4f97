import sys, torch
sys.path.insert(0, '.')
from paper_2403_06504_b200 import optim as F
dev = torch.device('cuda')
n = (1 << 20) + 37
g = torch.Generator(device=dev); g.manual_seed(11)
p0 = torch.randn(n, device=dev, generator=g) * 0.02
m0 = torch.randn(n, device=dev, generator=g) * 1e-3
v0 = (torch.randn(n, device=dev, generator=g) * 1e-3) ** 2
grads = [(torch.randn(n, device=dev, generator=g) * 1e-3).to(torch.bfloat16) for _ in range(3)]
lr, b1, b2, eps, wd, t0 = 1e-4, 0.9, 0.95, 1e-8, 0.1, 10
for steps in (1, 3):
    tp = torch.nn.Parameter(p0.clone())
    opt = torch.optim.AdamW([tp], lr=lr, betas=(b1, b2), eps=eps, weight_decay=wd, fused=True)
    opt.state[tp] = {"step": torch.tensor(float(t0), device=dev), "exp_avg": m0.clone(), "exp_avg_sq": v0.clone()}
    mp, mm, mv = p0.clone(), m0.clone(), v0.clone()
    for i in range(steps):
        tp.grad = grads[i].float()
        opt.step()
        F.adamw_chunk(mp, mm, mv, grads[i].clone(), F.Hparams(lr=lr, beta1=b1, beta2=b2, eps=eps, weight_decay=wd, step=t0 + 1 + i))
    torch.cuda.synchronize()
    st = opt.state[tp]
    for ours, theirs, name in ((mp, tp.detach(), "p"), (mm, st["exp_avg"], "m"), (mv, st["exp_avg_sq"], "v")):
        d = (ours - theirs).abs(); r = d / (theirs.abs() + 1e-30)
        i = int(r.argmax())
        print(steps, name, "max rel", float(r.max()), "at", i, "ours", float(ours[i]), "theirs", float(theirs[i]), "p0", float(p0[i]), "m", float(mm[i]), "v", float(mv[i]), "absmax", float(d.max()), "n>1e-6rel", int((r > 1e-6).sum()))
