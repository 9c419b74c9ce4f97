"""Where does the C1 step (12 x 7.08M params, 2.38 GB) lose to the HBM peak?
Arms, interleaved, 20 back-to-back steps each: the 12-chunk list launch, the
same bytes as ONE 85M-element chunk (no list overhead), that chunk without
the grad-norm pass, and the list launch replayed from a CUDA graph."""
import json
import statistics
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2403_06504_b200 import optim as F  # noqa: E402

dev = torch.device("cuda")
ws = torch.zeros(F.workspace_floats(), device=dev)
sq = torch.zeros(1, dtype=torch.float64, device=dev)
hp = F.Hparams()
L, n = 12, 12 * 768 * 768
st = [torch.rand(3 * n, device=dev) * 1e-3 for _ in range(L)]
g = [(torch.randn(n, device=dev) * 1e-3).to(torch.bfloat16) for _ in range(L)]
chunks = [(s[:n], s[n:2 * n], s[2 * n:], gg, gg) for s, gg in zip(st, g)]
N = L * n
big = torch.rand(3 * N, device=dev) * 1e-3
bg = (torch.randn(N, device=dev) * 1e-3).to(torch.bfloat16)


def multi():
    F.adamw_chunks(chunks, hp, grad_sq_sum=sq, workspace=ws)


from paper_2403_06504_b200._lib import LIB, check  # noqa: E402


def multi_148():  # the list launch capped at one CTA per SM (SM budget = 148)
    check(LIB.fy_adamw_sm_budget(148))
    F.adamw_chunks(chunks, hp, grad_sq_sum=sq, workspace=ws)
    check(LIB.fy_adamw_sm_budget(0))


def one_chunk():
    F.adamw_chunk(big[:N], big[N:2 * N], big[2 * N:], bg, hp, param_out=bg, grad_sq_sum=sq, workspace=ws)


def one_chunk_nostats():
    F.adamw_chunk(big[:N], big[N:2 * N], big[2 * N:], bg, hp, param_out=bg)


if len(sys.argv) > 1 and sys.argv[1] == "ncu":  # ncu target: list launch, then the single chunk
    multi()
    one_chunk()
    torch.cuda.synchronize()
    sys.exit(0)
s = torch.cuda.Stream()
graph = torch.cuda.CUDAGraph()
multi()
torch.cuda.synchronize()
with torch.cuda.graph(graph, stream=s):
    multi()
arms = {"multi_list": multi, "multi_list_148": multi_148, "one_chunk": one_chunk, "one_chunk_nostats": one_chunk_nostats,
        "multi_list_graph": graph.replay}
res = {k: [] for k in arms}
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for fn in arms.values():
    fn()
for _ in range(10):
    for k, fn in arms.items():
        torch.cuda.synchronize()
        a.record()
        for _ in range(20):
            fn()
        b.record()
        torch.cuda.synchronize()
        res[k].append(a.elapsed_time(b) / 20)
for k, v in res.items():
    ms = statistics.median(v)
    print(json.dumps({"arm": k, "ms": round(ms, 4), "gbs_at_28B": round(28 * N / ms / 1e6, 1)}))
