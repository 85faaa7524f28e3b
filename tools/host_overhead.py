"""Host-side cost of one sparse_attention fwd+bwd call (tiny problem, so the GPU work is
negligible): the floor of the host-buffer pipeline's per-group time.  Optional cProfile."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_13515_b200 as spa  # noqa: E402
from paper_2602_13515_b200.synthetic import wan_like_qkv  # noqa: E402

q, k, v = wan_like_qkv(1, 2, 2048, 128, 0.9, seed=1)
do = torch.randn_like(q)
cfg = spa.SparsityConfig(0.03, 0.2, 128, 64)


def step():
    qs, ks, vs = (t.detach().requires_grad_(True) for t in (q, k, v))
    res = spa.sparse_attention(qs, ks, vs, cfg)
    res.out.backward(do)


for _ in range(5):
    step()
torch.cuda.synchronize()
n = 100
t0 = time.perf_counter()
for _ in range(n):
    step()
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host issue {1e3 * (t1 - t0) / n:.3f} ms/call, wall incl. drain {1e3 * (t2 - t0) / n:.3f} ms/call")
if len(sys.argv) > 1:
    import cProfile, pstats
    cProfile.run("for _ in range(50): step()", "/tmp/hp.prof")
    pstats.Stats("/tmp/hp.prof").sort_stats("cumulative").print_stats(25)
