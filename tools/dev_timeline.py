"""Dev: per-CTA timeline of MMA warp 0 (timeline build libftblas_tl.so, FTBLAS_DEV_PROF slots 10..11 of each CTA):
waiting for the tile's first stage, its k-loop, its epilogue (check + store), averaged over the
CTAs.
usage: python tools/dev_timeline.py M N K [noft] [TRANS]"""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
M, N, K = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
noft = len(sys.argv) > 4 and sys.argv[4] == "noft"
tr = sys.argv[5] if len(sys.argv) > 5 else "NN"
ntiles = ((M + 126) // 127) * ((N + 126) // 127) + 1
prof = torch.zeros(ntiles * 12 * 2, dtype=torch.int64, device="cuda")
os.environ["FTBLAS_DEV_PROF"] = str(prof.data_ptr())
from paper_2104_00897_b200 import build as _build, ftblas as F
F.load(_build.build(timeline=True))  # timeline build: libftblas_tl.so (-DFTBLAS_DEV_TIMELINE)
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.rand(M * K, dtype=torch.float64, device="cuda", generator=g)
B = torch.rand(K * N, dtype=torch.float64, device="cuda", generator=g)
C = torch.zeros(M * N, dtype=torch.float64, device="cuda")
lda = M if tr[0] == "N" else K
ldb = K if tr[1] == "N" else N
def call():
    if noft:
        F.ftblas_dgemm_noft(tr[0], tr[1], M, N, K, 1.0, A, lda, B, ldb, 0.0, C, M)
    else:
        F.ftblas_dgemm(tr[0], tr[1], M, N, K, 1.0, A, lda, B, ldb, 0.0, C, M, report=False)
for _ in range(3):
    call()
torch.cuda.synchronize()
prof.zero_()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record(); call(); e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
pv = prof.view(-1, 24).double()
p = pv[:, 20:24]
sel = p[:, 0] > 0
p, q = p[sel], pv[sel][:, 16:19]
m, mq = p[:, 1:].mean(0), q.mean(0)
stages = (K + 15) // 16
print(json.dumps({
    "mode": "noft" if noft else "ft", "MNK": [M, N, K], "trans": tr, "ms": ms, "ctas": int(p.shape[0]),
    "first_ready_clk": round(m[0].item()), "kloop_clk_per_stage": round((m[1] - m[0]).item() / stages, 1),
    "ideal_clk_per_stage": 4096, "epilogue_clk": round((m[2] - m[1]).item()), "tile_clk": round(m[2].item()),
    "epilogue_split_clk": {"check": round((mq[0] - m[1]).item()) if not noft else 0,
                           "stage_and_ring_release": round((mq[1] - (mq[0] if not noft else m[1])).item()),
                           "decide_to_store": round((mq[2] - mq[1]).item()), "store": round((m[2] - mq[2]).item())},
}), flush=True)
# grid-level view: CTA start (globaltimer, ns) and end (start + role clocks at the SM clock)
ghz = float(os.environ.get("SM_GHZ", "1.965"))
st = p[:, 0] - p[:, 0].min()
en = st + p[:, 3] / ghz
span = en.max().item()
ss, es = st.sort().values, en.sort().values
nsm = torch.cuda.get_device_properties(0).multi_processor_count
print(json.dumps({
    "span_us": span / 1e3, "event_ms": ms, "busy_frac_of_sms_x_span": (p[:, 3] / ghz).sum().item() / (nsm * span),
    "mean_cta_us": (p[:, 3] / ghz).mean().item() / 1e3,
    "start_us": {"cta_%d" % nsm: ss[min(nsm, len(ss) - 1)].item() / 1e3, "last": ss[-1].item() / 1e3},
    "end_us": {"first": es[0].item() / 1e3, "median": es[len(es) // 2].item() / 1e3, "last": es[-1].item() / 1e3},
}), flush=True)
if os.environ.get("TL_DUMP"):  # per CTA: blockIdx, start (ns from the first), duration (ns), first-ready clk, k-loop end clk
    import numpy as np
    idx = torch.nonzero(sel).flatten().cpu().numpy()
    np.save(os.environ["TL_DUMP"], np.stack([idx, st.cpu().numpy(), (p[:, 3] / ghz).cpu().numpy(),
                                             p[:, 1].cpu().numpy(), p[:, 2].cpu().numpy()], 1))
