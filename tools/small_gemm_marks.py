import sys; sys.path.insert(0, '.')
import torch, tcxgen as g, paper_2206_02874_b200 as tcx
torch.cuda.set_device(0)
S, K = int(sys.argv[1]), int(sys.argv[2])
A = g.normal_matrix((S, K), "bf16", 0, g.STREAM_A, "cuda"); B = g.normal_matrix((S, K), "bf16", 0, g.STREAM_B, "cuda")
C = torch.zeros(S, S, device="cuda"); D = torch.empty_like(C)
for _ in range(5): tcx.gemm(A, B, C, D)
torch.cuda.synchronize()
buf = torch.zeros(64, dtype=torch.int64, device="cuda")
for rep in range(3):
    buf.zero_(); tcx.debug_trace(buf); tcx.gemm(A, B, C, D); torch.cuda.synchronize(); tcx.debug_trace(None)
    t = buf.cpu().tolist()
    t0 = t[60]
    rel = lambda x: round((x - t0) / 1e3, 2) if x else None
    print("entry->pdl_wait", rel(t[61]), "first MMA", rel(t[1]), "last commit", rel(t[2]), "epi marks", [rel(x) for x in t[4:14]], "epi end(store issue)", rel(t[3]), "bulk_wait done", rel(t[62]))
