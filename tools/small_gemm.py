import sys; sys.path.insert(0, '.')
import torch, tcxgen as g, paper_2206_02874_b200 as tcx
torch.cuda.set_device(0)
S = int(sys.argv[1]); K = int(sys.argv[2])
A = g.normal_matrix((S, K), "bf16", 0, g.STREAM_A, "cuda"); B = g.normal_matrix((S, K), "bf16", 0, g.STREAM_B, "cuda")
C = torch.zeros(S, S, device="cuda"); D = torch.empty_like(C)
for _ in range(5): tcx.gemm(A, B, C, D)
torch.cuda.synchronize()
if len(sys.argv) > 3:
    buf = torch.zeros(4 * ((S + 255) // 256) ** 2, dtype=torch.int64, device="cuda")
    tcx.debug_trace(buf); tcx.gemm(A, B, C, D); torch.cuda.synchronize(); tcx.debug_trace(None)
    t = buf.view(-1, 4).cpu()
    t0 = int(t[:, 1].min())
    print("trace (us from first MMA):", [(int(r[0]) & 0xffffffff, round((int(r[1]) - t0) / 1e3, 2), round((int(r[2]) - t0) / 1e3, 2), round((int(r[3]) - t0) / 1e3, 2)) for r in t[:4]])
