build/microbench/call_overhead
timeout 300 python - <<'PY'
import sys, time, torch
sys.path.insert(0, ".")
import paper_1304_7054_b200 as kb
n, e = 10, 100
for batch in (1, 64, 65536):
    X = torch.rand(e * batch, device="cuda"); Y = torch.empty_like(X)
    A = torch.rand(e, device="cuda"); B = torch.rand(e, device="cuda")
    s = torch.cuda.Stream(); ex = kb.Exec(stream=s, asynchronous=True)
    pr = kb.KronProblem2D(m_a=n, n_a=n, m_b=n, n_b=n)
    mA, mB = kb.MatrixView(A, n, n, n), kb.MatrixView(B, n, n, n)
    xv, yv = kb.BatchView(kb.MatrixView(X, n, n, n), batch, e), kb.BatchView(kb.MatrixView(Y, n, n, n), batch, e)
    for _ in range(50): kb.kron2(pr, mA, mB, xv, yv, exec_=ex)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(2000): kb.kron2(pr, mA, mB, xv, yv, exec_=ex)
    t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"python kb.kron2 batch {batch}: host {(t1-t0)/2000*1e6:.2f} us/call, total {(t2-t0)/2000*1e6:.2f} us/call")
PY
