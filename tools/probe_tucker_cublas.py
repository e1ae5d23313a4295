"""Diagnostic: cuBLAS DGEMM on the C5 Tucker-part shape (M = planes * n rows,
N = n, K = r3 = 132, C += A B^T) vs 8192^3, to calibrate k_tucker_gemm_res."""
import torch
torch.backends.cuda.matmul.allow_tf32 = False


def t(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


n = 2048
for planes, K in ((64, 132), (256, 132), (256, 136), (256, 40)):
    A = torch.randn(planes * n, K, dtype=torch.float64, device="cuda")
    B = torch.randn(n, K, dtype=torch.float64, device="cuda")
    C = torch.randn(planes * n, n, dtype=torch.float64, device="cuda")
    ms = t(lambda: C.addmm_(A, B.t()))
    ms0 = t(lambda: torch.mm(A, B.t(), out=C))
    fl = 2.0 * planes * n * n * K
    print(f"planes {planes} K {K}: C+=AB^T {ms:.3f} ms {fl / ms / 1e9:.1f} TF | C=AB^T {ms0:.3f} ms "
          f"{fl / ms0 / 1e9:.1f} TF")
    del A, B, C
a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
ms = t(lambda: a @ a, 3)
print(f"8192^3: {ms:.2f} ms {2 * 8192 ** 3 / ms / 1e9:.1f} TF")
