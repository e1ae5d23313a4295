"""Diagnostic: tcgen05 kind::i8 GEMM throughput (rs_tc8_gemm_s8, rs_oz_gemm)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1606_09218_b200 import _native as nat
L = nat.lib()
for M, N, K in [(148 * 128 * 2, 64, 8192), (148 * 128 * 2, 64, 2048)]:
    A = torch.randint(-100, 100, (M, K), dtype=torch.int8, device="cuda")
    B = torch.randint(-100, 100, (N, K), dtype=torch.int8, device="cuda")
    C = torch.empty((M, N), dtype=torch.int32, device="cuda")
    for _ in range(2):
        L.rs_tc8_gemm_s8(A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), N, M, N, K, nat.stream_ptr())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        L.rs_tc8_gemm_s8(A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), N, M, N, K, nat.stream_ptr())
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 5 * 1e-3
    ummas = (M // 128) * (N // 64) * (K // 32)
    print(f"s8 M={M} N={N} K={K}: {t*1e3:.3f} ms  {2*M*N*K/t/1e12:.1f} TOPS  "
          f"{t*1.965e9*148/ummas:.1f} clk/UMMA")
for M, N, K, S in [(65536, 256, 704, 7), (65536, 256, 704, 6)]:
    A = torch.randn(M, K, dtype=torch.float64, device="cuda")
    B = torch.randn(N, K, dtype=torch.float64, device="cuda")
    C = torch.empty((M, N), dtype=torch.float64, device="cuda")
    ws = torch.empty(L.rs_oz_workspace_bytes(M, N, K, S), dtype=torch.uint8, device="cuda")
    args = (A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), N, M, N, K, None, 1, S, 0,
            ws.data_ptr(), ws.numel(), nat.stream_ptr())
    L.rs_oz_gemm(*args); torch.cuda.synchronize()
    L.rs_prof_enable(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        L.rs_oz_gemm(*args)
    e1.record(); torch.cuda.synchronize()
    L.rs_prof_enable(0)
    ms, cnt = nat.prof_query("oz_mma")
    t = e0.elapsed_time(e1) / 5
    ummas = (M // 128) * (N // 64) * (K // 32) * S * (S + 1) // 2
    print(f"oz S={S} M={M} N={N} K={K}: total {t:.3f} ms, mma {ms/5:.3f} ms, "
          f"{ms/5*1e-3*1.965e9*148/ummas:.1f} clk/UMMA, fp64-equiv {2*M*N*K/(ms/5*1e-3)/1e12:.1f} TF")
