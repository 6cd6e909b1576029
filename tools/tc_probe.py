"""Validate the tcgen05 TF32 path and characterise its numerics (GPU box)."""
import ctypes as C, os, sys, numpy as np
L = C.CDLL(os.path.join(os.path.dirname(__file__), "libtcprobe.so"))
f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
L.tc_probe.argtypes = [f32p, f32p, f32p, C.c_int, C.c_int]

def run(A, B):
    N, K = B.shape
    D = np.zeros((128, N), np.float32)
    rc = L.tc_probe(np.ascontiguousarray(A, np.float32), np.ascontiguousarray(B, np.float32), D, N, K)
    assert rc == 0, f"cuda error {rc}"
    return D

def trunc(x):  # tf32 by truncation of the low 13 mantissa bits
    return (np.ascontiguousarray(x, np.float32).view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)

def rne(x):    # tf32 by round-to-nearest-even
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0xFFF + ((u >> 13) & 1)) & 0xFFFFE000
    return u.astype(np.uint32).view(np.float32)

rng = np.random.default_rng(0)
ok = True
for N, K in [(64, 48), (32, 64), (64, 8), (256, 32)]:
    A = rng.standard_normal((128, K)).astype(np.float32)
    B = rng.standard_normal((N, K)).astype(np.float32)
    D = run(A, B).astype(np.float64)
    exact = A.astype(np.float64) @ B.astype(np.float64).T
    et = trunc(A).astype(np.float64) @ trunc(B).astype(np.float64).T
    er = rne(A).astype(np.float64) @ rne(B).astype(np.float64).T
    scale = np.abs(A).astype(np.float64) @ np.abs(B).astype(np.float64).T
    e_exact = np.max(np.abs(D - exact) / scale)
    e_t = np.max(np.abs(D - et) / scale)
    e_r = np.max(np.abs(D - er) / scale)
    print(f"N={N} K={K}: max |D-exact|/sum|ab| = {e_exact:.3e}  vs trunc-tf32 {e_t:.3e}  vs rne-tf32 {e_r:.3e}")
    ok &= e_exact < 4e-3
# accumulation precision: tf32-exact inputs, so only the accumulation rounds
for K in (8, 64):
    A = trunc(rng.standard_normal((128, K)).astype(np.float32) * 1000)
    B = trunc(rng.standard_normal((64, K)).astype(np.float32))
    D = run(A, B).astype(np.float64)
    exact = A.astype(np.float64) @ B.astype(np.float64).T
    scale = np.abs(A).astype(np.float64) @ np.abs(B).astype(np.float64).T
    print(f"accumulation K={K}: max |D-exact|/sum|ab| = {np.max(np.abs(D-exact)/scale):.3e} "
          f"(fp32 recursive bound K*2^-24 = {K*2**-24:.3e})")
print("TC PROBE", "OK" if ok else "FAILED")
sys.exit(0 if ok else 1)
