"""Per-block timeline of the tcgen05 attention prefill (MMA-issuer clock64 stamps of CTA 0:
S issued, next S issued, P ready) via sn_experimental_fa5_timeline.

  python tools/fa5_timeline.py [T Hq Hkv]   (default 16384 32 8)
"""
import ctypes, math, os, sys, torch
os.environ.setdefault("SN_FA5_TWO", "0")  # the stamps are in the one-tile kernel
sys.path.insert(0, '.')
from paper_2604_19877_b200 import ops, _lib
lib = _lib.load()
f = lib.sn_experimental_fa5_timeline; f.argtypes = [ctypes.c_void_p]; f.restype = None
T, Hq, Hkv = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (16384, 32, 8)))
D = 128
q = torch.randn(T, Hq, D, device="cuda").to(torch.bfloat16); k = torch.randn(T, Hkv, D, device="cuda").to(torch.bfloat16); v = torch.randn_like(k)
cu = torch.tensor([0, T], dtype=torch.int32, device="cuda"); out = torch.empty(T, Hq * D, device="cuda", dtype=torch.bfloat16)
ops.attn_prefill(q, k, v, cu, out, Hq, Hkv, D, 0, 1 / math.sqrt(D))
dbg = torch.zeros(64 * 8, dtype=torch.int64, device="cuda")
f(dbg.data_ptr()); ops.attn_prefill(q, k, v, cu, out, Hq, Hkv, D, 0, 1 / math.sqrt(D)); torch.cuda.synchronize(); f(None)
d = dbg.view(64, 8).cpu().double(); t0 = d[0, 0]
nb = min(64, (T + 127) // 128)
for j in range(0, nb - 1, max(1, nb // 16)):
    print(j, ["%7.0f" % (x - t0) for x in d[j, :4].tolist()], "K(j) ready->S(j+1) issued %5.0f, P wait %5.0f, PV issue %5.0f, block %5.0f" % (d[j,1]-d[j,0], d[j,2]-d[j,1], d[j,3]-d[j,2], (d[j+1,0]-d[j,0]) if j < 63 else 0))
print("softmax warp 0 (CTA 0): S ready -> S loaded -> row max combined -> P handed over -> next S ready")
for j in range(0, nb - 1, max(1, nb // 16)):
    print(j, "ld %5.0f  max+bar %5.0f  exp/P %5.0f  wait next S %5.0f" % (d[j,5]-d[j,4], d[j,6]-d[j,5], d[j,7]-d[j,6], d[j+1,4]-d[j,7]))
