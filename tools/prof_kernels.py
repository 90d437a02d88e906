"""Tiny driver for ncu captures: runs the config-2 NTT/INTT/MAC once each
after a warm-up (usage: python tools/prof_kernels.py [ntt|ks])."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_01296_b200.engine import Engine
from paper_2402_01296_b200.params import make_params

what = sys.argv[1] if len(sys.argv) > 1 else "ntt"
if what == "ntt":
    hp = make_params(8192, 3, 60, dnum=1, n_special=1)
    eng = Engine(hp)
    data = eng.sample_uniform(8192, 4, 0, seed=1)
    pts = eng.to_montgomery(eng.sample_uniform(4096, 4, 0, seed=2))
    for _ in range(2):
        eng.ntt(data, 0)
        eng.ntt(data, 0, inverse=True)
        eng.mac(data.view(4096, 2, 4, 8192), pts, 25)
    torch.cuda.synchronize()
elif what == "ntt14":
    # bench_micro.ntt14 launch: 128 polys x 12 limbs of N = 2^14, 50-bit primes
    hp = make_params(16384, 14, 50, dnum=3)
    eng = Engine(hp)
    data = eng.sample_uniform(128, 12, 0, seed=1)
    for _ in range(2):
        eng.ntt(data, 0)
        eng.ntt(data, 0, inverse=True)
    torch.cuda.synchronize()
elif what == "convks":
    # cifar3 conv2 shape: 16 sources x 9 taps = 144 terms, 32 outputs, level 11, G = 32
    from paper_2402_01296_b200.params import galois_element as ge
    import ctypes
    from paper_2402_01296_b200 import _lib
    hp = make_params(16384, 14, 50, dnum=3)
    eng = Engine(hp)
    lvl, G, O = 11, int(os.environ.get("PROF_G", "32")), 32
    srcs = [eng.sample_uniform(2 * G, lvl + 1, 0, seed=9 + i).view(G, 2, lvl + 1, 16384) for i in range(16)]
    Us = [eng.modup(x, lvl) for x in srcs]
    rots = [0, 1, 2, 16, 17, 18, 32, 33, 34]
    terms = [(srcs[c], Us[c], ge(r, 16384) if r else 1) for c in range(16) for r in rots]
    nb = ctypes.c_uint64()
    _lib.call("bcn_planes_ext_bytes", eng._h, O, len(terms), lvl, ctypes.byref(nb))
    planes = torch.randint(0, 256, (int(nb.value),), dtype=torch.uint8, device="cuda")
    layout = int(os.environ.get("PROF_LAYOUT", "0"))     # 1: tcgen05 (use PROF_G=64)
    for _ in range(2):
        eng.conv_ks_mac([t[0] for t in terms], [t[1] if t[2] != 1 else None for t in terms], [t[2] for t in terms],
                        planes, O, lvl, layout)
    torch.cuda.synchronize()
elif what == "rotsum3":
    # pooling / compaction shape of cifar3: 3 rotations of one source at level 7, G = 32
    from paper_2402_01296_b200.params import galois_element as ge
    hp = make_params(16384, 14, 50, dnum=3)
    eng = Engine(hp)
    lvl, G = 7, 32
    ct = eng.sample_uniform(2 * G, lvl + 1, 0, seed=5).view(G, 2, lvl + 1, 16384)
    U = eng.modup(ct, lvl)
    pts = [eng.to_montgomery(eng.sample_uniform(1, lvl + 1 + hp.K, 0, seed=100 + i)) for i in range(3)]
    terms = [(ct, U, ge(r, 16384), pts[i]) for i, r in enumerate((1, 16, 17))]
    keys = [eng.premul_key(t[2], t[3], lvl) for t in terms]
    for _ in range(3):
        eng.rotsum(terms, lvl, keys=keys)
    torch.cuda.synchronize()
elif what in ("rotsum", "mac"):
    # fc1-like: one level-5 source (cifar3 chain), 96 rotate-multiply terms, G = 32 slot sets
    from paper_2402_01296_b200.params import galois_element as ge
    hp = make_params(16384, 14, 50, dnum=3)
    eng = Engine(hp)
    lvl, G = 5, 32
    ct = eng.sample_uniform(2 * G, lvl + 1, 0, seed=5).view(G, 2, lvl + 1, 16384)
    U = eng.modup(ct, lvl)
    pts = [eng.to_montgomery(eng.sample_uniform(1, lvl + 1 + hp.K, 0, seed=100 + i)) for i in range(96)]
    terms = [(ct, U, ge(i + 1, 16384), pts[i]) for i in range(96)]
    qterms = [(ct, eng.to_montgomery(eng.sample_uniform(1, lvl + 1, 0, seed=300 + i))) for i in range(96)]
    for _ in range(2):
        if what == "rotsum":
            eng.rotsum(terms, lvl)
        else:
            eng.mac_terms(qterms, lvl, rescale=False)
    torch.cuda.synchronize()
elif what == "multi":
    # conv2-like multi-output MAC: 144 rotated cts x 16 outputs, level 12, G = 8
    hp = make_params(16384, 14, 50, dnum=3)
    eng = Engine(hp)
    lvl, G, K = 12, int(os.environ.get('PROF_G', '8')), 144
    cts = [eng.sample_uniform(2 * G, lvl + 1, 0, seed=7 + k).view(G, 2, lvl + 1, 16384) for k in range(K)]
    pts = [[eng.to_montgomery(eng.sample_uniform(1, lvl + 1, 0, seed=1000 + 200 * o + k)) for k in range(K)]
           for o in range(16)]
    if os.environ.get("PROF_IMMA", "0") == "1":
        planes = eng.pack_planes(pts, lvl)
        for _ in range(2):
            eng.mac_multi_planes(cts, planes, 16, lvl)
    else:
        for _ in range(2):
            eng.mac_multi(cts, pts, lvl)
    torch.cuda.synchronize()
else:
    hp = make_params(16384, 7, 50, dnum=2, n_special=1)
    eng = Engine(hp)
    L = hp.max_level
    cts = eng.sample_uniform(256, 8, 0, seed=3).view(128, 2, 8, 16384)
    for _ in range(2):
        sq = eng.mul_cc(cts, cts, L, rescale=False)
        U = eng.modup(sq, L)
        eng.rotate(sq, 1, L, U=U)
    torch.cuda.synchronize()
print("done")
