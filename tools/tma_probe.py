"""One 3D apply per (p, n) in a fresh process each: does the TMA path run (and match the
cp.async path bit for bit)?  Debug tool."""
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if len(sys.argv) > 1 and sys.argv[1] == "one":
    import torch
    from paper_1805_10058_b200 import igacd as ig
    p, n, aux = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    h = ig.igacd_create(3, p, n, 0.3, 0.05, 1.0, (0.48, 0.6, 0.64), levels=1)
    N = ig.igacd_ndof(h) // (3 if aux else 1)
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn(N, dtype=torch.float64, device="cuda", generator=g)
    y = torch.zeros_like(x)
    (ig.igacd_apply_aux if aux else ig.igacd_apply)(h, 0, x, y)
    torch.cuda.synchronize()
    torch.save(y.cpu(), "/tmp/probe_%s.pt" % os.environ.get("IGACD_TMA", "1"))
    print("ok")
    sys.exit(0)

for p, n in [(3, 7), (2, 8), (4, 8), (1, 10), (4, 30), (4, 160)]:
    for aux in (0, 1):
        res = {}
        for tma in ("0", "1"):
            env = dict(os.environ, IGACD_TMA=tma, CUDA_LAUNCH_BLOCKING="1")
            r = subprocess.run([sys.executable, __file__, "one", str(p), str(n), str(aux)], env=env,
                               capture_output=True, text=True)
            res[tma] = r.stdout.strip()[-40:] or r.stderr.strip().splitlines()[-1][-120:]
        same = None
        if res["0"] == "ok" and res["1"] == "ok":
            import torch
            same = bool(torch.equal(torch.load("/tmp/probe_0.pt"), torch.load("/tmp/probe_1.pt")))
        print(json.dumps({"p": p, "n": n, "m": n + p - 2, "aux": aux, "cpasync": res["0"], "tma": res["1"],
                          "bitwise_equal": same}), flush=True)
