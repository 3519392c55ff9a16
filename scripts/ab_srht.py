"""A/B of the standalone SRHT tile kernels: each argument NAME=VALUE is the
environment of one child process (e.g. SQB_SRHT16_OLD=1); time + bitwise digest."""
import os, sys, subprocess, json, hashlib
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import torch
    import paper_2405_10923_b200 as P
    from paper_2405_10923_b200 import _lib
    from paper_2405_10923_b200.devarray import CODES, empty_colmajor, ld_of
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    out = []
    cases = [((1 << 20) - 128, 256, 128, "double"), ((1 << 22) - 201, 400, 16, "double"),
             ((1 << 20) - 128, 256, 128, "single"), ((1 << 22) - 201, 400, 1, "double"),
             ((1 << 20) - 128, 256, 1, "double"), (5000, 128, 3, "double"), ((1 << 14) - 32, 128, 32, "double"),
             ((1 << 24) - 256, 512, 16, "bf16"), ((1 << 20) - 128, 256, 16, "half"), (5000, 128, 3, "bf16"),
             ((1 << 22) - 201, 400, 4, "bf16")]
    for (n, ell, k, tag) in cases:
        om = P.SRHTSketch(ell, n, 8)
        g = torch.Generator(device="cuda"); g.manual_seed(5)
        X = empty_colmajor(n, k, tag)
        X.copy_(torch.randn(n, k, device="cuda", dtype=torch.float64, generator=g).to(X.dtype))
        Y = empty_colmajor(ell, k, "double")
        ctx = _lib.context(); d = om.desc()
        f = lambda: ctx.check(_lib.lib().sqb_sketch_apply(ctx.h, d, CODES[tag], X.data_ptr(), ld_of(X), k,
                                                          Y.data_ptr(), ld_of(Y)), "apply")
        for _ in range(3): f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        reps = 20
        e0.record()
        for _ in range(reps): f()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        b = X.element_size() * n * k + 8 * ell * k
        dig = hashlib.sha1(Y.cpu().numpy().tobytes()).hexdigest()[:12]
        out.append(f"n={n} ell={ell} k={k} {tag}: {ms*1e3:8.1f} us {b/ms/1e6:6.0f} GB/s = {b/ms/1e6/peak:.2f}  {dig}")
    print("\n".join(out))
else:
    for v in sys.argv[1:] or ["default"]:  # each argument: NAME=VALUE environment for one process
        env = dict(os.environ)
        if "=" in v:
            env[v.split("=")[0]] = v.split("=")[1]
        r = subprocess.run([sys.executable, __file__, "child"], env=env, capture_output=True, text=True)
        print(f"--- variant {v}\n{r.stdout}{r.stderr[-2000:]}")
