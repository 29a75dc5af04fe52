"""Graph-timed sweep of explicit GEMM plans (bn, mc, splits) for the verify / draft shapes."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import gemm_stream  # noqa: E402

shapes = [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]]
for n, t, k in shapes:
    res = []
    for bn in ((32, 64, 128) if t <= 512 and not os.environ.get('SWEEP_WIDE') else (64, 128, 256)):
        for mc in (1, 2, 4):
            if mc * bn > 512 or (n // 128) < mc:
                continue
            for sp in ((1, 2, 3, 4, 6, 8) if t <= 512 else (1, 2, 4)):
                if k // 64 // sp < 2:
                    continue
                try:
                    r = gemm_stream.run(n, t, k, bn=mc * 10000 + 2000 + bn, splits=sp, iters=40)
                except Exception as e:  # noqa: BLE001
                    continue
                res.append((r["us"], bn, mc, sp))
    res.sort()
    print(json.dumps({"n": n, "t": t, "k": k, "best": res[:6]}), flush=True)
