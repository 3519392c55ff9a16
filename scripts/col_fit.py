"""Fit t(c) = a + b c over an ncu launch list of rhqr_col_kernel (csv):
a = fixed per-pass cost (tail: lazy scale, w_c, tile FWHT, leaves), b = the
streaming cost of one more column."""
import collections
import csv
import sys

import numpy as np

rows = list(csv.reader(open(sys.argv[1])))
col_bytes = float(sys.argv[2]) if len(sys.argv) > 2 else 32 * 2 ** 20
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
hdr = rows[hi]
d = collections.defaultdict(dict)
for r in rows[hi + 1:]:
    x = dict(zip(hdr, r))
    v = float(x["Metric Value"].replace(",", ""))
    d[int(x["ID"])][x["Metric Name"]] = v / 1e3 if x["Metric Unit"] in ("ns", "nsecond") else v
ids = sorted(d)
ts = np.array([d[i]["gpu__time_duration.sum"] for i in ids])
cs = np.arange(1, len(ts) + 1, dtype=float)
a, b = np.linalg.lstsq(np.vstack([np.ones_like(cs), cs]).T, ts, rcond=None)[0]
print(f"t(c) = {a:.1f} us + {b:.3f} us * c   (streaming {col_bytes / b / 1e3:.0f} GB/s per extra column)")
for c in (1, 2, 8, 32, 64, 128, len(ts)):
    if c <= len(ts):
        print(f"  c={c:4d}: {ts[c - 1]:8.1f} us")
print(f"sum {ts.sum() / 1e3:.2f} ms over {len(ts)} launches; fixed part {a * len(ts) / 1e3:.2f} ms")
