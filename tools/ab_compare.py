import sys
import numpy as np
a, b = np.load(sys.argv[1]), np.load(sys.argv[2])
ok = True
for k in a.files:
    same = np.array_equal(a[k], b[k])
    rel = float(np.max(np.abs(a[k].astype(np.float64) - b[k]) / np.abs(b[k].astype(np.float64)).clip(1e-6)))
    print(f"{k:24s} {'IDENTICAL' if same else 'DIFFERENT'} max_rel={rel:.3e}")
    ok &= same
print("ALL IDENTICAL" if ok else "SOME DIFFER")
