# Diagnostic: per-pixel forward mismatches (counts / colour) against the oracle for one case.
#   python scripts/gpu/fwd_mismatch.py c4 2 [view]
import os
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import pipeline as orc  # noqa: E402
from paper_2501_18630_b200 import PrimitiveSet, render_tiled  # noqa: E402
from paper_2501_18630_b200 import rasterizer as rz  # noqa: E402
from paper_2501_18630_b200.scenes import make_workload  # noqa: E402

cfg, seed = sys.argv[1], int(sys.argv[2])
view = int(sys.argv[3]) if len(sys.argv) > 3 else 0
wl = make_workload(cfg, seed=seed, views=(view + 1) if cfg == "c3" else None)
scene, cam, bg = wl.scene, wl.cameras[view], wl.background
ref = orc.forward(scene, cam, bg, core="c", threads=os.cpu_count())
prims = PrimitiveSet.from_scene(scene)
out = render_tiled(prims, cam, bg)
torch.cuda.synchronize()
cnt = out.pixel_count.cpu().numpy()
col = out.raw_color.cpu().numpy()
T = out.transmittance.cpu().numpy()
rc = ref["pix_count"]
bad = np.argwhere(cnt != rc)
print("mismatching pixels", len(bad), "flagged", rz.frame_status(out.frame)["flagged_pixels"])
for y, x in bad[:20]:
    print(f"  px ({x},{y}) count dev {cnt[y, x]} ref {rc[y, x]}  T dev {T[y, x]:.6g} ref {ref["T"][y, x]:.6g}"
          f"  raw err {np.abs(col[y, x] - ref['raw'][y, x]).max():.3g}")
err = np.abs(col - ref["raw"]).max(axis=2)
yy, xx = np.unravel_index(np.argmax(err), err.shape)
print("max raw err", err.max(), "at", (xx, yy), "count dev", cnt[yy, xx], "ref", rc[yy, xx])

# the primitives whose contribution counts differ, and the mismatching pixel's chain in fp64
dc = out.contributions.cpu().numpy() - ref["contributions"]
diff_src = np.nonzero(dc)[0]
print("primitives with different counts:", [(int(i), int(dc[i])) for i in diff_src[:10]])
if len(bad):
    y, x = bad[0]
    s = ref["shaded"]["sorted"]
    src_of_sorted = ref["batch"]["indices"][ref["order"]]
    tw = (cam.width + 15) // 16
    t = (y // 16) * tw + x // 16
    lst = ref["lists"][ref["offsets"][t]:ref["offsets"][t + 1]]
    T = 1.0
    taken = 0
    for k, e in enumerate(lst):
        b = s["bounds"][e]
        if not (b[0] <= x <= b[1] and b[2] <= y <= b[3]):
            continue
        mx, my = s["means"][e]
        ca, cb, cc = s["conics"][e]
        dx, dy = x - mx, y - my
        r2 = ca * dx * dx + 2.0 * cb * dx * dy + cc * dy * dy
        xx = min(max(r2, 0.0), 1.0)
        kern = 0.0 if (xx == 1.0 and s["betas"][e] > 0) else (1.0 - xx) ** s["betas"][e]
        a = s["opac"][e] * kern
        src = int(src_of_sorted[e])
        mark = " <== count differs" if dc[src] != 0 else ""
        if a < orc.ALPHA_MIN:
            if a > 0.9 * orc.ALPHA_MIN or mark:
                print(f"    entry {k} src {src} alpha {a:.9g} (below cutoff by {(orc.ALPHA_MIN - a) / orc.ALPHA_MIN:.3g} rel) r2 {r2:.9g}{mark}")
            continue
        Tn = T * (1.0 - a)
        taken += 1
        print(f"  entry {k} src {src} alpha {a:.9g} T {T:.9g} -> {Tn:.9g} beta {s['betas'][e]:.4g} r2 {r2:.9g}{mark}")
        T = Tn
        if T < orc.T_STOP:
            print("  reference stops here after", taken)
            break
