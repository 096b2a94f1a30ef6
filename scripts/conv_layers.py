"""Per-layer table of a ResNet-50 conv launch list (ncu gpu__time_duration)."""
import csv
import io
import sys

LAYERS = [(56, 64, 64, 1, 1, 1), (56, 64, 64, 3, 1, 3), (56, 64, 256, 1, 1, 3), (56, 64, 256, 1, 1, 1),
          (56, 256, 64, 1, 1, 2), (56, 256, 128, 1, 1, 1), (56, 128, 128, 3, 2, 1), (28, 128, 128, 3, 1, 3),
          (28, 128, 512, 1, 1, 4), (56, 256, 512, 1, 2, 1), (28, 512, 128, 1, 1, 3), (28, 512, 256, 1, 1, 1),
          (28, 256, 256, 3, 2, 1), (14, 256, 256, 3, 1, 5), (14, 256, 1024, 1, 1, 6), (28, 512, 1024, 1, 2, 1),
          (14, 1024, 256, 1, 1, 5), (14, 1024, 512, 1, 1, 1), (14, 512, 512, 3, 2, 1), (7, 512, 512, 3, 1, 2),
          (7, 512, 2048, 1, 1, 3), (14, 1024, 2048, 1, 2, 1), (7, 2048, 512, 1, 1, 2)]
txt = open(sys.argv[1]).read()
txt = txt[txt.index('"ID"'):]
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[0]
ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
conv = [float(r[iv]) / 1e3 for r in rows[1:] if "fill" not in r[ik]]
i = tot = totf = 0
for (H, C, OC, k, s, cnt) in LAYERS:
    OH = (H + 2 * (1 if k == 3 else 0) - k) // s + 1
    f = 2 * 256 * OH * OH * OC * C * k * k
    x_read = 256 * OH * OH * C if (k == 1 and s > 1) else 256 * H * H * C  # strided 1x1: every s-th pixel
    by = 2 * (x_read + 256 * OH * OH * OC + OC * C * k * k)
    t = sum(conv[i:i + cnt]) / cnt
    i += cnt
    tot += t * cnt
    totf += f * cnt
    print(f"{H:3d} {C:5d}->{OC:5d} k{k} s{s} x{cnt}: {t:7.1f} us {f / t / 1e6:7.1f} TF/s "
          f"{by / t / 1e3:6.0f} GB/s  AI {f / by:5.0f}  floor {max(f / 1614e6, by / 6547e3):6.1f} us")
print(f"total {tot:.1f} us, {totf / tot / 1e6:.1f} TF/s")
