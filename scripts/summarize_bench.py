"""Turns a bench.py JSON line (default run: headline + workloads) into the
markdown table of profiles/<round>/SUMMARY.md."""
import json
import sys


def main(path):
    d = json.loads(open(path).read().strip().splitlines()[-1])
    rows = [("gemm_bf16_16384 (headline)", d)]
    rows += list(d.get("workloads", {}).items())
    print("| workload | value | unit | step ms | roofline frac | bound | peak | clocks (MHz, reasons) |")
    print("|---|---|---|---|---|---|---|---|")
    for name, w in rows:
        if "error" in w:
            print(f"| {name} | error: {w['error']} |||||||")
            continue
        if "roofline" not in w:  # host-clock workloads (the graph API path)
            print(f"| {name} | {w['value']:.2f} | {w['unit']} | {w['ms_per_step']:.1f} | "
                  f"host clock | - | - | - |")
            continue
        r = w["roofline"]
        c = w.get("clocks", {})
        extra = f" (of op floor {r['frac_of_op_floor']:.2f})" if r.get("frac_of_op_floor") else ""
        print(f"| {name} | {w['value']:.1f} | {w['unit']} | {w['ms_per_step']:.4f} | "
              f"{r['frac']:.3f}{extra} | {r['bound']} | {r['peak']:.0f} {r['unit']} | "
              f"{c.get('sm_mhz')} {','.join(c.get('reasons', []))} |")
    e = d.get("e2e", {})
    print(f"\nHeadline e2e (C ABI, pinned host buffers, H2D + D2H inside the step): "
          f"{e.get('value', 0):.1f} {e.get('unit')} ({e.get('ms_per_step', 0):.2f} ms/step, "
          f"{e.get('h2d_bytes_per_step', 0) / 1e9:.2f} GB H2D + "
          f"{e.get('d2h_bytes_per_step', 0) / 1e9:.2f} GB D2H).")
    cb = d.get("cpu_baseline") or {}
    if cb:
        print(f"CPU baseline ({cb.get('kind')}, {cb.get('cores')} threads): {cb.get('value'):.3e} "
              f"{cb.get('unit')} on {cb.get('sample')}.")


if __name__ == "__main__":
    main(sys.argv[1])
