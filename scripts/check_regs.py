"""Build-time guard for kernels that redistribute registers with setmaxnreg:
setmaxnreg.inc only completes if the CTA's register pool (the per-thread
count ptxas allocated x threads) covers the requested split, otherwise the
warps wait forever. With setmaxnreg in a kernel ptxas allocates the
launch-bound maximum; this checks that it did, for every variant.

  gemm_tc_kernel<..., NG>   : 384 threads (NG = 2) -> 168 regs, 640 (NG = 4) -> 96
                              split 56 x 128 + {224 x 256 | 104 x 512}
  attn_fwd_kernel<D, BF16>  : 384 threads -> 168 regs (split 56/224 or 72/216)
"""
import re
import sys


def check(log, pattern, expect):
    bad = []
    cur = None
    n = 0
    for line in open(log):
        m = re.search(r"Compiling entry function '([^']+)'", line) or \
            re.search(r"Function properties for (\S+)", line)
        if m:
            cur = m.group(1)
        m = re.search(r"Used (\d+) registers", line)
        if m and cur and re.search(pattern, cur):
            n += 1
            want = expect(cur)
            if want is not None and int(m.group(1)) != want:
                bad.append((cur, int(m.group(1)), want))
    return n, bad


def gemm_expect(name):
    m = re.search(r"gemm_tc_kernelILi\d+ELi\d+ELb\dELb\dE.*?ELi(\d)EEEv", name)
    if not m:
        return None
    return 168 if m.group(1) == "2" else 96


def main(root="."):
    ok = True
    for log, pat, exp in ((f"{root}/build/afg/gemm_tc.ptxas.log", r"gemm_tc_kernel", gemm_expect),
                          (f"{root}/build/afg/attention.ptxas.log", r"attn_fwd_kernel", lambda n: 168)):
        n, bad = check(log, pat, exp)
        if n == 0:
            print(f"check_regs: no {pat} entries in {log}")
            ok = False
        for b in bad:
            print(f"check_regs: {b[0]} uses {b[1]} registers, setmaxnreg split needs {b[2]}")
            ok = False
    print("check_regs:", "ok" if ok else "FAILED")
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main(*sys.argv[1:]))
