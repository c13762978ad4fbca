"""Opcode mix, divergence and shared-memory wavefronts of one kernel from an
`ncu --page source --csv --print-source sass` export (profiling helper)."""
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    data = []
    for r in rows[2:]:
        if r and r[0] == "Kernel Name":
            break  # first kernel instance only
        if len(r) == len(hdr):
            data.append(r)
    return hdr, data


def main(path, top=18):
    hdr, data = load(path)
    ix = {h: i for i, h in enumerate(hdr)}
    num = lambda r, c: float(r[ix[c]] or 0) if c in ix else 0.0
    tot = sum(num(r, "Instructions Executed") for r in data)
    thr = sum(num(r, "Thread Instructions Executed") for r in data)
    wf = sum(num(r, "L1 Wavefronts Shared") for r in data)
    wfi = sum(num(r, "L1 Wavefronts Shared Ideal") for r in data)
    print(f"{path}: {len(data)} SASS lines, {tot / 1e6:.2f}M warp instructions, "
          f"{thr / max(tot, 1):.1f} threads/instruction, shared wavefronts {wf / 1e6:.2f}M (ideal {wfi / 1e6:.2f}M)")
    ops = {}
    for r in data:
        src = r[ix["Source"]].strip().split()
        if not src:
            continue
        op = src[1] if src[0].startswith("@") and len(src) > 1 else src[0]
        op = op.split(".")[0]
        ops[op] = ops.get(op, 0) + num(r, "Instructions Executed")
    print(" ".join(f"{k}:{100 * v / tot:.1f}%" for k, v in sorted(ops.items(), key=lambda x: -x[1])[:top]))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
