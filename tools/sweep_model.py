"""Split the sweep kernel's instructions into a per-move part and a
per-accepted-move part from an ncu SASS source page (`ncu -i rep --page source
--csv --print-source sass`), so the issue fraction of a sweep launch can be
quoted at that launch's own acceptance (the ncu-captured launch and the timed
ones come from different points of the Markov chain: their acceptances differ).

Every warp executes the per-move instructions once per move (count M = warps
per walker x W x S, the most common count); the update of an accepted move runs in
both warps of the walker (count A = acceptance x M) and the owner's write in
one (A / (warps per walker)).  Instructions with those two counts are the
per-accepted-move part, the rest (including the rare staging / fp64-decision
paths) the per-move part.  Both are normalised per (move, partner):

    thread instructions per launch = S W N (per_move_partner + acceptance x per_accepted_move_partner)

    python tools/sweep_model.py SOURCE.csv CONFIG W S N [profiles/r02_kernels.json]
"""
import collections
import csv
import json
import re
import sys


def model(src, W, S, N):
    rows = list(csv.reader(open(src)))
    kname = rows[0][1]
    tpb = int(re.search(r"j2_sweep_kernel<\(int\)(\d+)", kname).group(1))
    hdr = rows[1]
    ie = hdr.index("Instructions Executed")
    counts = [int(r[ie]) for r in rows[2:] if r[ie].strip()]
    nw = tpb // 32
    M = nw * W * S
    assert collections.Counter(counts).most_common(1)[0][0] == M   # the per-move body dominates
    mid = collections.Counter(c for c in counts if 0.05 * M < c < 0.99 * M)
    A = mid.most_common(1)[0][0]                 # the accepted-move update (every warp of the walker)
    owner = {c for c in mid if abs(c * nw - A) <= 1}
    acc_inst = sum(c for c in counts if c == A or c in owner)
    tot = sum(counts)
    mp = S * W * N
    acc = A / M
    return {"kernel": kname, "tpb": tpb, "acceptance_captured": acc,
            "per_move_partner": 32 * (tot - acc_inst) / mp,
            "per_accepted_move_partner": 32 * acc_inst / mp / acc,
            "thread_inst_per_move_partner_captured": 32 * tot / mp,
            "source": src.split("/")[-1]}


def main():
    src, cfg, W, S, N = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
    m = model(src, W, S, N)
    print(json.dumps(m))
    if len(sys.argv) > 6:
        rec = json.load(open(sys.argv[6]))
        m.pop("kernel")
        rec[cfg]["sweep_model"] = m
        json.dump(rec, open(sys.argv[6], "w"), indent=1)


if __name__ == "__main__":
    main()
