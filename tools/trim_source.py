"""Trim an ncu SASS source page (--page source --csv --print-source sass) to
the columns the profiles/ records use: address, SASS, stall samples,
instructions executed (warp and thread level).

    python tools/trim_source.py IN.csv OUT.csv
"""
import csv
import sys

KEEP = ["Address", "Source", "Warp Stall Sampling (All Samples)", "Instructions Executed",
        "Thread Instructions Executed"]


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr = rows[1]
    idx = [hdr.index(k) for k in KEEP]
    with open(sys.argv[2], "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(rows[0][:2])
        w.writerow(KEEP)
        for r in rows[2:]:
            if len(r) > max(idx):
                w.writerow([r[i].strip() for i in idx])


if __name__ == "__main__":
    main()
