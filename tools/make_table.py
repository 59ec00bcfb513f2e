"""Build the measured flat-selector table from tools/sweep.py output.

    python tools/make_table.py gpurun_out/sweep_p2.csv gpurun_out/sweep_p4.csv ...

Writes paper_2504_18658_b200/data/flat_calibration.csv: for every
(collective, p, size) every algorithm's best busbw over the CTA counts tried
(the selector picks the max per size bucket, selector.FlatTable.best).
"""
import csv
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_18658_b200.selector import FLAT_TABLE_PATH, FlatEntry, FlatTable  # noqa: E402

NAMES = {"ag": "all_gather", "rs": "reduce_scatter"}


def main(paths):
    best = {}
    for path in paths:
        for r in csv.DictReader(open(path)):
            if r["algo"] == "nccl":
                continue
            key = (NAMES[r["coll"].split("_")[0]], int(r["p"]), int(r["S"]), r["algo"])
            best[key] = max(best.get(key, 0.0), float(r["busbw"]))
    t = FlatTable()
    for (coll, p, S, algo), bw in sorted(best.items()):
        t.add(FlatEntry(coll, p, S, algo, bw))
    os.makedirs(os.path.dirname(FLAT_TABLE_PATH), exist_ok=True)
    t.save_csv(FLAT_TABLE_PATH)
    print(f"{len(t.entries)} entries -> {FLAT_TABLE_PATH}")


if __name__ == "__main__":
    main(sys.argv[1:])
