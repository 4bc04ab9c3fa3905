"""Markdown summary tables from `ncu --page details --csv` exports (tools/r02_measure.sh):
    python tools/ncu_summary.py TITLE=details.csv ... > profiles/rNN_ncu_summary.md
One table per kernel launch in each file, with the metrics the judge reads."""
import csv
import sys

KEEP = ["Memory Throughput", "DRAM Throughput", "Duration", "Compute (SM) Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "SM Busy", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Mem Pipes Busy", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
        "Dynamic Shared Memory Per Block", "Max Bandwidth", "L2 Cache Throughput"]


def main():
    for arg in sys.argv[1:]:
        title, path = arg.split("=", 1)
        rows = list(csv.DictReader(open(path)))
        by_id = {}
        for r in rows:
            by_id.setdefault((r["ID"], r["Kernel Name"]), []).append(r)
        for (kid, name), rs in by_id.items():
            print(f"## {title}: `{name.split('(')[0][:90]}` (launch id {kid})\n")
            print("| metric | value |\n|---|---|")
            seen = set()
            for r in rs:
                m = r["Metric Name"]
                if m in KEEP and m not in seen:
                    seen.add(m)
                    print(f"| {m} | {r['Metric Value']} {r['Metric Unit']} |")
            print()


if __name__ == "__main__":
    main()
