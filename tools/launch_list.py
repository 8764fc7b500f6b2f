"""Per-round kernel times of the last search in an ncu launch list.

    python tools/launch_list.py gpurun_out/launches.csv

Input: the csv of `ncu --metrics gpu__time_duration.sum --csv --log-file`.
Prints the filter / select durations (us) of every round of the last
search call (the launches after the last init_state_kernel).
"""
import csv
import sys


def load(path):
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rows = list(csv.reader(lines))
    h = rows[0]
    out = []
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        if d["Metric Unit"] == "ns":
            v /= 1000.0
        elif d["Metric Unit"] == "ms":
            v *= 1000.0
        out.append((d["Kernel Name"], v))
    return out


def short(name):
    for key in ("filter_tc_kernel", "filter_simt_kernel", "select_reg_kernel", "select_kernel",
                "init_state", "finalize", "reset_kernel", "group_ranges", "encode", "merge"):
        if key in name:
            return key
    return name.split("(")[0][-40:]


def main():
    ks = load(sys.argv[1])
    back = int(sys.argv[2]) if len(sys.argv) > 2 else 1  # n-th last search call
    inits = [i for i, (n, _) in enumerate(ks) if "init_state" in n]
    last = inits[-back]
    if back > 1:
        ks = ks[:inits[-back + 1]]
    # include the group-range / encode launches just before init_state
    seq = ks[last:]
    fil = [round(v, 1) for n, v in seq if "filter" in n]
    sel = [round(v, 1) for n, v in seq if "select" in n]
    other = [(short(n), round(v, 1)) for n, v in seq if "filter" not in n and "select" not in n]
    print("filter", fil, "sum", round(sum(fil), 1))
    print("select", sel, "sum", round(sum(sel), 1))
    print("other", other, "sum", round(sum(v for _, v in other), 1))


if __name__ == "__main__":
    main()
