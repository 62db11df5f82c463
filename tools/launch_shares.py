"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into kernel shares."""
import collections
import csv
import sys


def main(path, out=None):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in csv.DictReader(lines[start:]):
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].replace("(anonymous namespace)::", "")
        name = name.replace("void ", "").replace("unnamed>::", "").replace("bddc::", "")
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6}.get(unit, 1e-3)
        tot[name] += v * scale
        cnt[name] += 1
    T = sum(tot.values())
    text = [f"{path}: {sum(cnt.values())} launches, {T / 1e3:.2f} ms total device time "
            "(ncu: cold-cache, serialised; compare shares)"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        text.append(f"{100 * v / T:6.2f}%  {v / 1e3:9.3f} ms  n={cnt[k]:6d}  avg {v / cnt[k]:10.2f} us  {k}")
    s = "\n".join(text)
    if out:
        open(out, "w").write(s + "\n")
    print(s)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
