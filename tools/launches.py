"""Summarise an ncu launch-list CSV: the last compress+decompress step."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
for i, r in enumerate(rows):
    if r and r[0] == "ID":
        h = r; data = rows[i + 1:]; break
ix = {k: i for i, k in enumerate(h)}
ks = [(r[ix["Kernel Name"]].split("(")[0].replace("void ", "").replace("cszi::", ""),
       float(r[ix["Metric Value"]].replace(",", ""))) for r in data]
# last step = from the last k_ctl_init before the final k_range to the end
start = max(i for i, k in enumerate(ks) if k[0] == "k_range") - 1
step = ks[start:]
tot = sum(v for _, v in step)
for n, v in step:
    print(f"{v/1000:10.1f} us  {100*v/tot:5.1f}%  {n}")
print(f"{tot/1000:10.1f} us total")
