import csv,sys
for path in sys.argv[1:]:
    with open(path) as f:
        lines=[l for l in f if l.startswith('"')]
    rows=list(csv.DictReader(lines))
    print("==",path)
    tot=0
    for r in rows:
        if r["Metric Name"]!="gpu__time_duration.sum": continue
        v=float(r["Metric Value"].replace(",","")); u=r["Metric Unit"]
        ms = v/1e6 if u in("nsecond","ns") else v/1e3 if u in ("usecond","us") else v
        n=r["Kernel Name"]
        if n.startswith("k_probe_runs"): print("  -- total", round(tot,3)); tot=0
        tot+=ms
        if ms>0.2: print(f"  {ms:8.3f} {n[:50]}")
    print("  -- total", round(tot,3))
