# PAPER Table 1 (k = 5..9) on the B200 via tools/bench_cli.py
for k in 5 6 7 8 9; do timeout 900 python tools/bench_cli.py --k $k --output gpurun_out/table1_k$k.json > gpurun_out/table1_k$k.log 2>&1; echo k$k $?; done
python - <<'PY'
import json, os
rows = []
for k in range(5, 10):
    p = f"gpurun_out/table1_k{k}.json"
    if os.path.exists(p):
        d = json.load(open(p))
        rows.append(d[0] if isinstance(d, list) else d)
json.dump(rows, open("gpurun_out/table1_b200.json", "w"), indent=1)
for r in rows:
    print(r["k"], round(r["t_s"], 2), round(r["t_apply"], 4), round(r["t_nf"], 4), round(r["t_ff"], 4), r["N_SC"], r["N_C"], "%.2g" % r["sampled_rel_error"], round(r.get("speedup_vs_paper_apply", 0)))
PY
