# A/B of build_rs(prefetch_groups=k) in the bench step (BENCH_GROUPS; diagnostic)
for c in ${CONFIGS:-C4 C5}; do for g in ${GROUPS_:-1 2 4}; do
BENCH_GROUPS=$g timeout 600 python bench.py --config $c --no-cpu-baseline --steps ${STEPS:-5} > gpurun_out/grp_${c}_$g.json 2>/dev/null
done; done
python - <<'PY'
import glob, json
for f in sorted(glob.glob("gpurun_out/grp_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        st = d["stages_ms_per_step"]
        print(f, round(d["ms_per_step"], 2), {k: round(v, 2) for k, v in st.items() if v})
    except Exception as e:
        print(f, "failed", e)
PY
