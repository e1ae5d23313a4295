# A/B of the A-resident Tucker GEMM (RSB200_TUCKER_RES = 64 default, 128, 0 = per-tile plane GEMM; diagnostic)
for c in ${CONFIGS:-C3 C4 C5}; do for t in ${RES:-1 0}; do
RSB200_TUCKER_RES=$t timeout 600 python bench.py --config $c --no-cpu-baseline --steps ${STEPS:-5} > gpurun_out/tres_${c}_$t.json 2>/dev/null
done; done
python - <<'PY'
import glob, json
for f in sorted(glob.glob("gpurun_out/tres_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        st = d["stages_ms_per_step"]
        print(f, round(d["ms_per_step"], 2), "e2e", round(d["e2e"]["ms_per_step"], 1), {k: round(v, 2) for k, v in st.items() if v})
    except Exception as e:
        print(f, "failed", e)
PY
