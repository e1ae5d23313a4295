# A/B sweep of the plane GEMM's row blocks per launch (RSB200_PLANE_RBG; diagnostic)
for c in ${CONFIGS:-C3 C4}; do for g in ${RBGS:-0 18 37 74}; do
RSB200_PLANE_RBG=$g timeout 400 python bench.py --config $c --no-cpu-baseline --steps ${STEPS:-5} > gpurun_out/rbg_${c}_${g}.json 2>/dev/null
done; done
python - <<'EOF'
import glob, json
for f in sorted(glob.glob("gpurun_out/rbg_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d["ms_per_step"], 2), {k: round(v, 2) for k, v in d["stages_ms_per_step"].items() if v})
    except Exception as e:
        print(f, "failed", e)
EOF
