# A/B of the eigen block's CTA widths (RSB200_ORTH_THREADS x RSB200_JACOBI_THREADS; diagnostic)
for c in ${CONFIGS:-C2}; do for o in 256 1024; do for j in 256 512; do for rep in 1 2; do
RSB200_ORTH_THREADS=$o RSB200_JACOBI_THREADS=$j timeout 300 python bench.py --config $c --no-cpu-baseline --steps ${STEPS:-20} > gpurun_out/eig_${c}_${o}_${j}_$rep.json 2>/dev/null
done; done; done; done
python - <<'PY'
import glob, json
for f in sorted(glob.glob("gpurun_out/eig_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        st = d["stages_ms_per_step"]
        print(f, round(d["ms_per_step"], 3), "e2e", round(d["e2e"]["ms_per_step"], 3), "topeig", round(st["topeig"], 3))
    except Exception as e:
        print(f, "failed", e)
PY
