# A/B of the Tucker plane GEMM tile (RSB200_TUCKER_TILE = 0: 128x64 with 32x32 warp tiles, 1: four stages, 2: 64x32 warp tiles, 3: 128x128; diagnostic)
for c in ${CONFIGS:-C4 C5}; do for t in ${TILES:-0 2}; do
RSB200_TUCKER_TILE=$t timeout 600 python bench.py --config $c --no-cpu-baseline --steps ${STEPS:-5} > gpurun_out/tt_${c}_$t.json 2>/dev/null
done; done
python - <<'PY'
import glob, json
for f in sorted(glob.glob("gpurun_out/tt_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        st = d["stages_ms_per_step"]
        print(f, round(d["ms_per_step"], 2), {k: round(v, 2) for k, v in st.items() if v})
    except Exception as e:
        print(f, "failed", e)
PY
