# A/B sweep of the Tucker row kernel's rows-per-CTA / rows-per-batch (diagnostic)
for c in ${CONFIGS:-C2 C3}; do for r in ${ROWS:-64}; do for u in ${US:-4 8 16}; do
RSB200_TA_ROWS=$r RSB200_TA_U=$u timeout 200 python bench.py --config $c --no-cpu-baseline --steps 10 > gpurun_out/sw_${c}_${r}_${u}.json 2>/dev/null
done; done; done
