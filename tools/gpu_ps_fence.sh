# k_prio_settle: 2-stage TMA ring with the cross-proxy fence (the 2-stage ring without it failed s22 parity)
mkdir -p gpurun_out
for tag in s3 s2; do
  if [ $tag = s2 ]; then rm -f paper_2605_29604_b200/_obj/solver.cu.o; TCMIS_NVCC_EXTRA=-DTCMIS_PS_STAGES=2 python -m paper_2605_29604_b200.build > gpurun_out/psf_build.log 2>&1; fi
  for c in rmat22 rmat26; do
    timeout 300 python bench.py --config $c --no-e2e --no-cpu-baseline > gpurun_out/psf${tag}_$c.json 2> gpurun_out/psf${tag}_$c.log; echo "$tag $c rc=$? $(tail -1 gpurun_out/psf${tag}_$c.log | cut -c1-150)"
  done
  timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "golden" > gpurun_out/psf_pytest_$tag.txt 2>&1; echo "$tag pytest=$? $(tail -1 gpurun_out/psf_pytest_$tag.txt)"
done
