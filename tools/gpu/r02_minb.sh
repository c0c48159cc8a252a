for spec in ${SPECS}; do
  VDI_NVCC_EXTRA="$(echo $spec | tr ',' ' ')" python -m paper_2206_08660_b200.build > /dev/null 2>&1 || { echo "build fail $spec"; continue; }
  echo "$spec C3: $(timeout 300 python tools/run_pipeline.py --config C3 --reps 3 2>&1 | grep -o "'gen': [0-9.]*\|'render': [0-9.]*" | tr '\n' ' ')"
done
python -m paper_2206_08660_b200.build > /dev/null 2>&1
