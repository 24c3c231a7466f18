timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/exp15_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/exp15_tests.txt 2>&1
cat gpurun_out/exp15_tests.txt
