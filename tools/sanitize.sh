#!/bin/bash
# compute-sanitizer passes over a small slice of the GPU tests: memcheck (out-of-bounds / misaligned accesses in every
# kernel the slice launches) and racecheck (shared-memory hazards of the staged probe engine and the bin build).
OUT=gpurun_out/${1:-sanitize}; mkdir -p $OUT
SLICE='tests/test_gpu_parity.py::test_build_parity_routed tests/test_gpu_parity.py::test_find_on_oracle_built_table tests/test_gpu_parity.py::test_build_parity tests/test_gpu_parity.py::test_build_default_values_and_host_memory tests/test_gpu_edge.py tests/test_gpu_workload.py::test_generate_keys_golden_fixture tests/test_gpu_workload.py::test_workload_golden_fixture tests/test_gpu_sharded_handle.py tests/test_gpu_parity.py::test_keys_only_insert_pairs_every_key_with_value_for_key tests/test_gpu_chunked.py::test_chunked_build_equals_one_bulk_insert tests/test_gpu_chunked.py::test_chain_cap_of_zero_fails_without_eviction tests/test_gpu_chunked.py::test_chunked_build_reports_overfull_table tests/test_gpu_sharded.py::test_fixed_segment_partition_against_numpy'
timeout 1700 compute-sanitizer --tool memcheck --error-exitcode 9 --log-file $OUT/memcheck.log python -m pytest $SLICE -x -q -m gpu > $OUT/memcheck_pytest.log 2>&1
echo "memcheck exit $?" | tee -a $OUT/memcheck_pytest.log; tail -3 $OUT/memcheck_pytest.log; tail -5 $OUT/memcheck.log
timeout 1700 compute-sanitizer --tool racecheck --error-exitcode 9 --log-file $OUT/racecheck.log python -m pytest 'tests/test_gpu_parity.py::test_build_parity_routed' tests/test_gpu_scenarios.py 'tests/test_gpu_chunked.py::test_chunked_build_equals_one_bulk_insert' -x -q -m gpu > $OUT/racecheck_pytest.log 2>&1
echo "racecheck exit $?" | tee -a $OUT/racecheck_pytest.log; tail -3 $OUT/racecheck_pytest.log; tail -5 $OUT/racecheck.log
