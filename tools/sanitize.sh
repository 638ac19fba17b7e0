#!/bin/bash
# compute-sanitizer over every kernel family of libvsbp.so, run
# under gpurun from the repo root:   tools/sanitize.sh TAG [tools...]
# Each tool runs a selection of small GPU parity tests (C1, reduced C2 shapes,
# ragged tails, every storage width / kernel variant) with only the library's
# kernels (namespace vsbp) checked.  Logs: gpurun_out/san_TAG_<tool>.log; the
# summary line of each is printed.  --error-exitcode makes any finding visible.
TAG=${1:-run}
shift
TOOLS=${@:-memcheck racecheck synccheck initcheck}
mkdir -p gpurun_out
python -c "from paper_1902_09733_b200 import build as B; B.build()" || exit 1
T=tests/test_gpu_parity.py
SEL=(
  "$T::test_config1_shift" "$T::test_config1_row_plane_hierarchical"
  "$T::test_bp_fuzz[0]" "$T::test_bp_fuzz[3]" "$T::test_bp_fuzz[7]" "$T::test_bp_fuzz[12]"
  "$T::test_storage_widths_agree" "$T::test_wide_tau_q_u16_and_i32_storage"
  "$T::test_level0_data_term_from_images_or_memory" "$T::test_generic_and_fused_kernels_agree_with_oracle"
  "$T::test_costpyr_wide_tiles_ragged" "$T::test_batch_equals_single"
  "$T::test_prep_bit_exact" "$T::test_prep_s4_kernels"
  "$T::test_jbu_small" "$T::test_jbu_large_radius_scalar_path" "$T::test_jbu_vector_path_equals_scalar_path"
  "$T::test_jbu_far_pixels_vector_equals_scalar_and_oracle" "$T::test_reproject_matches_oracle"
  "$T::test_jbu_reproject_ragged" "$T::test_rectify_prep_bit_exact" "$T::test_harris_corners_bit_exact"
  "$T::test_zssd_match_bit_exact" "$T::test_csbp_config1_shift" "$T::test_csbp_fuzz[0]" "$T::test_csbp_fuzz[5]"
  "$T::test_icp_constructed_motion_matches_oracle" "$T::test_icp_failure_and_identity"
  "$T::test_fused_final_iteration_matches_oracle"
)
EXTRA=${SAN_EXTRA_TESTS:-}
for tool in $TOOLS; do
  extra_opts=""
  [ "$tool" = racecheck ] && extra_opts="--racecheck-report all"
  timeout ${SAN_TIMEOUT:-1500} /usr/local/cuda/bin/compute-sanitizer --tool $tool $extra_opts \
      --kernel-name regex:vsbp --error-exitcode 99 --print-limit 50 \
      --log-file gpurun_out/san_${TAG}_${tool}.log \
      python -m pytest -q -p no:cacheprovider "${SEL[@]}" $EXTRA > gpurun_out/san_${TAG}_${tool}.pytest 2>&1
  rc=$?
  echo "$tool rc=$rc; $(tail -1 gpurun_out/san_${TAG}_${tool}.pytest); $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_${TAG}_${tool}.log | tail -1)"
done
