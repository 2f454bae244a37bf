"""paper_2411_07351_b200 -- B200-native (sm_100a) FHT2D merge DP (arXiv 2411.07351).

The hot path of the reference (transform_columns, transform.cpp:35-58, driven
by fht2d_counted and fht2d_quadrants) as hand-written CUDA kernels behind a
C ABI (include/fht_b200.h).  See DESIGN.md.
"""
from .fht import (CountedTransform, InvalidArgument, OverflowBudget, Pattern, Plan, QUADRANTS, QuadrantSet,
                  SplitStrategy, check_overflow_budget, count_additions_tree, fht2d, fht2d_counted, fht2d_pattern,
                  fht2d_quadrants, pattern_set, round_half_up_ratio, slow_hough, slow_hough_device, split_simple,
                  split_tweaked, split_width, strategy_from_string)

__all__ = ["CountedTransform", "InvalidArgument", "OverflowBudget", "Pattern", "Plan", "QUADRANTS", "QuadrantSet",
           "fht2d_pattern", "pattern_set", "slow_hough", "slow_hough_device",
           "SplitStrategy", "check_overflow_budget", "count_additions_tree", "fht2d", "fht2d_counted",
           "fht2d_quadrants", "round_half_up_ratio", "split_simple", "split_tweaked", "split_width",
           "strategy_from_string"]
