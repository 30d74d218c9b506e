"""paper_1410_1599_b200 -- B200-native multiple-precision Simple / Block /
Strassen / Winograd matrix multiplication and blocked LU (drop-in for the MPFR
reference's mpmm hot path).  See DESIGN.md and include/mpgpu.h."""
from .mpmm import (EXP_ZERO, Algorithm, BlockLUConfig, DeviceError, DeviceGroup, DeviceMatrix, Dims3, DimensionError,
                   DomainError, Error, FastMMConfig, FastMMResult, LUFactors, Matrix, OpCounter,
                   PrecisionContext, RecursionLevel, SingularError, Stats, TopTrace, add, algorithm_name,
                   block_mul, count_fast, count_simple, equal_values, fast_mul, gemm_host, gemm_into, handle, identical,
                   lu_blocked, lu_blocked_host, lu_columnwise, lu_solve, mat_vec_mul, nlimbs_for, pad_even, parse_algorithm,
                   record_words, recursion_plan, set_device, set_stream, simple_mul, solve,
                   solve_columnwise, sub, vec_op, UndefinedMetricError, RelErrorStats, SolutionError,
                   max_rel_error, max_rel_error_solution, one_norm, convert, lu_solve_many,
                   inverse, cond_one, AUTO_NMIN, choose_n_min)
from .matgen import Prng64, from_ints, gen_random, gen_scaled, gen_uniform_full, to_fractions
from .codec import IoError, ParseError, from_hex, read_matrix, to_hex, write_matrix
from .benchdrv import (CSV_HEADER, BenchRecord, LUOutcome, LURequest, MatmulRequest, append_csv, bench_reference,
                       gen_bench_pair, gen_linear_system, gen_lotkin, print_csv, run_lu, run_matmul, ratio_table,
                       format_ratio_csv, format_ratio_table)

__all__ = [n for n in dir() if not n.startswith("_")]
