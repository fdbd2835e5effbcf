"""lazypca_b200: B200-native Lazy SPCA / SPCA / random projection.

The product is the C-ABI library liblazypca_b200.so (include/lazypca_b200.h),
hand-written CUDA for sm_100a behind the reference `lazypca` entry points.
This package is the Python mirror of that API (see api.py) plus the build.
"""
from .api import (  # noqa: F401
    Context, ConvergenceError, CudaError, DensityPolicy, DimensionError, EigenDecomposition, Error,
    InvalidArgumentError, NcclError, ParseError, ProjectionKind, ProjectionMatrix, ProjectionSpec,
    RankDeficiencyError, ReducerConfig, ReducerMethod, ReducerTimings, ReductionMap, SketchMatrix,
    SparseMatrix, TruncatedSVD, apply_map, build_sketch, default_context, dense_aat, density_for, eigh,
    fit_transform, gemm_t, gemm_t_f32, gen_gaussian, gen_very_sparse, jacobi_eigh, projection_kind_from_string,
    reduce, reduce_lazy_spca, reduce_lazy_spca_streaming, reduce_rp, reduce_spca, reduce_spca_streaming,
    reducer_method_from_string, regenerate, RowBlock, RowBlockStream, SliceRowBlockStream, split_rows,
    load_map_file, read_map_file, save_map_file, write_map_file, chordal_distance, distance_preservation,
    DistancePreservationReport, ReconstructionErrorReport, ResidualRoute, bound_value, reconstruction_error,
    row_space_reconstruction_error, spectral_norm, read_sparse_matrix_market, read_dense_matrix_market,
    read_dense_csv, write_sparse_matrix_market, write_dense_matrix_market, write_dense_csv,
    MatrixMarketRowBlockStream, CsvRowBlockStream,
    set_thread_count, sketch_f32, spmm, synth_lowrank, thread_count, to_string, tridiag_eigh,
    truncated_svd_via_gram,
)
