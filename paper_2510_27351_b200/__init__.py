"""B200-native (sm_100a) FP64 tridiagonal partition solver — a drop-in for the
reference `tridpart` solver path (arXiv 2510.27351). See DESIGN.md."""
from .tridpart import (  # noqa: F401
    BadNumberError, Block, Context, DepthOutOfRangeError, DeviceError, EmptyTrainingSetError,
    Error, HeuristicModel, InvalidSizeError, KTooLargeError, MalformedHeaderError, Observation,
    ObservationSet, PartitionPlan, RecursionPolicy, SchemaError, TrainingPair, Tridiagonal,
    TridiagonalSystem, VersionMismatchError, ZeroPivotError, check_device_error, context,
    b200_size_model, default_depth_model, default_fp32_size_model, default_size_model, fit_depth_model, fit_knn,
    generate_system,
    kMaxRecursionDepth, kModelFormatVersion, kPivotFloor, load_model, make_plan, plan_levels,
    predict, predicted_policy, read_observations, recursion_sizes, residual_inf, save_model,
    solve_partition, solve_partition_async, thomas_solve, torch_stream,
    ReducedBlock, reduce_block, assemble_interface, back_substitute)

__version__ = "0.2.0"
