"""B200-native video front end of the arXiv 1310.3322 teamwork framework.

motion detection -> (3x3 morphology) -> connected components -> blob
statistics -> mean-shift tracking, as hand-written sm_100a kernels behind a
C ABI (include/trb.h, libtrb.so), mirrored here with the reference's names.
"""
from .api import (ACTIVE, EIGHT, FOUR, LOST, MEAN, MODE, CapacityError, ConfigError, CudaError, InvalidArgument,
                  IoError, Labeling, MotionConfig, MotionDetector, SegmentationConfig, Streams, TeamrecError, Tracker,
                  TrackerConfig, build, device_count, extract_blob_features, histogram, label_blocked,
                  label_sequential, lib,
                  meanshift_step, quantize_colors, synth_raster, warp_frame, decode_pnm, load_pnm,
                  load_frame_sequence, format_track_log, parse_track_log, save_track_log, load_track_log)

__all__ = [
    "ACTIVE", "EIGHT", "FOUR", "LOST", "MEAN", "MODE", "CapacityError", "ConfigError", "CudaError",
    "InvalidArgument", "IoError", "Labeling", "MotionConfig", "MotionDetector", "SegmentationConfig", "Streams",
    "TeamrecError", "Tracker", "TrackerConfig", "build", "device_count", "extract_blob_features", "histogram",
    "label_blocked",
    "label_sequential", "lib", "meanshift_step", "quantize_colors", "synth_raster", "warp_frame", "decode_pnm",
    "load_pnm", "load_frame_sequence", "format_track_log", "parse_track_log", "save_track_log", "load_track_log",
]
