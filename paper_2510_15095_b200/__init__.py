"""B200-native Hive hash table (arXiv 2510.15095): sm_100a CUDA behind a C ABI
(include/hive.h, libhive.so) with a thin ctypes binding."""
from .hive import (HIVE_KEYS_UNIQUE, INVALID_KEY, OP_ERASE, OP_FIND, OP_INSERT, HiveError,  # noqa: F401
                   HiveTable, lib, route, u8, u32, unpack_kv, unroute)
