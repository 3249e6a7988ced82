// Adapter shim -- TEST INFRASTRUCTURE ONLY. Placed ahead of the reference's
// include directory, it makes the UNMODIFIED reference sources (Scheduler,
// SimEngine, and its own doctest suites) compile against the B200 block pool:
// the reference header is included under a renamed class
// (KvCacheManager -> KvCacheManagerReference, still defined by the reference's
// kv_cache.cpp, which the same Makefile compiles with that rename), and
// coserve::KvCacheManager becomes the C-ABI adapter of include/conserve_b200_kv.hpp.
#pragma once
#define KvCacheManager KvCacheManagerReference
#include_next <coserve/kv_cache.hpp>
#undef KvCacheManager
#include "conserve_b200_kv.hpp"
namespace coserve {
using KvCacheManager = ::conserve_b200::KvCacheManager;
}
