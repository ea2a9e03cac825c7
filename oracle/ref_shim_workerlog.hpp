// Build shim for compiling the reference's proj/src/workload.cpp with GCC 13
// (SURVEY.md Appendix A): Recorder's implicit inline destructor needs the
// complete Recorder::WorkerLog, which the reference defines only inside
// proj/src/instrumentation.cpp:15-22.  Force-included (-include) for that one
// translation unit; the layout must stay identical to the reference's.
#pragma once
#include "batchheap/instrumentation.hpp"

namespace batchheap {
struct Recorder::WorkerLog {
    std::uint32_t worker = 0;
    std::uint64_t next_opid = 1;
    bool op_open = false;
    OpRecord pending;
    std::vector<LockSpan> open_locks;
    std::vector<OpRecord> done;
};
}  // namespace batchheap
