// alsncg/harness.hpp -- drop-in subset of the reference's harness API
// (proj/include/alsncg/harness.hpp:68-72): the per-run trace CSV that
// cmd_train writes and speedup / rank-eval read back (harness.cpp:80-127).
// The rest of the reference harness (cmd_train, speedup tables, rank-eval
// drivers, the CLI) is orchestration around the hot path and is out of scope
// (SURVEY.md section 2 rows 13-14); including this header for those names
// fails at compile time rather than silently.
#pragma once

#include <string>

#include "alsncg/config.hpp"

namespace alsncg::harness {

// Header "iter,loss,grad_norm,elapsed_s,backtracks,shuffled_columns", one row
// per TraceRecord, doubles in %.17g (round-trip exact).  DataError when the
// file cannot be written.
void write_trace_csv(const std::string& path, const ConvergenceTrace& trace);
// Parses what write_trace_csv wrote (header skipped, CRLF and blank lines
// tolerated); DataError on an unreadable file, a row without 6 fields, a bad
// number or an empty trace; records are appended through
// ConvergenceTrace::append (so out-of-order iterations throw logic_error).
ConvergenceTrace read_trace_csv(const std::string& path);
// (last.elapsed - first.elapsed) / (last.iter - first.iter); 0 for a single
// iteration; DataError on an empty trace.
double mean_iteration_seconds(const ConvergenceTrace& trace);

}  // namespace alsncg::harness
