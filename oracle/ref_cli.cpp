// TEST INFRASTRUCTURE ONLY — never linked into or called by the product path.
//
// The reference command line's text-mode reporting (tools/cohere_main.cpp), driven through
// the UNMODIFIED reference headers, so golden CLI outputs can be produced here for any
// program text (the reference CLI itself needs CLI11 and nlohmann/json, which are not in
// this image: SURVEY §8(c)).  Built into oracle/_ref/libcohere_ref.so with ref_harness.cpp.
//
// ref_cli(command, src, raw, no_overlap, fuel, schedule, trace, out, out_cap, err, err_cap, &exit)
// follows cmd_check / cmd_run / cmd_infer / cmd_translate and the exception-to-exit-code
// mapping of main() (tools/cohere_main.cpp:80-274), text output only.
#include <cstring>
#include <sstream>
#include <string>

#include "cohere/cohere.hpp"

using namespace cohere;

namespace {

void put(const std::string& s, char* buf, size_t cap) {
  if (!buf || !cap) return;
  const size_t n = s.size() < cap - 1 ? s.size() : cap - 1;
  std::memcpy(buf, s.data(), n);
  buf[n] = '\0';
}

std::string diag_line(const std::string& rule, const std::string& view, SourcePos pos, const std::string& msg) {
  return std::to_string(pos.line) + ":" + std::to_string(pos.col) + ": " + rule + " [" + view + "] " + msg + "\n";
}

int report(const RunResult& r, bool schedule_given, bool trace, std::ostringstream& out, std::ostringstream& err) {
  if (trace) {
    int idx = 0;
    for (const auto& step : r.trace) {
      std::ostringstream line;
      line << ++idx << " " << name_of(step.rule);
      while (line.str().size() < 16) line << " ";
      line << to_string(step.head);
      const char* sep = " => ";
      for (const auto& [key, pair] : step.delta) {
        line << sep << to_string(key) << "=" << to_string(pair);
        sep = " ";
      }
      out << line.str() << "\n";
    }
  }
  out << "outcome: " << name_of(r.status) << "\n";
  out << "steps: " << r.steps << "\n";
  if (r.stuck) out << "stuck at: " << r.stuck->describe() << "\n";
  for (const auto& [key, pair] : r.store) out << to_string(key) << " " << to_string(pair) << "\n";
  if (r.schedule_overflowed && schedule_given) err << "note: schedule exhausted; later opaque conditions answered false\n";
  switch (r.status) {
    case RunStatus::Done: return 0;
    case RunStatus::Stuck: return 3;
    case RunStatus::FuelExhausted: return 4;
  }
  return 0;
}

int command(const std::string& cmd, const std::string& src, bool raw, bool no_overlap, int fuel,
            const std::string& schedule, bool trace, std::ostringstream& out, std::ostringstream& err) {
  if (cmd == "check") {
    if (raw) {
      RawProgram p = parse_raw(src);
      DeclBlock pseudo({}, p.body);
      auto diags = check_localised(pseudo);
      for (const auto& d : diags) out << diag_line(d.rule, d.view, d.pos, d.message);
      return diags.empty() ? 0 : 1;
    }
    AnnotatedProgram p = parse_program(src);
    OverlapRegistry reg = no_overlap ? OverlapRegistry() : build_registry(p.decls);
    auto diags = check_program(p, reg);
    for (const auto& d : diags) out << diag_line(d.rule, d.view, d.pos, d.message);
    for (const auto& n : check_notes(p)) out << "note: " << diag_line(n.rule, n.view, n.pos, n.message);
    return diags.empty() ? 0 : 1;
  }
  if (cmd == "run" || cmd == "trace") {
    trace = trace || cmd == "trace";
    const TraceMode mode = trace ? TraceMode::Full : TraceMode::None;
    Schedule sched = Schedule::from_string(schedule);
    if (raw) {
      RawProgram p = parse_raw(src);
      return report(run(p, fuel, sched, mode), !schedule.empty(), trace, out, err);
    }
    AnnotatedProgram p = parse_program(src);
    OverlapRegistry reg = no_overlap ? OverlapRegistry() : build_registry(p.decls);
    if (!no_overlap) p = rewrite_program(p, reg);
    auto diags = check_program(p, reg);
    if (!diags.empty()) {
      for (const auto& d : diags) err << diag_line(d.rule, d.view, d.pos, d.message);
      return 1;
    }
    return report(run(translate_program(p), initial_store(p.decls), fuel, sched, mode), !schedule.empty(), trace, out,
                  err);
  }
  if (cmd == "infer" || cmd == "translate") {
    if (raw) throw std::runtime_error(cmd + " needs an annotated program");
    AnnotatedProgram p = parse_program(src);
    if (!no_overlap) p = rewrite_program(p, build_registry(p.decls));
    if (cmd == "infer") {
      out << pretty(p);
    } else {
      for (size_t i = 0; i < p.blocks.size(); ++i)
        out << "block " << i << ": " << to_string(translate_block(p.blocks[i], p.decls)) << "\n";
    }
    return 0;
  }
  throw std::runtime_error("unknown command");
}

}  // namespace

extern "C" int ref_cli(const char* cmd, const char* src, int raw, int no_overlap, int fuel, const char* schedule,
                       int trace, char* out, size_t out_cap, char* err, size_t err_cap, int* exit_code) {
  std::ostringstream o, e;
  int code;
  try {
    code = command(cmd, src, raw != 0, no_overlap != 0, fuel, schedule ? schedule : "", trace != 0, o, e);
  } catch (const ParseError& x) {
    e << "error: " << x.what() << "\n";
    code = 2;
  } catch (const OverlapInferenceError& x) {
    e << "error: " << x.what() << "\n";
    code = 1;
  } catch (const ConstructionError& x) {
    e << "error: " << x.what() << "\n";
    code = 2;
  } catch (const std::exception& x) {
    e << "error: " << x.what() << "\n";
    code = 2;
  }
  put(o.str(), out, out_cap);
  put(e.str(), err, err_cap);
  *exit_code = code;
  return (o.str().size() >= out_cap || e.str().size() >= err_cap) ? -1 : 0;
}

// Acceptance criterion 1 (tests/acceptance.cpp:107-138) through the reference itself:
// enumerate_raw_programs + run from initial_store, one status per program (RunStatus
// ordinals), and whether any step left a key (I,I) (checked after every step of a traced run).
extern "C" int ref_enum_straight_line(int max_len, int fuel, unsigned char* statuses, long cap, long* unsafe_programs) {
  EnumLimits limits;
  limits.max_len = max_len;
  std::vector<Stmt> programs = enumerate_raw_programs(limits);
  Declarations d;
  d.add_scalar({"x", {}});
  const Store s0 = initial_store(d);
  long unsafe = 0;
  for (size_t i = 0; i < programs.size(); ++i) {
    RunResult r = run(programs[i], s0, fuel, Schedule(), TraceMode::Full);
    Store s = s0;
    bool bad = is_unsafe(s);
    for (const auto& step : r.trace)
      for (const auto& [key, pair] : step.delta) bad = bad || pair == kBothInvalid;
    unsafe += bad ? 1 : 0;
    if ((long)i < cap) statuses[i] = (unsigned char)r.status;
  }
  *unsafe_programs = unsafe;
  return (int)programs.size();
}
