// offsim command-line client of the B200 library — links the C ABI only
// (like the reference CLI, proj/tools/CMakeLists.txt:2), same subcommands
// and exit codes (0 ok, 2 config, 3 infeasible, 4 invariant), plus
// `execute`, which runs the scenario's task graph on the GPU
// (offsim_execute) instead of simulating it.
//
//   offsim plan      --preset 13b-a100-b32
//   offsim simulate  --preset 13b-a100-b64 [--trace trace.json]
//   offsim execute   --scenario s.json [--exec '{"tier":"file"}'] [--trace t.json]
//   offsim sweep     --preset 13b-a100-b32 --axis batch_size --values 8,16,32,64
//   offsim capacity  --preset 13b-a100-b32 --cpu-mem-gb 128,256,512
//   offsim validate  --preset 13b-a100-b32
//   offsim presets
// Common: --variant serial|pipelined|overlapped, --batch N, --n-ssd N,
// --planner auto|<coef>, --out FILE, --workers N.

#include "offsim/offsim_c.h"

#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

namespace {

int usage() {
    std::fprintf(stderr,
                 "usage: offsim <plan|simulate|execute|sweep|capacity|validate|presets> "
                 "[--preset NAME | --scenario FILE] [--variant V] [--batch N] [--n-ssd N] "
                 "[--planner auto|C] [--axis A --values v1,v2] [--cpu-mem-gb g1,g2] "
                 "[--workers N] [--exec JSON] [--trace FILE] [--out FILE]\n");
    return 2;
}

int fail(int status) {
    std::fprintf(stderr, "offsim: %s\n", offsim_last_error());
    return status;
}

std::vector<double> numbers(const std::string& csv) {
    std::vector<double> out;
    std::stringstream ss(csv);
    for (std::string item; std::getline(ss, item, ',');) out.push_back(std::strtod(item.c_str(), nullptr));
    return out;
}

void emit(const std::map<std::string, std::string>& flags, const char* text) {
    const auto it = flags.find("--out");
    if (it == flags.end()) {
        std::fputs(text, stdout);
        return;
    }
    std::ofstream(it->second) << text;
}

} // namespace

int main(int argc, char** argv) {
    if (argc < 2) return usage();
    const std::string cmd = argv[1];
    std::map<std::string, std::string> flags;
    for (int i = 2; i < argc; ++i) {
        const std::string k = argv[i];
        if (k.rfind("--", 0) != 0 || i + 1 >= argc) return usage();
        flags[k] = argv[++i];
    }
    if (cmd == "presets") {
        char* names = nullptr;
        if (int st = offsim_preset_names(&names)) return fail(st);
        std::fputs(names, stdout);
        offsim_string_free(names);
        return 0;
    }

    offsim_scenario* sc = nullptr;
    if (flags.count("--preset")) {
        if (int st = offsim_scenario_from_preset(flags["--preset"].c_str(), &sc)) return fail(st);
    } else if (flags.count("--scenario")) {
        std::ifstream in(flags["--scenario"]);
        if (!in) {
            std::fprintf(stderr, "offsim: cannot read %s\n", flags["--scenario"].c_str());
            return 2;
        }
        std::stringstream text;
        text << in.rdbuf();
        if (int st = offsim_scenario_parse(text.str().c_str(), &sc)) return fail(st);
    } else {
        return usage();
    }
    const std::pair<const char*, const char*> overrides[] = {
        {"--variant", "variant"}, {"--batch", "batch_size"}, {"--n-ssd", "n_ssd"}, {"--planner", "planner"}};
    for (const auto& [flag, key] : overrides)
        if (flags.count(flag))
            if (int st = offsim_scenario_override(sc, key, flags[flag].c_str())) return fail(st);

    char* out = nullptr;
    char* trace = nullptr;
    const bool want_trace = flags.count("--trace") > 0;
    int st = 0;
    if (cmd == "plan") {
        st = offsim_plan(sc, &out);
    } else if (cmd == "simulate") {
        st = offsim_simulate(sc, &out, want_trace ? &trace : nullptr);
    } else if (cmd == "execute") {
        const std::string opts = flags.count("--exec") ? flags["--exec"] : "";
        st = offsim_execute(sc, opts.empty() ? nullptr : opts.c_str(), &out, want_trace ? &trace : nullptr);
    } else if (cmd == "validate") {
        st = offsim_validate(sc, &out);
    } else if (cmd == "sweep") {
        if (!flags.count("--axis") || !flags.count("--values")) return usage();
        const std::vector<double> v = numbers(flags["--values"]);
        const int workers = flags.count("--workers") ? std::atoi(flags["--workers"].c_str()) : 1;
        st = offsim_sweep(sc, flags["--axis"].c_str(), v.data(), v.size(), workers, &out);
    } else if (cmd == "capacity") {
        const std::vector<double> v = numbers(flags.count("--cpu-mem-gb") ? flags["--cpu-mem-gb"] : "768");
        st = offsim_capacity(sc, v.data(), v.size(), &out);
    } else {
        offsim_scenario_free(sc);
        return usage();
    }
    if (out) emit(flags, out);
    if (trace) std::ofstream(flags["--trace"]) << trace;
    offsim_string_free(out);
    offsim_string_free(trace);
    offsim_scenario_free(sc);
    return st ? fail(st) : 0;
}
