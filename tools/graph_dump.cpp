// Dump the B200-mapped task graph (the one offsim::execute runs) as JSON:
// [{"id","name","resource","work","deps":[...]}] — for offline critical-path
// analysis of executed traces (scripts/critical_path.py).
#include <offsim/exec.hpp>
#include <offsim/offsim.hpp>

#include <fstream>
#include <iostream>
#include <sstream>

int main(int argc, char** argv) {
    if (argc < 2) {
        std::cerr << "usage: graph_dump scenario.json [resident_groups|all]\n";
        return 2;
    }
    std::ifstream f(argv[1]);
    std::stringstream ss;
    ss << f.rdbuf();
    const offsim::Scenario s = offsim::load_scenario(ss.str());
    const offsim::SwapPlan plan = offsim::plan_for_scenario(s);
    const offsim::TaskGraph ref = offsim::build_schedule(s.model, s.hardware, plan, s.variant);
    std::uint32_t resident = 0;
    if (argc > 2) resident = std::string(argv[2]) == "all" ? 0xffffffffu : static_cast<std::uint32_t>(std::stoul(argv[2]));
    offsim::TaskGraph g = offsim::map_graph_for_b200(ref, offsim::StateTier::host, 3, resident);
    offsim::ExecOptions o;
    offsim::add_host_ring_edges(g, offsim::host_ring_depths(g, o));
    std::cout << "[\n";
    for (std::size_t i = 0; i < g.tasks.size(); ++i) {
        const offsim::Task& t = g.tasks[i];
        std::cout << "{\"id\":" << t.id << ",\"name\":\"" << t.name << "\",\"resource\":\""
                  << offsim::to_string(t.resource) << "\",\"work\":" << t.work << ",\"deps\":[";
        for (std::size_t d = 0; d < t.deps.size(); ++d) std::cout << (d ? "," : "") << t.deps[d];
        std::cout << "]}" << (i + 1 < g.tasks.size() ? ",\n" : "\n");
    }
    std::cout << "]\n";
    return 0;
}
