// Host harness for the NUMA placement helpers of hoststage.cpp
// (tests/test_numa_host.py builds and runs it; no GPU needed).
#include <sched.h>

#include <cstdio>
#include <cstdlib>
#include <string>

#include "hoststage.hpp"

static int fails = 0;
#define CHECK(c)                                                  \
    do {                                                          \
        if (!(c)) {                                               \
            std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c); \
            ++fails;                                              \
        }                                                         \
    } while (0)

int main(int argc, char** argv) {
    using t3b::parse_cpulist;
    CHECK((parse_cpulist("0-3,8,10-11") == std::vector<int>{0, 1, 2, 3, 8, 10, 11}));
    CHECK((parse_cpulist("5") == std::vector<int>{5}));
    CHECK((parse_cpulist("0-1\n") == std::vector<int>{0, 1}));
    CHECK(parse_cpulist("").empty());
    CHECK(parse_cpulist("3-1").empty());
    CHECK(parse_cpulist("a-b").empty());
    // argv[1]: fake sysfs with two nodes; device 0000:1b:00.0 on node 1 (cpus 4-7)
    setenv("T3DES_SYSFS_ROOT", argv[1], 1);
    t3b::NumaNode n = t3b::numa_node_of_pci("0000:1B:00.0");
    CHECK(n.node == 1);
    CHECK((n.cpus == std::vector<int>{4, 5, 6, 7}));
    CHECK(t3b::numa_node_of_pci("0000:99:00.0").node == -1);  // unknown device
    setenv("T3DES_NUMA", "0", 1);
    CHECK(t3b::numa_node_of_pci("0000:1b:00.0").node == -1);  // disabled
    unsetenv("T3DES_NUMA");
    setenv("T3DES_SYSFS_ROOT", argv[2], 1);  // argv[2]: single-node sysfs
    CHECK(t3b::numa_node_of_pci("0000:1b:00.0").node == -1);
    {
        cpu_set_t before, during, after;
        sched_getaffinity(0, sizeof before, &before);
        {
            t3b::NumaBind b(n);
            CHECK(b.active());
            sched_getaffinity(0, sizeof during, &during);
            CHECK(CPU_COUNT(&during) == 4 && CPU_ISSET(4, &during) && !CPU_ISSET(0, &during));
        }
        sched_getaffinity(0, sizeof after, &after);
        CHECK(CPU_EQUAL(&before, &after));
        t3b::NumaBind none(t3b::NumaNode{});
        CHECK(!none.active());
    }
    std::printf(fails ? "failed\n" : "ok\n");
    return fails ? 1 : 0;
}
